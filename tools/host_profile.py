"""Host-side cost of the bench loop (3 streams, 4096^2): cProfile of K bench
steps, top functions by own time and cumulative time.

    python tools/host_profile.py [K]
"""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import streams_probe as sp  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for eq in sp.eqs:
    kap = {"heat": 2.0 * sp.specs[eq].c / sp.specs[eq].tau,
           "wave": 1.0 / (sp.specs[eq].theta * sp.specs[eq].tau ** 2),
           "schrodinger": 2j / sp.specs[eq].tau}[eq]
    sp.ctxs[eq].workspace.ensure_operator(kap, eq == "schrodinger")
sp.K = K
sp.loop(True)
sp.fresh(True)
pr = cProfile.Profile()
pr.enable()
sp.loop(True, do_fresh=False)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(35)
