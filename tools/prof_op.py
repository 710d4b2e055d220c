"""Profiling driver for the operator-form Richardson sweeps: a few heat steps
at one size with the trace operator built.  python tools/prof_op.py [M] [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200.timestepping import heat_startup, heat_step  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
heat = k.HeatPlaneDecay()
tau = 16.0 / m
geo = k.build_grid((-1.5, 1.5, -1.5, 1.5), m, k.StarCurve(1.0, 0.2, 8))
spec = k.ProblemSpec(equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                     lap_u0=heat.lap_u0, tau=tau, t_final=1000 * tau)
ctx = k.StepContext(geo, operator=True)
t0 = time.time()
ctx.workspace.ensure_operator(2.0 / tau, False)
torch.cuda.synchronize()
print(f"operator build M={m} n_ctl={ctx.n_ctl}: {time.time() - t0:.2f} s", flush=True)
st = heat_startup(spec, ctx)
for _ in range(steps):
    st = heat_step(st, spec, ctx)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    st = heat_step(st, spec, ctx)
b.record()
torch.cuda.synchronize()
print(f"heat step M={m}: {a.elapsed_time(b) / steps:.3f} ms, sweeps {st.last_iterations}")
