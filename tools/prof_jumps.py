"""One pipeline Richardson solve (3 sweeps) of the bench's heat / Schrödinger
step at M (default 4096), for ncu captures of the jumps / edge-value kernels:

    ncu --set full -k regex:"spec_block|edges_spectral|circ_block|corr_edges" \
        python tools/prof_jumps.py [M] [heat|schrodinger]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200.bvp import solve_device  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
eq = sys.argv[2] if len(sys.argv) > 2 else "heat"
box, curve, kw = bench.workload(m)[eq]
ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
cplx = eq == "schrodinger"
dt = torch.complex128 if cplx else torch.float64
kappa = 2j * m if cplx else 2.0 * m
n = ws.cps.m
g = torch.Generator(device="cuda").manual_seed(0)
F = torch.randn((m + 1) * (m + 1), generator=g, device="cuda", dtype=dt)
fg = torch.randn(n, generator=g, device="cuda", dtype=dt)
gb = torch.randn(n, generator=g, device="cuda", dtype=dt)
for _ in range(2):
    dens = torch.zeros(n, dtype=dt, device="cuda")
    try:
        solve_device(ws, kappa=kappa, F=F, f_gamma=fg, g=gb, density=dens, max_iter=3, tol=1e-30)
    except Exception as e:      # max_iter reached: expected
        pass
torch.cuda.synchronize()
print("done", eq, m, n, "spectral" if ws.plan.spectral_edges else "w rows")
