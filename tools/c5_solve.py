"""C5 (BASELINE.json configs[4]) on one GPU: one modified-Helmholtz KFBI
solve at M = 16384 (flower star on [-1.5, 1.5]^2, StaticPlaneWave, kappa =
2/tau with tau = 1/1024), timed: host setup, device Richardson solve, the
slab-decomposed box solve (P virtual ranks) vs the one-GPU box solve.

    python tools/c5_solve.py [M]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200 import dist as D  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
kappa = 2.0 * 1024
box = (-1.5, 1.5, -1.5, 1.5)
out = {"m": m, "kappa": kappa}
t0 = time.time()
geo = k.build_grid(box, m, k.StarCurve(1.0, c=0.2, lobes=8))
ws = k.InterfaceWorkspace(geo)
out["setup_s"] = time.time() - t0
out["n_ctl"] = int(ws.cps.m)
sol = k.StaticPlaneWave(kappa=kappa)
cps = ws.cps
X, Y = geo.grid.X, geo.grid.Y
F = np.where(geo.classification.interior, sol.f(X, Y), 0.0)
prob = k.BvpProblem(kappa=kappa, F=F, f_gamma=sol.f(cps.x, cps.y), bc_kind="dirichlet",
                    bc_values=sol.dirichlet(cps.x, cps.y))
t0 = time.time()
res = k.richardson_solve(prob, ws)
out["first_solve_s"] = time.time() - t0
torch.cuda.synchronize()
t0 = time.time()
res = k.richardson_solve(prob, ws)
out["solve_s"] = time.time() - t0
out["iterations"] = int(res.iterations)
inside = geo.classification.interior
err = np.max(np.abs(res.u[inside] - sol.u(X, Y)[inside]))
out["max_err_interior"] = float(err)
del X, Y, F
# box solve: one GPU vs P virtual slabs (bit-identical), device time
grid = geo.grid
rhs = torch.randn((m + 1, m + 1), dtype=torch.float64, device="cuda")
bs = k.BoxSolver(grid, kappa, "dirichlet-zero")
ref = bs.solve(rhs)
for _ in range(2):
    bs.solve(rhs)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    bs.solve(rhs)
b.record()
torch.cuda.synchronize()
out["box_solve_ms"] = a.elapsed_time(b) / 5
for p in (2, 8):
    u = D.solve_virtual(grid, kappa, rhs, p)
    out[f"virtual_slabs_{p}_bit_identical"] = bool(torch.equal(u, ref))
print(json.dumps(out), flush=True)
