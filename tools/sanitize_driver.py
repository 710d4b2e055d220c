"""Small invocations of every hot-path kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): box solves (tridiagonal and DST column
stages, DCT-I), a Dirichlet Richardson solve, heat and Schrodinger runs in
the operator form (op_solve_* kernels and the hand-rolled grid barrier), a
Neumann heat run, GMRES, the slab passes with fused peer stores and the
peer-flag barrier (two virtual ranks on two streams), and the reduced-work
FACR paths at 512² (trace-only and masked sweeps, graphs, one-CTA sweeps)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200 import _native as N  # noqa: E402
from paper_2404_14864_b200 import dist as D  # noqa: E402

BOX = (-1.5, 1.5, -1.5, 1.5)
PI_BOX = (-np.pi, np.pi, -np.pi, np.pi)
m = int(os.environ.get("SAN_M", "128"))
rng = np.random.default_rng(0)
grid = k.CartesianGrid(BOX, m)
for kappa in (2048.0, 0.5, 512j):
    for bc in ("dirichlet-zero", "neumann-zero"):
        s = k.BoxSolver(grid, kappa, bc)
        for mode in ("auto", "tridiagonal", "dst"):
            s.plan.set_colsolver(mode)
            s.solve(rng.standard_normal((m + 1, m + 1)))
        s.plan.set_colsolver("auto")
print("box ok", flush=True)

geo = k.build_grid(BOX, m, k.StarCurve(1.0, c=0.2, lobes=5))
ws = k.InterfaceWorkspace(geo)
sol = k.StaticPlaneWave(kappa=32.0)
cps = ws.cps
F = np.where(geo.classification.interior, sol.f(geo.grid.X, geo.grid.Y), 0.0)
prob = k.BvpProblem(kappa=32.0, F=F, f_gamma=sol.f(cps.x, cps.y), bc_kind="dirichlet",
                    bc_values=sol.dirichlet(cps.x, cps.y))
k.richardson_solve(prob, ws)
k.gmres_solve(prob, ws, restart=8)
print("bvp ok", flush=True)

heat = k.HeatPlaneDecay()
spec = k.ProblemSpec(equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                     lap_u0=heat.lap_u0, tau=1 / 64, t_final=3 / 64)
k.run(spec, geo, operator=True)
nspec = k.ProblemSpec(equation="heat", bc_kind="neumann", g=heat.neumann, u0=heat.u0,
                      lap_u0=heat.lap_u0, tau=1 / 64, t_final=2 / 64)
k.run(nspec, geo, operator=True)
schr = k.SchrodingerPhaseRotation()
pgeo = k.build_grid(PI_BOX, m, k.StarCurve(1.5, c=0.2, lobes=3))
sspec = k.ProblemSpec(equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
                      lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=1 / 32, t_final=2 / 32)
k.run(sspec, pgeo, operator=True)
print("runs ok", flush=True)

# the reduced-work FACR paths need M >= 512: trace-only sweeps
# (rows_odd_facr_sparse, row_need, zero-row flags), the masked final sweep
# (field chunks), zero-exterior rings, CUDA-graph steps, one-CTA operator
# sweeps, and the pipeline form's trace-only sweeps + final pipeline
m2 = int(os.environ.get("SAN_M2", "512"))
geo2 = k.build_grid(BOX, m2, k.StarCurve(1.0, c=0.2, lobes=8))
spec2 = k.ProblemSpec(equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                      lap_u0=heat.lap_u0, tau=1 / 256, t_final=4 / 256)
for op in (True, False):
    ctx2 = k.StepContext(geo2, backend=k.CudaBackend(0, timing=False), operator=op)
    k.run(spec2, geo2, context=ctx2, operator=op, graph="auto" if op else False)
pgeo2 = k.build_grid(PI_BOX, m2, k.StarCurve(1.5, c=0.2, lobes=3))
sspec2 = k.ProblemSpec(equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
                       lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=1 / 128, t_final=3 / 128)
ctx3 = k.StepContext(pgeo2, backend=k.CudaBackend(0, timing=False), operator=True)
k.run(sspec2, pgeo2, context=ctx3, operator=True, graph="auto")
print("reduced-work runs ok", flush=True)

rhs = torch.from_numpy(rng.standard_normal((m + 1, m + 1))).cuda()
D.solve_virtual(grid, 40.0, rhs, 2, p2p=True)
D.solve_virtual(grid, 40.0, rhs, 2, p2p=False)
lib = N.lib()
flags = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(2)]
tab = (C.c_void_p * 2)(*[f.data_ptr() for f in flags])
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(2)]
for epoch in (1, 2):
    for r in (1, 0):
        N.check(lib.kfbi_p2p_barrier(tab, 2, r, epoch, 1 << 26, bad.data_ptr(), streams[r].cuda_stream))
    torch.cuda.synchronize()
assert int(bad.item()) == 0
print("slab/p2p ok", flush=True)
