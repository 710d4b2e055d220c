"""GMRES vs Richardson on static BVPs: iterations, agreement, max_iter path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402

for m, kappa in ((128, 16.0), (1024, 2048.0), (4096, 512.0)):
    geo = k.build_grid((-1.5, 1.5, -1.5, 1.5), m, k.StarCurve(1.0, c=0.2, lobes=8))
    ws = k.InterfaceWorkspace(geo)
    sol = k.StaticPlaneWave(kappa=kappa)
    cps = ws.cps
    F = np.where(geo.classification.interior, sol.f(geo.grid.X, geo.grid.Y), 0.0)
    prob = k.BvpProblem(kappa=kappa, F=F, f_gamma=sol.f(cps.x, cps.y), bc_kind="dirichlet",
                        bc_values=sol.dirichlet(cps.x, cps.y))
    r = k.richardson_solve(prob, ws)
    for restart in (8, 20, 40):
        g = k.gmres_solve(prob, ws, restart=restart)
        d = np.max(np.abs(g.u - r.u)) / np.max(np.abs(r.u))
        print(f"M={m} kappa={kappa} n_ctl={cps.m} richardson {r.iterations} sweeps; gmres({restart}) "
              f"{g.iterations} (matvecs+sweeps) res {g.residual:.2e} rel diff {d:.2e} "
              f"hist {[f'{h:.1e}' for h in g.residual_history[:6]]}", flush=True)
    prob.max_iter = 2
    try:
        g = k.gmres_solve(prob, ws)
        print("max_iter=2: no error", g.iterations, g.residual, g.residual_history)
    except k.ConvergenceError as e:
        print("max_iter=2: ConvergenceError", e)
