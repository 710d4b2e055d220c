"""Small box solves in every column mode (compute-sanitizer target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [16, 64, 256]
for m in sizes:
    grid = k.CartesianGrid((-1.5, 1.5, -1.5, 1.5), m)
    for kappa in (0.0, 2048.0, 512j):
        rhs = np.random.default_rng(m).standard_normal((m + 1, m + 1))
        for mode in ("auto", "tridiagonal", "dst"):
            s = k.BoxSolver(grid, kappa, "dirichlet-zero")
            s.plan.set_colsolver(mode)
            u = s.solve(rhs)
            print(m, kappa, mode, float(np.abs(u).max()), flush=True)
        s.plan.set_colsolver("auto")
