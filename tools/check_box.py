"""GPU check of the box solve at every supported size: error against the
oracle's scipy box solve and device time per solve.  M = 16384 runs the f64 case only
(host memory of the scipy oracle).

    python tools/check_box.py [sizes...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402
from oracle import kfbi_oracle as O  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [16, 32, 64, 128, 256, 512, 1024, 2048, 4096]
eng = os.environ.get("KFBI_COLS", "tridiagonal")
rng = np.random.default_rng(0)
for m in sizes:
    grid = k.CartesianGrid((-1.5, 1.5, -1.5, 1.5), m)
    for cplx in ((False, True) if m <= 8192 else (False,)):
        kappa = 2j * m if cplx else 2.0 * m
        rhs = rng.standard_normal((m + 1, m + 1))
        if cplx:
            rhs = rhs + 1j * rng.standard_normal((m + 1, m + 1))
        solver = k.BoxSolver(grid, kappa, "dirichlet-zero")
        solver.plan.set_colsolver(eng)
        u = solver.solve(rhs)
        ref = O.box_solve(m, grid.h, kappa, rhs)
        err = np.max(np.abs(u - ref)) / np.max(np.abs(ref))
        ring = max(np.max(np.abs(u[0])), np.max(np.abs(u[-1])), np.max(np.abs(u[:, 0])),
                   np.max(np.abs(u[:, -1])))
        rd = torch.from_numpy(rhs).cuda()
        for _ in range(3):
            solver.solve(rd)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        a.record()
        for _ in range(reps):
            solver.solve(rd)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        # column pass alone (transform-cols) from the plan's per-name event timings
        pl = solver.plan
        pl.set_timing(True)
        pl.reset_kernel_times()
        for _ in range(reps):
            solver.solve(rd)
        torch.cuda.synchronize()
        kms, kc = pl.kernel_times()
        cols = kms["transform-cols"] / max(kc["transform-cols"], 1)
        rows = kms["transform-rows"] / max(kc["transform-rows"], 1)
        s = 16 if cplx else 8
        gbs = 2 * (m - 1) ** 2 * s / (cols / 1e3) / 1e9
        print(f"[{eng}] M={m:5d} {'c128' if cplx else 'f64 '} rel_err={err:.2e} ring={ring:.1e} "
              f"{ms:.4f} ms/solve  cols {cols * 1e3:.1f} us ({gbs:.0f} GB/s)  rows {rows * 1e3:.1f} us",
              flush=True)
