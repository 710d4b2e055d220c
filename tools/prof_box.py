"""Profiling driver: a few box solves (and optionally operator sweeps) at one
size, for ncu captures of the DST kernels in isolation.

    python tools/prof_box.py [M] [reps] [real|complex]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cplx = len(sys.argv) > 3 and sys.argv[3] == "complex"
grid = k.CartesianGrid((-1.5, 1.5, -1.5, 1.5), m)
dt = torch.complex128 if cplx else torch.float64
rhs = torch.randn((m + 1, m + 1), dtype=dt, device="cuda")
solver = k.BoxSolver(grid, 2j * m if cplx else 2.0 * m, "dirichlet-zero")
for _ in range(reps):
    u = solver.solve(rhs)
torch.cuda.synchronize()
start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
start.record()
for _ in range(reps):
    u = solver.solve(rhs)
end.record()
torch.cuda.synchronize()
print(f"box solve M={m} {'c128' if cplx else 'f64'}: {start.elapsed_time(end) / reps:.3f} ms")
