"""C1 (heat flower8 128^2, tau 0.01, 100 steps) through run() with and
without the captured step: wall time per run (context reused), several runs.

    python tools/graph_probe.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402
from conftest import run_cases  # noqa: E402

for name in ("c1_heat_flower128", "wave_ellipse128"):
    box, m, curve, kw = run_cases()[name]
    geo = k.build_grid(box, m, curve)
    for graph in (False, True, False, True):
        ctx = k.StepContext(geo, backend=k.CudaBackend(0, timing=False))
        spec = k.ProblemSpec(**kw)
        k.run(spec, geo, context=ctx, operator=True, graph=graph)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = k.run(spec, geo, context=ctx, operator=True, graph=graph)
            ts.append(time.perf_counter() - t0)
        n = len(res.iterations)
        best = min(ts)
        print(f"{name} graph={graph}: {n} steps, best {best * 1e3:.1f} ms = {n / best:.0f} steps/s "
              f"(runs {[round(x * 1e3, 1) for x in ts]}), sweeps {sum(res.iterations)}", flush=True)
# where the time goes in one captured step (host side)
box, m, curve, kw = run_cases()["c1_heat_flower128"]
geo = k.build_grid(box, m, curve)
ctx = k.StepContext(geo, backend=k.CudaBackend(0, timing=False))
spec = k.ProblemSpec(**kw)
k.run(spec, geo, context=ctx, operator=True, graph=True)
sg = ctx._step_graph
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    sg.advance()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"advance(): host {1e6 * (t1 - t0) / 200:.1f} us/step, device-drained {1e6 * (t2 - t0) / 200:.1f} us/step")
ctx._pending.clear()
