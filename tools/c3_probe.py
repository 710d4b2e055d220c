"""C3 (Schrödinger Strang, star3, 2048^2, tau 1/128) through run(): the
marginal cost per step (two run lengths, context reused), with and without
the captured step.   python tools/c3_probe.py"""
import dataclasses
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402

for name, (desc, box, m, curve, kw) in bench.config_cases().items():
    geo = k.build_grid(box, m, curve)
    spec = k.ProblemSpec(**kw)
    be = k.CudaBackend(0, timing=False)
    for graph in (False, True):
        ctx = k.StepContext(geo, backend=be)
        k.run(spec, geo, context=ctx, graph=graph, operator=True)
        walls = {}
        for nsteps in (16, 64):
            sp = dataclasses.replace(spec, t_final=nsteps * spec.tau)
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                k.run(sp, geo, context=ctx, graph=graph, operator=True)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            walls[nsteps] = best
        per = (walls[64] - walls[16]) / 48
        print(f"{name} m={m} graph={graph}: fixed {1e3 * (walls[16] - 16 * per):.1f} ms per run, "
              f"{1e3 * per:.3f} ms per step ({1 / per:.0f} steps/s marginal)", flush=True)
