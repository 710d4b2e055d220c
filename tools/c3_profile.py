"""cProfile of one C3 run() (context reused, operator form, captured step)."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402

desc, box, m, curve, kw = bench.config_cases()["C3"]
geo = k.build_grid(box, m, curve)
spec = k.ProblemSpec(**kw)
ctx = k.StepContext(geo, backend=k.CudaBackend(0, timing=False))
k.run(spec, geo, context=ctx)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
k.run(spec, geo, context=ctx)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
