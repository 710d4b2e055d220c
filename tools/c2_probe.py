"""C2 (wave 1024^2, 64 steps) through run(): fresh-context and reused-context
wall times, repeated (checks the configs' steady-rate number)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402

desc, box, m, curve, kw = bench.config_cases()["C2"]
backend = k.CudaBackend(0, timing=False)
geo = k.build_grid(box, m, curve)
spec = k.ProblemSpec(**kw)
k.run(spec, geo, backend=backend)
ctx = k.StepContext(geo, backend=backend)
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k.run(spec, geo, backend=backend)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    k.run(spec, geo, context=ctx)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: fresh {t1 - t0:.4f} s, reused context {t2 - t1:.4f} s", flush=True)
