"""A few asynchronous 4096^2 Schrödinger bench steps (for ncu captures of the
step kernels).   python tools/schr_steps.py [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200.timestepping import _stepper_for  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
box, curve, kw = bench.workload(4096)["schrodinger"]
ctx = k.StepContext(k.build_grid(box, 4096, curve), backend=k.CudaBackend(0, timing=False), operator=True)
spec = k.ProblemSpec(**kw)
startup, step = _stepper_for(spec)
st = startup(spec, ctx)
for _ in range(steps):
    st = step(st, spec, ctx)
torch.cuda.synchronize()
print("iterations", ctx.flush())
