"""Wave (theta = 1/4, ellipse) error vs time on the device, C4 sizes: the
default path and the pipeline form with the DST column stage."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200.timestepping import _stepper_for  # noqa: E402

box, curve, sol, kw = bench.c4_cases()["wave"]
for m in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096]:
    geo = k.build_grid(box, m, curve)
    mask = geo.classification.interior
    for mode in ("default", "pipeline-dst"):
        spec = k.ProblemSpec(tau=0.25 * 64 / m, t_final=1.0, **kw)
        ctx = k.StepContext(geo, operator=(mode == "default"))
        if mode != "default":
            ctx.plan.set_colsolver("dst")
        startup, step = _stepper_for(spec)
        st = startup(spec, ctx)
        out = []
        while st.n < spec.n_steps():
            st = step(st, spec, ctx)
            if st.n % max(spec.n_steps() // 8, 1) == 0:
                u = st.u.detach().cpu().numpy().reshape(m + 1, m + 1)
                e = np.max(np.abs(u - sol.u(geo.grid.X, geo.grid.Y, st.t))[mask])
                it = ctx.flush() if ctx.asynchronous else [st.last_iterations]
                out.append((st.n, round(float(st.t), 4), float(e), it[-1] if it else None))
        print(m, mode, out, flush=True)
