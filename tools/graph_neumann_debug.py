import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2404_14864_b200 as k
from conftest import BOX

wave = k.WaveStanding(phase=0.0)
for tau in (0.25, 1 / 32):
    kw = dict(equation="wave", bc_kind="neumann", g=wave.neumann, u0=wave.u0,
              lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=tau, t_final=10 * tau)
    geo = k.build_grid(BOX, 64, k.EllipseCurve(1.2, 0.8))
    spec = k.ProblemSpec(**kw)
    be = k.CudaBackend(0, timing=False)
    for graph in (False, True):
        try:
            r = k.run(spec, geo, context=k.StepContext(geo, operator=True, backend=be), operator=True, graph=graph)
            print(tau, graph, r.iterations, float(np.abs(r.state.u).max()), flush=True)
        except Exception as e:
            print(tau, graph, "ERROR", type(e).__name__, e, flush=True)
    try:
        r = k.run(spec, geo, context=k.StepContext(geo, operator=False, backend=be), operator=False)
        print(tau, "pipeline", r.iterations, flush=True)
    except Exception as e:
        print(tau, "pipeline ERROR", e, flush=True)
