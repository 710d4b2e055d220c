"""Field-by-field comparison of one uncaptured step and the first replay of
the captured step from the same state (wave / C1 heat).

    python tools/graph_debug.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2404_14864_b200 as k  # noqa: E402
from conftest import run_cases  # noqa: E402
from paper_2404_14864_b200.timestepping import StepGraph, _stepper_for  # noqa: E402

for name in ("wave_ellipse128", "c1_heat_flower128"):
    box, m, curve, kw = run_cases()[name]
    geo = k.build_grid(box, m, curve)
    ctx = k.StepContext(geo, backend=k.CudaBackend(0, timing=False), operator=True)
    spec = k.ProblemSpec(**kw)
    startup, step = _stepper_for(spec)
    st = startup(spec, ctx)
    kap = {"heat": 2.0 * spec.c / spec.tau, "wave": 1.0 / (spec.theta * spec.tau ** 2)}[spec.equation]
    ctx.workspace.ensure_operator(kap, False, spec.bc_kind)
    st = step(st, spec, ctx)
    st = step(st, spec, ctx)
    s2 = st
    s3n = step(s2, spec, ctx)
    torch.cuda.synchronize()
    it_n = ctx.flush()
    sg = StepGraph(ctx, spec, step, s2)
    s3g = sg.advance()
    torch.cuda.synchronize()
    it_g = ctx.flush()
    print(name, "iterations normal", it_n, "graph", it_g)
    for f in StepGraph.FIELDS:
        a, b = getattr(s3n, f, None), getattr(s3g, f, None)
        if a is None or b is None or not hasattr(a, "reshape"):
            continue
        a, b = a.reshape(-1), b.reshape(-1)
        d = float((a - b).abs().max())
        print(f"  {f:14s} max|diff| {d:.3e}  (max|a| {float(a.abs().max()):.3e})  equal {torch.equal(a, b)}")
    # a second replay from the same input (the other graph)
    sg.reset(s2)
    sg.k = 1
    s3g2 = sg.advance()
    torch.cuda.synchronize()
    print("  graph 1 iterations", ctx.flush(), "u equal", torch.equal(s3g2.u.reshape(-1), s3n.u.reshape(-1)))
