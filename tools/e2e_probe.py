"""Where does the e2e loop lose time against the device-resident loop?
Alternates K steps of: plain, gather-only, gather + D2H (packed), on the bench
workload.  python tools/e2e_probe.py [K]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200.timestepping import _stepper_for  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
wl = bench.workload(4096)
eqs = bench.EQUATIONS
backend = k.CudaBackend(0, timing=False)
ctxs, specs, states, steppers = {}, {}, {}, {}
for eq in eqs:
    box, curve, kw = wl[eq]
    ctxs[eq] = k.StepContext(k.build_grid(box, 4096, curve), backend=backend, operator=True)
    specs[eq] = k.ProblemSpec(**kw)
    st, step = _stepper_for(specs[eq])
    steppers[eq] = step
    states[eq] = st(specs[eq], ctxs[eq])


def adv(eq):
    s = steppers[eq](states[eq], specs[eq], ctxs[eq])
    ctxs[eq].check_stable(s, specs[eq])
    states[eq] = s
    return s


pinned = {eq: torch.empty(ctxs[eq].interior_index.numel(),
                          dtype=torch.complex128 if eq == "schrodinger" else torch.float64,
                          pin_memory=True) for eq in eqs}
startups = {eq: _stepper_for(specs[eq])[0] for eq in eqs}


def fresh():
    # every loop from t = 0 (+ 3 warm steps), as bench.py: the same steps timed
    for c in ctxs.values():
        c.flush()
    for eq in eqs:
        states[eq] = startups[eq](specs[eq], ctxs[eq])
    for _ in range(3):
        for eq in eqs:
            adv(eq)
    torch.cuda.synchronize()
    for c in ctxs.values():
        c.flush()


fresh()


full = {eq: torch.empty((4097 * 4097,), dtype=torch.complex128 if eq == "schrodinger" else torch.float64,
                        pin_memory=True) for eq in eqs}
side = torch.cuda.Stream()


def loop(mode):
    fresh()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record()
    for _ in range(K):
        for eq in eqs:
            s = adv(eq)
            if mode == "gather":
                c = ctxs[eq]
                buf = torch.empty(c.interior_index.numel(), dtype=s.u.dtype, device="cuda")
                c.plan.gather(c.interior_index, s.u, buf)
            elif mode == "copy":
                ctxs[eq].field_to_host(s.u, pinned[eq], packed=True)
            elif mode == "fullcopy":
                ctxs[eq].field_to_host(s.u, full[eq], packed=False)
    for c in ctxs.values():
        c.host_sync()
    b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    for c in ctxs.values():
        c.flush()
    return a.elapsed_time(b) / K, wall * 1e3 / K


for rep in range(2):
    for mode in ("plain", "gather", "copy", "fullcopy", "plain"):
        dev, wall = loop(mode)
        print(f"{mode:7s} device {dev:7.3f} ms / bench step   host wall {wall:7.3f} ms", flush=True)
