"""The 4096^2 bench step (one time step each of heat / wave / Schrödinger)
with the three equations on one stream vs on three streams (they are
independent problems): device ms per bench step.

    python tools/streams_probe.py [K]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402
from paper_2404_14864_b200.timestepping import _stepper_for  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl = bench.workload(4096)
eqs = bench.EQUATIONS
backend = k.CudaBackend(0, timing=False)
ctxs, specs, states, steppers, startups = {}, {}, {}, {}, {}
for eq in eqs:
    box, curve, kw = wl[eq]
    ctxs[eq] = k.StepContext(k.build_grid(box, 4096, curve), backend=backend, operator=True)
    specs[eq] = k.ProblemSpec(**kw)
    startups[eq], steppers[eq] = _stepper_for(specs[eq])
streams = {eq: torch.cuda.Stream() for eq in eqs}
main = torch.cuda.current_stream()


def adv(eq):
    s = steppers[eq](states[eq], specs[eq], ctxs[eq])
    ctxs[eq].check_stable(s, specs[eq])
    states[eq] = s


def fresh(conc):
    torch.cuda.synchronize()
    for c in ctxs.values():
        c.flush()
    for eq in eqs:
        with torch.cuda.stream(streams[eq] if conc else main):
            states[eq] = startups[eq](specs[eq], ctxs[eq])
            for _ in range(3):
                adv(eq)
    torch.cuda.synchronize()
    for c in ctxs.values():
        c.flush()


def loop(conc, do_fresh=True):
    if do_fresh:
        fresh(conc)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    t0 = time.perf_counter()
    if conc:
        for s in streams.values():
            s.wait_stream(main)
    for _ in range(K):
        for eq in eqs:
            if conc:
                with torch.cuda.stream(streams[eq]):
                    adv(eq)
            else:
                adv(eq)
    if conc:
        for s in streams.values():
            main.wait_stream(s)
    b.record(main)
    host = (time.perf_counter() - t0) / K * 1e3
    torch.cuda.synchronize()
    its = {eq: ctxs[eq].flush() for eq in eqs}
    return a.elapsed_time(b) / K, its, host


if __name__ == "__main__":
    ctxs["heat"].workspace.ensure_operator(2.0 * specs["heat"].c / specs["heat"].tau, False)
    for eq in eqs:
        kap = {"heat": 2.0 * specs[eq].c / specs[eq].tau,
               "wave": 1.0 / (specs[eq].theta * specs[eq].tau ** 2),
               "schrodinger": 2j / specs[eq].tau}[eq]
        ctxs[eq].workspace.ensure_operator(kap, eq == "schrodinger")
    ref = None
    for rep in range(3):
        for conc in (False, True):
            ms, its, host = loop(conc)
            if ref is None:
                ref = its
            print(f"{'3 streams' if conc else '1 stream '}: {ms:.3f} ms per bench step "
                  f"({3000.0 / ms:.1f} time steps/s), host issue {host:.3f} ms per bench step, "
                  f"iterations equal: {its == ref}", flush=True)
