"""Generate the golden fixtures that pin the oracle and the host setup.

Runs the UNMODIFIED reference package (`/root/reference/pkg/src/kfbi`) in this
container and records its outputs as small ``.npz`` files next to this script.
The reference imports matplotlib at package import time (`report.py:23`),
which is not installed here, so a two-function stub is placed in
``sys.modules`` first; nothing on the solver path touches it.

The GPU box has no ``/root/reference``: tests only ever read the committed
``.npz`` files, never the reference itself.  Re-run with

    python tests/golden/make_golden.py [name ...]   (default: all files)

Inputs that are large (random right-hand sides) are regenerated in the tests
from the same ``np.random.default_rng(seed)`` streams instead of being stored.
"""

from __future__ import annotations

import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

BOX = (-1.5, 1.5, -1.5, 1.5)
PI_BOX = (-np.pi, np.pi, -np.pi, np.pi)


def load_reference():
    mpl = types.ModuleType("matplotlib")
    mpl.use = lambda *a, **k: None
    plt = types.ModuleType("matplotlib.pyplot")

    def _disabled(*a, **k):
        raise RuntimeError("figures disabled in fixture generation")

    plt.subplots = _disabled
    mpl.pyplot = plt
    sys.modules.setdefault("matplotlib", mpl)
    sys.modules.setdefault("matplotlib.pyplot", plt)
    sys.path.insert(0, REF_SRC)
    import kfbi  # noqa: E402

    return kfbi


# geometry cases shared by the setup / interface / extraction fixtures
def setup_cases(k):
    return {
        "disc32": (BOX, 32, k.CircleCurve(1.0)),
        "star64": (BOX, 64, k.StarCurve(1.0, c=0.2, lobes=3)),
        "flower128": (BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8)),
        "ellipse128": (BOX, 128, k.EllipseCurve(1.2, 0.8)),
        "pistar128": (PI_BOX, 128, k.StarCurve(1.5, c=0.2, lobes=3)),
    }


def box_rhs(m, seed, complex_rhs):
    rng = np.random.default_rng(seed)
    rhs = rng.standard_normal((m + 1, m + 1))
    if complex_rhs:
        rhs = rhs + 1j * rng.standard_normal((m + 1, m + 1))
    return rhs


BOX_CASES = [
    # (tag, m, kappa, bc, seed, complex_rhs)
    ("d16_k3p7", 16, 3.7, "dirichlet-zero", 101, False),
    ("d32_k3p7", 32, 3.7, "dirichlet-zero", 102, False),
    ("d128_k2048", 128, 2048.0, "dirichlet-zero", 103, False),
    ("d128_k0", 128, 0.0, "dirichlet-zero", 104, False),
    ("d64_kc", 64, 256j, "dirichlet-zero", 105, True),
    ("d32_kc_realrhs", 32, 2j, "dirichlet-zero", 106, False),
    ("n16_k3p7", 16, 3.7, "neumann-zero", 107, False),
    ("n64_k200", 64, 200.0, "neumann-zero", 108, False),
    ("n32_kc", 32, 256j, "neumann-zero", 109, True),
]


def sketch(seed, n, k=4):
    return np.random.default_rng(seed).standard_normal((n, k))


def gen_setup(k):
    out = {}
    for name, (box, m, curve) in setup_cases(k).items():
        geo = k.build_grid(box, m, curve)
        ws = k.InterfaceWorkspace(geo)
        ex = k.TraceExtractor(ws)
        rec = geo.records
        cps = ws.cps
        p = f"{name}__"
        out[p + "level"] = geo.classification.level
        out[p + "interior"] = geo.classification.interior
        out[p + "irregular"] = geo.classification.irregular
        for key in ("owner_flat", "arm", "theta", "d", "owner_interior", "x", "y",
                    "group_starts", "group_owners"):
            out[p + "rec_" + key] = getattr(rec, key)
        out[p + "cps_m"] = np.array(cps.m)
        for key in ("theta", "pos", "tangent", "normal", "dtan_ds", "speed"):
            out[p + "cps_" + key] = getattr(cps, key)
        out[p + "inv3"] = ws._inv3
        w = ws.w_records
        if w.size <= 64 * 64 * 8:
            out[p + "W"] = w
        out[p + "W_sketch"] = w @ sketch(7, cps.m)
        out[p + "W_rows"] = w[:: max(1, rec.n // 8)]
        out[p + "ex_stencil"] = ex.stencil_flat
        out[p + "ex_ainv"] = ex._ainv
        out[p + "ex_jcoef"] = ex._jcoef
        try:
            ox = k.OneSidedExtractor(ws)
            out[p + "os_stencil"] = ox.stencil_flat
            out[p + "os_rows"] = ox._rows
            out[p + "os_fallback"] = ox._fallback
        except Exception as exc:  # pragma: no cover - recorded, not fatal
            print("one-sided extractor failed for", name, exc)
    return out


def gen_box(k):
    from kfbi.grid import CartesianGrid

    out = {}
    for tag, m, kappa, bc, seed, cplx in BOX_CASES:
        grid = CartesianGrid(BOX, m)
        rhs = box_rhs(m, seed, cplx)
        u = k.BoxSolver(grid, kappa, bc).solve(rhs)
        out[tag + "__u"] = u
    return out


def gen_interface(k):
    out = {}
    pf = k.PiecewiseField(kappa=2.0)
    for name, (box, m, curve) in setup_cases(k).items():
        if box is PI_BOX:
            continue
        geo = k.build_grid(box, m, curve)
        ws = k.InterfaceWorkspace(geo)
        cps = ws.cps
        X, Y = geo.grid.X, geo.grid.Y
        interior = geo.classification.interior
        data = k.InterfaceData(
            kappa=2.0,
            F=np.where(interior, pf.f_jump(X, Y), 0.0),
            phi=pf.phi(cps.x, cps.y),
            psi=pf.psi(cps.x, cps.y, cps.normal),
            f_gamma=pf.f_jump(cps.x, cps.y),
        )
        js = k.compute_jumps(data, ws)
        c = k.corrections(js, ws)
        u = k.solve_interface(data, ws, box_bc="dirichlet-zero")
        tu, tx, ty = k.TraceExtractor(ws).extract(u, js)
        p = f"{name}__"
        out[p + "jumps"] = js.as_matrix()
        out[p + "corr"] = c
        out[p + "u"] = u
        out[p + "trace"] = np.stack([tu, tx, ty])
        # complex jumps with a complex kappa (Schrödinger-type data)
        rng = np.random.default_rng(55)
        phi_c = rng.standard_normal(cps.m) + 1j * rng.standard_normal(cps.m)
        fg_c = rng.standard_normal(cps.m) + 1j * rng.standard_normal(cps.m)
        data_c = k.InterfaceData(kappa=64j, F=np.zeros((m + 1, m + 1), complex),
                                 phi=phi_c, psi=np.zeros(cps.m, complex), f_gamma=fg_c)
        js_c = k.compute_jumps(data_c, ws)
        out[p + "jumps_c"] = js_c.as_matrix()
        out[p + "corr_c"] = k.corrections(js_c, ws)
    return out


def gen_richardson(k):
    out = {}
    cases = {
        "disc64_k16": (BOX, 64, k.CircleCurve(1.0), 16.0),
        "flower128_k200": (BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8), 200.0),
        "pistar64_kc": (PI_BOX, 64, k.StarCurve(1.5, c=0.2, lobes=3), 16j),
    }
    for name, (box, m, curve, kappa) in cases.items():
        geo = k.build_grid(box, m, curve)
        ws = k.InterfaceWorkspace(geo)
        cps = ws.cps
        X, Y = geo.grid.X, geo.grid.Y
        interior = geo.classification.interior
        kr = abs(kappa)
        sol = k.StaticPlaneWave(kappa=kr)
        if isinstance(kappa, complex):
            # u = sin(0.6x+0.8y) solves Δu − κu = −(1+κ)u for any κ
            F = np.where(interior, -(1.0 + kappa) * sol.u(X, Y), 0.0)
            fg = -(1.0 + kappa) * sol.u(cps.x, cps.y)
        else:
            F = np.where(interior, sol.f(X, Y), 0.0)
            fg = sol.f(cps.x, cps.y)
        g = sol.dirichlet(cps.x, cps.y)
        prob = k.BvpProblem(kappa=kappa, F=F, f_gamma=fg, bc_kind="dirichlet", bc_values=g)
        s = k.richardson_solve(prob, ws)
        p = f"{name}__"
        out[p + "u"] = s.u
        out[p + "density"] = s.density
        out[p + "trace_u"] = s.trace_u
        out[p + "trace_un"] = s.trace_un
        out[p + "iterations"] = np.array(s.iterations)
        out[p + "residual"] = np.array(s.residual)
        out[p + "history"] = np.array(s.residual_history)
    return out


def run_cases(k):
    heat = k.HeatPlaneDecay(c=1.0)
    wave = k.WaveStanding(phase=0.0)
    schr = k.SchrodingerPhaseRotation()
    return {
        # C1 of BASELINE.json: heat CN, flower star(1,0.2,8), 128², τ=0.01, 100 steps
        "c1_heat_flower128": (BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8), dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=0.01, t_final=1.0, c=1.0)),
        "heat_flower64": (BOX, 64, k.StarCurve(1.0, c=0.2, lobes=5), dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=0.25, t_final=1.0, c=1.0)),
        "wave_ellipse128": (BOX, 128, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=0.125,
            t_final=1.0, theta=0.25)),
        "wave_ellipse64_th05": (BOX, 64, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=0.25,
            t_final=1.0, theta=0.5)),
        "schr_star128": (PI_BOX, 128, k.StarCurve(1.5, c=0.2, lobes=3), dict(
            equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
            lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=0.125,
            t_final=1.0)),
        "godunov_star64": (PI_BOX, 64, k.StarCurve(1.5, c=0.2, lobes=3), dict(
            equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
            lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=0.25,
            t_final=1.0, splitting="godunov")),
    }


def gen_runs(k):
    out = {}
    for name, (box, m, curve, kw) in run_cases(k).items():
        geo = k.build_grid(box, m, curve)
        spec = k.ProblemSpec(**kw)
        res = k.run(spec, geo)
        p = f"{name}__"
        out[p + "u"] = res.state.u
        out[p + "density"] = res.state.density
        out[p + "iterations"] = np.array(res.iterations)
        out[p + "t"] = np.array(res.state.t)
        out[p + "n"] = np.array(res.state.n)
        print(name, "iterations", res.iterations[:6], "... total", sum(res.iterations))
    return out


def gen_nonlinear(k):
    from kfbi.timestepping import nonlinear_phase_step

    rng = np.random.default_rng(77)
    n = 4096
    u = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) * 1.5
    v = rng.uniform(0.0, 2.0, n)
    return {"u": u, "v": v, "out": nonlinear_phase_step(u, v, 1.0, 0.0625),
            "out_w3": nonlinear_phase_step(u, v, 3.0, 0.25)}


def gen_neumann(k):
    """Neumann path: neumann-zero interface solves + one-sided extraction,
    Neumann Richardson solves, Neumann heat / wave runs."""
    out = {}
    pf = k.PiecewiseField(kappa=2.0)
    for name in ("flower128", "ellipse128"):
        box, m, curve = setup_cases(k)[name]
        geo = k.build_grid(box, m, curve)
        ws = k.InterfaceWorkspace(geo)
        cps = ws.cps
        X, Y = geo.grid.X, geo.grid.Y
        interior = geo.classification.interior
        data = k.InterfaceData(kappa=2.0, F=np.where(interior, pf.f_jump(X, Y), 0.0),
                               phi=np.zeros(cps.m), psi=pf.psi(cps.x, cps.y, cps.normal),
                               f_gamma=pf.f_jump(cps.x, cps.y))
        js = k.compute_jumps(data, ws)
        u = k.solve_interface(data, ws, box_bc="neumann-zero")
        tu, tx, ty = k.OneSidedExtractor(ws).extract(u, js)
        p = f"{name}__"
        out[p + "u"] = u
        out[p + "trace"] = np.stack([tu, tx, ty])
    cases = {
        "disc64_k16": (BOX, 64, k.CircleCurve(1.0), 16.0),
        "flower128_k200": (BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8), 200.0),
    }
    for name, (box, m, curve, kappa) in cases.items():
        geo = k.build_grid(box, m, curve)
        ws = k.InterfaceWorkspace(geo)
        cps = ws.cps
        X, Y = geo.grid.X, geo.grid.Y
        interior = geo.classification.interior
        sol = k.StaticPlaneWave(kappa=kappa)
        F = np.where(interior, sol.f(X, Y), 0.0)
        prob = k.BvpProblem(kappa=kappa, F=F, f_gamma=sol.f(cps.x, cps.y), bc_kind="neumann",
                            bc_values=sol.neumann(cps.x, cps.y, cps.normal))
        s = k.richardson_solve(prob, ws)
        p = f"rich_{name}__"
        out[p + "u"] = s.u
        out[p + "density"] = s.density
        out[p + "trace_u"] = s.trace_u
        out[p + "trace_un"] = s.trace_un
        out[p + "iterations"] = np.array(s.iterations)
        out[p + "history"] = np.array(s.residual_history)
    heat = k.HeatPlaneDecay(c=1.0)
    wave = k.WaveStanding(phase=0.0)
    runs = {
        "heat_flower64": (BOX, 64, k.StarCurve(1.0, c=0.2, lobes=5), dict(
            equation="heat", bc_kind="neumann", g=heat.neumann, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=0.25, t_final=1.0, c=1.0)),
        "wave_ellipse64": (BOX, 64, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="neumann", g=wave.neumann, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=0.25,
            t_final=1.0, theta=0.25)),
    }
    for name, (box, m, curve, kw) in runs.items():
        geo = k.build_grid(box, m, curve)
        res = k.run(k.ProblemSpec(**kw), geo)
        p = f"run_{name}__"
        out[p + "u"] = res.state.u
        out[p + "density"] = res.state.density
        out[p + "iterations"] = np.array(res.iterations)
        print(name, "iterations", res.iterations)
    return out


def main():
    k = load_reference()
    import scipy

    stamp = np.array(f"kfbi {k.__version__}; numpy {np.__version__}; scipy {scipy.__version__}")
    gens = (("setup", gen_setup), ("box", gen_box), ("interface", gen_interface),
            ("richardson", gen_richardson), ("runs", gen_runs),
            ("nonlinear", gen_nonlinear), ("neumann", gen_neumann))
    only = set(sys.argv[1:])
    for fname, gen in gens:
        if only and fname not in only:
            continue
        data = gen(k)
        data["stamp"] = stamp
        path = os.path.join(HERE, f"{fname}.npz")
        np.savez_compressed(path, **data)
        print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
