"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The golden files come from the unmodified reference package
(tests/golden/make_golden.py).  The oracle consumes setup tables produced by
the product's host setup, so these tests pin both at once.
"""

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import (BOX, BOX_CASES, NEUMANN_RICH_CASES, box_rhs, curve_of, golden,
                      neumann_run_cases, oracle_spec, rel_linf, run_cases, setup_cases)
from oracle import kfbi_oracle as O


def _tables(name):
    box, m, curve = setup_cases()[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    return ws, O.tables_from_workspace(ws)


@pytest.mark.parametrize("case", BOX_CASES, ids=lambda c: c[0])
def test_box_solve_matches_reference(case):
    tag, m, kappa, bc, seed, cplx = case
    grid = k.CartesianGrid(BOX, m)
    u = O.box_solve(m, grid.h, kappa, box_rhs(m, seed, cplx), bc=bc)
    assert np.array_equal(u, golden("box")[tag + "__u"])


@pytest.mark.parametrize("name", ["disc32", "star64", "flower128", "ellipse128"])
def test_interface_pieces_match_reference(name):
    ws, t = _tables(name)
    g = golden("interface")
    pf = k.PiecewiseField(kappa=2.0)
    cps = ws.cps
    X, Y = ws.grid.X, ws.grid.Y
    interior = ws.geometry.classification.interior
    jm = O.jumps(t, 2.0, pf.phi(cps.x, cps.y), pf.psi(cps.x, cps.y, cps.normal),
                 pf.f_jump(cps.x, cps.y))
    assert np.array_equal(jm, g[name + "__jumps"])
    c = O.corrections(t, jm)
    assert np.array_equal(c, g[name + "__corr"])
    F = np.where(interior, pf.f_jump(X, Y), 0.0)
    u = O.box_solve(t.m, t.h, 2.0, F + c)
    assert np.array_equal(u, g[name + "__u"])
    tr = np.stack(O.extract(t, u, jm))
    assert np.array_equal(tr, g[name + "__trace"])
    rng = np.random.default_rng(55)
    phi_c = rng.standard_normal(cps.m) + 1j * rng.standard_normal(cps.m)
    fg_c = rng.standard_normal(cps.m) + 1j * rng.standard_normal(cps.m)
    jm_c = O.jumps(t, 64j, phi_c, np.zeros(cps.m, complex), fg_c)
    assert np.array_equal(jm_c, g[name + "__jumps_c"])
    assert np.array_equal(O.corrections(t, jm_c), g[name + "__corr_c"])


def test_richardson_matches_reference():
    from conftest import PI_BOX

    g = golden("richardson")
    cases = {
        "disc64_k16": (BOX, 64, k.CircleCurve(1.0), 16.0),
        "flower128_k200": (BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8), 200.0),
        "pistar64_kc": (PI_BOX, 64, k.StarCurve(1.5, c=0.2, lobes=3), 16j),
    }
    for name, (box, m, curve, kappa) in cases.items():
        ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
        t = O.tables_from_workspace(ws)
        sol = k.StaticPlaneWave(kappa=abs(kappa))
        interior = ws.geometry.classification.interior
        X, Y, cps = ws.grid.X, ws.grid.Y, ws.cps
        F = np.where(interior, -(1.0 + kappa) * sol.u(X, Y), 0.0)
        fg = -(1.0 + kappa) * sol.u(cps.x, cps.y)
        s = O.richardson(t, kappa, F, fg, sol.dirichlet(cps.x, cps.y))
        p = name + "__"
        assert s.iterations == int(g[p + "iterations"])
        assert np.array_equal(np.array(s.history), g[p + "history"])
        assert np.array_equal(s.u, g[p + "u"])
        assert np.array_equal(s.density, g[p + "density"])


@pytest.mark.parametrize("name", list(run_cases()))
def test_full_runs_match_reference(name):
    box, m, curve, kw = run_cases()[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    st = O.run(O.tables_from_workspace(ws), oracle_spec(kw))
    g = golden("runs")
    assert st.iterations == list(g[name + "__iterations"])
    assert rel_linf(st.u, g[name + "__u"]) == 0.0


def test_nonlinear_phase_matches_reference():
    g = golden("nonlinear")
    assert np.array_equal(O.nonlinear_phase(g["u"], g["v"], 1.0, 0.0625), g["out"])
    assert np.array_equal(O.nonlinear_phase(g["u"], g["v"], 3.0, 0.25), g["out_w3"])


def test_oracle_residual_oracle():
    # the reference's own oracle: relative residual of the 5-point operator
    grid = k.CartesianGrid(BOX, 32)
    rhs = box_rhs(32, 5, False)
    u = O.box_solve(32, grid.h, 3.7, rhs)
    r = k.apply_box_operator(grid, u, 3.7, "dirichlet-zero") - rhs
    assert np.max(np.abs(r[1:-1, 1:-1])) / np.max(np.abs(rhs)) < 1e-11


# ---------------------------------------------------------------------------
# Neumann path (neumann-zero box, one-sided extraction, psi iteration)

@pytest.mark.parametrize("name", ["flower128", "ellipse128"])
def test_neumann_interface_and_onesided_match_reference(name):
    box, m, curve = setup_cases()[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    t = O.tables_from_workspace(ws, onesided=True)
    g = golden("neumann")
    pf = k.PiecewiseField(kappa=2.0)
    cps = ws.cps
    interior = ws.geometry.classification.interior
    jm = O.jumps(t, 2.0, np.zeros(cps.m), pf.psi(cps.x, cps.y, cps.normal),
                 pf.f_jump(cps.x, cps.y))
    c = O.corrections(t, jm)
    F = np.where(interior, pf.f_jump(ws.grid.X, ws.grid.Y), 0.0)
    u = O.box_solve(t.m, t.h, 2.0, F + c, bc="neumann-zero")
    assert np.array_equal(u, g[name + "__u"])
    assert np.array_equal(np.stack(O.extract_onesided(t, u, jm)), g[name + "__trace"])


@pytest.mark.parametrize("name", list(NEUMANN_RICH_CASES))
def test_neumann_richardson_matches_reference(name):
    box, m, ctag, kappa = NEUMANN_RICH_CASES[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve_of(ctag)))
    t = O.tables_from_workspace(ws, onesided=True)
    sol = k.StaticPlaneWave(kappa=kappa)
    cps = ws.cps
    interior = ws.geometry.classification.interior
    F = np.where(interior, sol.f(ws.grid.X, ws.grid.Y), 0.0)
    s = O.richardson(t, kappa, F, sol.f(cps.x, cps.y), sol.neumann(cps.x, cps.y, cps.normal),
                     bc_kind="neumann")
    g = golden("neumann")
    p = "rich_" + name + "__"
    assert s.iterations == int(g[p + "iterations"])
    assert np.array_equal(np.array(s.history), g[p + "history"])
    assert np.array_equal(s.u, g[p + "u"])
    assert np.array_equal(s.density, g[p + "density"])
    assert np.array_equal(s.trace_un, g[p + "trace_un"])


@pytest.mark.parametrize("name", list(neumann_run_cases()))
def test_neumann_runs_match_reference(name):
    box, m, curve, kw = neumann_run_cases()[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    st = O.run(O.tables_from_workspace(ws, onesided=True), oracle_spec(kw))
    g = golden("neumann")
    assert st.iterations == list(g["run_" + name + "__iterations"])
    assert rel_linf(st.u, g["run_" + name + "__u"]) == 0.0
