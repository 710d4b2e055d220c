"""Neumann path on the device against the reference (tests/golden/neumann.npz,
box.npz) and the oracle: the neumann-zero box solve (DCT-I), the one-sided
trace extraction, the psi Richardson iteration and Neumann heat / wave runs.

Bar (north_star): 1e-10 relative L-inf, identical Richardson iteration counts.
"""

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import (BOX, BOX_CASES, NEUMANN_RICH_CASES, box_rhs, curve_of, golden,
                      neumann_run_cases, rel_linf, setup_cases)
from oracle import kfbi_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [c for c in BOX_CASES if c[3] == "neumann-zero"],
                         ids=lambda c: c[0])
def test_neumann_box_vs_reference(case):
    tag, m, kappa, bc, seed, cplx = case
    grid = k.CartesianGrid(BOX, m)
    u = k.BoxSolver(grid, kappa, bc).solve(box_rhs(m, seed, cplx))
    ref = golden("box")[tag + "__u"]
    assert u.dtype == ref.dtype
    assert rel_linf(u, ref) < 1e-12


@pytest.mark.parametrize("m", [16, 32, 256, 1024, 4096])
def test_neumann_eigenfunctions_and_oracle(m):
    # the reference's test_discrete_eigenfunctions_solved_exactly (cos modes)
    # and test_neumann_constant_mode, then larger sizes against the oracle
    grid = k.CartesianGrid(BOX, m)
    xi = (grid.X - grid.box[0]) / 3.0
    eta = (grid.Y - grid.box[2]) / 3.0
    kappa = 5.0
    for p, q in ((1, 1), (3, 2), (7, 12), (0, 5)):
        lam = ((2 * np.cos(p * np.pi / m) - 2) + (2 * np.cos(q * np.pi / m) - 2)) / grid.h**2
        ue = np.cos(p * np.pi * xi) * np.cos(q * np.pi * eta)
        u = k.BoxSolver(grid, kappa, "neumann-zero").solve((lam - kappa) * ue)
        assert np.max(np.abs(u - ue)) < 1e-11
    rhs = np.full((m + 1, m + 1), -2.5 * 0.75)
    u = k.BoxSolver(grid, 2.5, "neumann-zero").solve(rhs)
    assert np.max(np.abs(u - 0.75)) < 1e-12
    if m <= 1024:
        r = box_rhs(m, 11 + m, m == 256)
        kap = 3j * m if m == 256 else 40.0
        u = k.BoxSolver(grid, kap, "neumann-zero").solve(r)
        assert rel_linf(u, O.box_solve(m, grid.h, kap, r, bc="neumann-zero")) < 1e-12


def test_neumann_kappa_zero_rejected():
    with pytest.raises(k.ConfigError):
        k.BoxSolver(k.CartesianGrid(BOX, 16), 0.0, "neumann-zero")


@pytest.mark.parametrize("name", ["flower128", "ellipse128"])
def test_neumann_interface_and_onesided_extraction(name):
    box, m, curve = setup_cases()[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    g = golden("neumann")
    pf = k.PiecewiseField(kappa=2.0)
    cps = ws.cps
    X, Y = ws.grid.X, ws.grid.Y
    interior = ws.geometry.classification.interior
    data = k.InterfaceData(kappa=2.0, F=np.where(interior, pf.f_jump(X, Y), 0.0),
                           phi=np.zeros(cps.m), psi=pf.psi(cps.x, cps.y, cps.normal),
                           f_gamma=pf.f_jump(cps.x, cps.y))
    js = k.compute_jumps(data, ws)
    u = k.solve_interface(data, ws, box_bc="neumann-zero")
    assert rel_linf(u, g[name + "__u"]) < 1e-12
    tr = np.stack(k.OneSidedExtractor(ws).extract(u, js))
    assert rel_linf(tr, g[name + "__trace"]) < 1e-10


@pytest.mark.parametrize("name", list(NEUMANN_RICH_CASES))
def test_neumann_richardson_vs_reference(name):
    box, m, ctag, kappa = NEUMANN_RICH_CASES[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve_of(ctag)))
    sol = k.StaticPlaneWave(kappa=kappa)
    cps = ws.cps
    interior = ws.geometry.classification.interior
    F = np.where(interior, sol.f(ws.grid.X, ws.grid.Y), 0.0)
    prob = k.BvpProblem(kappa=kappa, F=F, f_gamma=sol.f(cps.x, cps.y), bc_kind="neumann",
                        bc_values=sol.neumann(cps.x, cps.y, cps.normal))
    s = k.richardson_solve(prob, ws)
    g = golden("neumann")
    p = "rich_" + name + "__"
    assert s.iterations == int(g[p + "iterations"])
    assert rel_linf(s.u, g[p + "u"]) < 1e-10
    assert rel_linf(s.density, g[p + "density"]) < 1e-10
    assert rel_linf(s.trace_un, g[p + "trace_un"]) < 1e-10


@pytest.mark.parametrize("operator", [False, True])
@pytest.mark.parametrize("name", list(neumann_run_cases()))
def test_neumann_runs_vs_reference(name, operator):
    box, m, curve, kw = neumann_run_cases()[name]
    geo = k.build_grid(box, m, curve)
    res = k.run(k.ProblemSpec(**kw), geo, operator=operator)
    g = golden("neumann")
    assert res.iterations == list(g["run_" + name + "__iterations"])
    assert rel_linf(res.state.u, g["run_" + name + "__u"]) < 1e-10
