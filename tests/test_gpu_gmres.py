"""Opt-in GMRES on the boundary integral equation (kfbi_gmres, bvp.gmres_solve)
against the reference's Richardson iteration (bvp.py:276-351).

GMRES converges to the same fixed point by a different iterate, so the
accuracy gate is tolerance-level, not bitwise: the field agrees with the
Richardson field to GATE relative L-inf (tol = 1e-8 on the density update),
the error against the manufactured solution is unchanged to within the same
margin, and it takes fewer pipeline evaluations.  PAPER.md:768.
"""

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import BOX, PI_BOX, rel_linf

pytestmark = pytest.mark.gpu
GATE = 1e-6


def _problem(m, kappa, curve, box=BOX, bc="dirichlet"):
    geo = k.build_grid(box, m, curve)
    ws = k.InterfaceWorkspace(geo)
    sol = k.StaticPlaneWave(kappa=kappa)
    cps = ws.cps
    F = np.where(geo.classification.interior, sol.f(geo.grid.X, geo.grid.Y), 0.0)
    if bc == "dirichlet":
        g = sol.dirichlet(cps.x, cps.y)
    else:
        g = sol.neumann(cps.x, cps.y, cps.normal)
    prob = k.BvpProblem(kappa=kappa, F=F, f_gamma=sol.f(cps.x, cps.y), bc_kind=bc, bc_values=g)
    return geo, ws, sol, prob


@pytest.mark.parametrize("m,kappa", [(64, 16.0), (256, 16.0), (1024, 2048.0)])
def test_gmres_matches_richardson_dirichlet(m, kappa):
    geo, ws, sol, prob = _problem(m, kappa, k.StarCurve(1.0, c=0.2, lobes=5))
    r = k.richardson_solve(prob, ws)
    g = k.gmres_solve(prob, ws)
    assert rel_linf(g.u, r.u) < GATE
    mask = geo.classification.interior
    exact = sol.u(geo.grid.X, geo.grid.Y)
    e_r = np.max(np.abs(r.u - exact)[mask])
    e_g = np.max(np.abs(g.u - exact)[mask])
    assert abs(e_g - e_r) <= GATE * np.max(np.abs(exact[mask])) + 0.05 * e_r
    assert g.iterations < r.iterations, (g.iterations, r.iterations)
    assert g.residual <= prob.tol


def test_gmres_complex_kappa():
    # Schrodinger-type complex kappa (timestepping.py:378) on the pi box
    geo = k.build_grid(PI_BOX, 256, k.StarCurve(1.5, c=0.2, lobes=3))
    ws = k.InterfaceWorkspace(geo)
    kappa = 2j * 64
    rng = np.random.default_rng(3)
    F = np.where(geo.classification.interior, np.exp(1j * (geo.grid.X + 0.5 * geo.grid.Y)), 0.0)
    n = ws.cps.m
    prob = k.BvpProblem(kappa=kappa, F=F, f_gamma=rng.standard_normal(n) + 0j,
                        bc_kind="dirichlet", bc_values=np.cos(ws.cps.x) + 1j * np.sin(ws.cps.y))
    r = k.richardson_solve(prob, ws)
    g = k.gmres_solve(prob, ws)
    assert g.u.dtype == np.complex128
    assert rel_linf(g.u, r.u) < GATE
    assert g.iterations < r.iterations


def test_gmres_neumann():
    geo, ws, sol, prob = _problem(128, 200.0, k.StarCurve(1.0, c=0.2, lobes=5), bc="neumann")
    r = k.richardson_solve(prob, ws)
    g = k.gmres_solve(prob, ws)
    assert rel_linf(g.u, r.u) < GATE


def test_gmres_restart_and_max_iter():
    geo, ws, sol, prob = _problem(128, 16.0, k.StarCurve(1.0, c=0.2, lobes=5))
    r = k.richardson_solve(prob, ws)
    g = k.gmres_solve(prob, ws, restart=4)        # several restart cycles
    assert rel_linf(g.u, r.u) < GATE
    short = k.BvpProblem(kappa=prob.kappa, F=prob.F, f_gamma=prob.f_gamma, bc_kind="dirichlet",
                         bc_values=prob.bc_values, max_iter=2)
    with pytest.raises(k.ConvergenceError) as ei:
        out = k.gmres_solve(short, ws)
        print("no raise:", out.iterations, out.residual, out.residual_history)
    assert ei.value.iterations == 2


@pytest.mark.parametrize("operator", [False, True], ids=["pipeline", "operator"])
def test_gmres_time_stepping(operator):
    # a short heat run with GMRES steps (matvecs via the pipeline, or the
    # explicit trace operator) against the Richardson run
    heat = k.HeatPlaneDecay()
    geo = k.build_grid(BOX, 256, k.StarCurve(1.0, c=0.2, lobes=8))
    spec = k.ProblemSpec(equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                         lap_u0=heat.lap_u0, tau=1 / 64, t_final=4 / 64)
    ref = k.run(spec, geo, operator=False)
    ctx = k.StepContext(geo, operator=operator, solver="gmres")
    res = k.run(spec, geo, context=ctx, operator=operator)
    assert rel_linf(res.state.u, ref.state.u) < GATE
    assert sum(res.iterations) < sum(ref.iterations)
