"""Host setup (grid, records, control points, tables) against the reference's
golden setup vectors, plus API-level validation behaviour.  CPU only."""

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import BOX, PI_BOX, golden, setup_cases
from paper_2404_14864_b200.interface import MIN_CONTROL_SPACING, default_control_count


@pytest.mark.parametrize("name", list(setup_cases()))
def test_grid_and_records_bitwise(name):
    box, m, curve = setup_cases()[name]
    geo = k.build_grid(box, m, curve)
    g = golden("setup")
    p = name + "__"
    assert np.array_equal(geo.classification.level, g[p + "level"])
    assert np.array_equal(geo.classification.interior, g[p + "interior"])
    assert np.array_equal(geo.classification.irregular, g[p + "irregular"])
    for key in ("owner_flat", "arm", "theta", "d", "owner_interior", "x", "y",
                "group_starts", "group_owners"):
        assert np.array_equal(getattr(geo.records, key), g[p + "rec_" + key]), key
    # both records of an edge share its crossing parameter
    assert np.array_equal(geo.edge_theta[geo.records.edge], geo.records.theta)


@pytest.mark.parametrize("name", list(setup_cases()))
def test_workspace_tables_bitwise(name):
    box, m, curve = setup_cases()[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    g = golden("setup")
    p = name + "__"
    cps = ws.cps
    assert cps.m == int(g[p + "cps_m"])
    for key in ("theta", "pos", "tangent", "normal", "dtan_ds", "speed"):
        assert np.array_equal(getattr(cps, key), g[p + "cps_" + key]), key
    assert np.array_equal(ws._inv3, g[p + "inv3"])
    w = ws.w_records
    if p + "W" in g:
        assert np.array_equal(w, g[p + "W"])
    assert np.array_equal(w[:: max(1, ws.records.n // 8)], g[p + "W_rows"])
    sk = np.random.default_rng(7).standard_normal((cps.m, 4))
    assert np.allclose(w @ sk, g[p + "W_sketch"], rtol=0, atol=1e-13)
    stencil, ainv, jcoef = ws.trace_tables()
    assert np.array_equal(stencil, g[p + "ex_stencil"])
    assert np.array_equal(ainv, g[p + "ex_ainv"])
    assert np.array_equal(jcoef, g[p + "ex_jcoef"])


@pytest.mark.parametrize("name", ["disc32", "star64", "flower128"])
def test_one_sided_tables_bitwise(name):
    box, m, curve = setup_cases()[name]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    ox = k.OneSidedExtractor(ws)
    g = golden("setup")
    p = name + "__"
    assert np.array_equal(ox.stencil_flat, g[p + "os_stencil"])
    assert np.array_equal(ox._rows, g[p + "os_rows"])
    assert np.array_equal(ox._fallback, g[p + "os_fallback"])


def test_device_tables_layout():
    box, m, curve = setup_cases()["flower128"]
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    t = ws.device_tables()
    rec = ws.records
    n_groups = rec.group_starts.size
    assert t["group_start"][-1] == rec.n and t["group_start"].size == n_groups + 1
    # row CSR covers every group exactly once, in row order
    rows = rec.group_owners // (m + 1)
    for j in range(m + 1):
        lo, hi = t["row_group"][j], t["row_group"][j + 1]
        assert np.all(rows[lo:hi] == j)
    assert t["row_group"][-1] == n_groups
    assert t["ainv_rows"].shape == (ws.cps.m, 3, 6)
    # the circulant column reproduces the spectral derivative
    v = np.sin(3 * ws.cps.theta) + 0.2 * np.cos(11 * ws.cps.theta)
    circ = np.array([np.dot(t["deriv_col"][(i - np.arange(v.size)) % v.size], v)
                     for i in range(v.size)])
    from paper_2404_14864_b200.geometry import periodic_derivative

    assert np.max(np.abs(circ - periodic_derivative(v, ws.cps.dtheta))) < 1e-12


def test_control_count_rules():
    # interface.py:111-126 and test_interface.py:155-187 of the reference
    assert default_control_count(k.build_grid(BOX, 64, k.CircleCurve(1.0))) == 64
    assert default_control_count(k.build_grid(BOX, 128, k.CircleCurve(1.0))) == 128
    assert default_control_count(k.build_grid(PI_BOX, 64, k.StarCurve(1.5, 0.2, 3))) == 32
    assert default_control_count(k.build_grid(PI_BOX, 128, k.StarCurve(1.5, 0.2, 3))) == 64
    geo = k.build_grid(BOX, 128, k.StarCurve(1.0, c=0.2, lobes=3))
    n = default_control_count(geo)
    theta = 2.0 * np.pi * np.arange(4096) / 4096
    vel = geo.curve.velocity(theta)
    smin = np.min(np.hypot(vel[:, 0], vel[:, 1]))
    assert n % 2 == 0 and smin * 2 * np.pi / n >= MIN_CONTROL_SPACING * geo.grid.h - 1e-12
    assert k.InterfaceWorkspace(k.build_grid(BOX, 64, k.CircleCurve(1.0)), n_controls=40).cps.m == 40


def test_grid_validation_and_layout():
    grid = k.CartesianGrid(BOX, 16)
    assert grid.h == pytest.approx(3.0 / 16)
    assert grid.flat_index(4, 11) == 4 + 11 * 17
    assert k.neighbors(grid, 4, 11) == ((5, 11), (3, 11), (4, 12), (4, 10))
    with pytest.raises(IndexError):
        k.neighbors(grid, 0, 5)
    for box, m in (((-1.0, 1.0, -1.0, 2.0), 16), ((-1.0, -2.0, -1.0, -2.0), 16), (BOX, 24), (BOX, 8)):
        with pytest.raises(k.GridError):
            k.CartesianGrid(box, m)
    with pytest.raises(k.GridError):
        k.build_grid(BOX, 32, k.CircleCurve(1.45))   # too close to the box


def test_geometry_api():
    with pytest.raises(k.ConfigError):
        k.make_curve("hexagon")
    with pytest.raises(k.ConfigError):
        k.make_curve("circle", radius=1.0, bogus=3)
    with pytest.raises(k.GeometryError):
        k.StarCurve(1.0, c=0.6)
    c = k.make_curve("ellipse", a=1.3, b=0.6)
    xi, th = k.edge_intersection(c, (0.0, 0.0), (2.0, 0.0))
    assert abs(xi[0] - 1.3) < 1e-12 and abs(th) < 1e-12
    cps = k.control_points(k.CircleCurve(2.0), 64)
    d1, d2 = k.differentiate_density(np.sin(3 * cps.theta), cps)
    assert np.max(np.abs(d1 - 1.5 * np.cos(3 * cps.theta))) < 1e-12
    assert np.max(np.abs(d2 + 2.25 * np.sin(3 * cps.theta))) < 1e-12
    sp = k.SplineCurve(np.stack([np.cos(np.linspace(0, 2 * np.pi, 24, endpoint=False)),
                                 np.sin(np.linspace(0, 2 * np.pi, 24, endpoint=False))], 1))
    assert sp.implicit(np.array([0.0]), np.array([0.0]))[0] < 0
    assert k.classify_point(k.CircleCurve(1.0), 0.2, 0.1)


def test_problem_validation():
    geo = k.build_grid(BOX, 32, k.CircleCurve(1.0))
    m = k.InterfaceWorkspace(geo).cps.m
    ok = dict(kappa=1.0, F=np.zeros_like(geo.grid.X), f_gamma=np.zeros(m), bc_kind="dirichlet",
              bc_values=np.zeros(m))
    k.BvpProblem(**ok)
    for bad in ({"bc_kind": "robin"}, {"gamma": 0.0}, {"gamma": 1.0}, {"tol": 0.0},
                {"max_iter": 0}, {"box_bc": "periodic"}):
        with pytest.raises(k.ConfigError):
            k.BvpProblem(**{**ok, **bad})
    with pytest.raises(k.ConfigError):
        k.BoxSolver(geo.grid, 0.0, "neumann-zero")
    with pytest.raises(k.ConfigError):
        k.BoxProblem(geo.grid, 1.0, "periodic", np.zeros((33, 33)))
    heat = k.HeatPlaneDecay()
    with pytest.raises(k.ConfigError):
        k.ProblemSpec(equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                      tau=0.3, t_final=1.0).n_steps()
    with pytest.raises(k.ConfigError):
        k.ProblemSpec(equation="wave", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
                      theta=0.2)


def test_backend_selectors():
    for bad in ("gpu", "serial", "workers:2", "cuda:x"):
        with pytest.raises(k.ConfigError):
            k.make_backend(bad)
    assert k.KernelSpec("rhs-update", 10, 4).chunk_bounds() == [(0, 4), (4, 8), (8, 10)]
    with pytest.raises(k.ConfigError):
        k.KernelSpec("not-a-kernel", 1)


def test_errors_carry_fields():
    e = k.ConvergenceError("x", iterations=3, last_residual=0.5)
    assert e.iterations == 3 and e.last_residual == 0.5
    e = k.InstabilityError(4, 0.5, 1e11, 1e10)
    assert e.step == 4 and e.threshold == 1e10
    e = k.DispatchError("transform-rows", "boom")
    assert e.kernel_name == "transform-rows" and "boom" in str(e)
    assert issubclass(k.ExtractionError, k.KfbiError)
