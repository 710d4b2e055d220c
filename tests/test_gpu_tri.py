"""Tridiagonal column stage of the dirichlet box solve (csrc/box_tri.cuh)
against the reference's DST route (boxsolve.py:70-82).

The column stage of BoxSolver.solve is DST_y -> divide by
(lam_kx + lam_q - kappa) -> DST_y, i.e. the inverse of the 1-D three-point
operator of every spectral column; the default device path applies that
inverse by factored recurrences.  Bar: 1e-10 relative L-inf (north_star);
measured deviations are ~1e-13 (the recurrences are closer to a long-double
solve than the FFT route, see box_tri.cuh).
"""

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import BOX, PI_BOX, rel_linf
from oracle import kfbi_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _solve(grid, kappa, rhs, mode):
    s = k.BoxSolver(grid, kappa, "dirichlet-zero")
    s.plan.set_colsolver(mode)
    try:
        return s.solve(rhs)
    finally:
        s.plan.set_colsolver("auto")


@pytest.mark.parametrize("m", [16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
@pytest.mark.parametrize("kappa", [0.0, 3.7, 2048.0, 262144.0, 512j, 2j])
def test_tri_vs_oracle_and_dst(m, kappa):
    rng = np.random.default_rng(m + int(abs(kappa)))
    cplx = isinstance(kappa, complex)
    rhs = rng.standard_normal((m + 1, m + 1))
    if cplx:
        rhs = rhs + 1j * rng.standard_normal((m + 1, m + 1))
    grid = k.CartesianGrid(BOX, m)
    ref = O.box_solve(m, grid.h, kappa, rhs)
    # the reference's rounded eigenvalues lam_q = (2cos - 2)/h^2 bound how far
    # its DST route can sit from the exact three-point inverse (E); the
    # recurrences apply the exact inverse
    choice, bound = k.BoxSolver(grid, kappa, "dirichlet-zero").plan.colsolver_for(kappa)
    assert choice == ("tridiagonal" if bound <= 1e-11 else "dst")
    u_auto = _solve(grid, kappa, rhs, "auto")
    assert rel_linf(u_auto, ref) < (1e-11 if choice == "tridiagonal" else TOL)
    u_tri = _solve(grid, kappa, rhs, "tridiagonal")
    assert u_tri.dtype == ref.dtype
    assert rel_linf(u_tri, ref) < max(4 * bound, 1e-12), (rel_linf(u_tri, ref), bound)
    if m <= 2048:
        u_dst = _solve(grid, kappa, rhs, "dst")
        assert rel_linf(u_dst, ref) < TOL
    # zero ring exactly
    for edge in (u_tri[0], u_tri[-1], u_tri[:, 0], u_tri[:, -1]):
        assert np.all(edge == 0)


@pytest.mark.parametrize("m", [8192, 16384])
def test_tri_large_residual(m):
    # large grids: the discrete operator residual (test_boxsolve.py:29-43 form)
    import torch

    grid = k.CartesianGrid(PI_BOX, m)
    for kappa in (2.0 * m, 2j * m):
        cplx = isinstance(kappa, complex)
        g = torch.Generator(device="cuda").manual_seed(m)
        dt = torch.complex128 if cplx else torch.float64
        rhs = torch.randn((m + 1, m + 1), dtype=dt, device="cuda", generator=g)
        s = k.BoxSolver(grid, kappa, "dirichlet-zero")
        assert s.plan.colsolver_for(kappa)[0] == "tridiagonal"
        u = s.solve(rhs)
        h2 = grid.h * grid.h
        lap = (u[1:-1, :-2] + u[1:-1, 2:] + u[:-2, 1:-1] + u[2:, 1:-1] - 4 * u[1:-1, 1:-1]) / h2
        r = lap - kappa * u[1:-1, 1:-1] - rhs[1:-1, 1:-1]
        rel = (r.abs().max() / rhs[1:-1, 1:-1].abs().max()).item()
        assert rel < 1e-11, (m, kappa, rel)
        del u, rhs, r, lap
        torch.cuda.empty_cache()


@pytest.mark.usefixtures("_three_pass_reference")
@pytest.mark.parametrize("p2p", [False, True])
def test_tri_slab_virtual_ranks_bit_identical(p2p):
    # the slab layout ([rank][panels][rows][w] blocks, or the peer stores of
    # the fused transposes) gives the same bits as the one-slab solve
    import torch

    from paper_2404_14864_b200 import dist as D

    m = 1024
    grid = k.CartesianGrid(BOX, m)
    rhs = torch.from_numpy(np.random.default_rng(7).standard_normal((m + 1, m + 1))).cuda()
    one = k.BoxSolver(grid, 40.0, "dirichlet-zero").solve(rhs)
    for p in (2, 4, 8):
        got = D.solve_virtual(grid, 40.0, rhs, p, p2p=p2p)
        assert torch.equal(got, one), p


@pytest.mark.parametrize("m,cplx", [(256, False), (1024, False), (1024, True), (4096, False),
                                    (4096, True)])
def test_slab_carry_matches_one_gpu(m, cplx):
    # transpose-free slab column stage (kfbi_slab_cols_tri): P virtual ranks
    # in one launch exchange three values per column; equal to the one-slab
    # solve up to the order the carries are combined in
    import torch

    from paper_2404_14864_b200 import dist as D

    grid = k.CartesianGrid(BOX, m)
    g = torch.Generator(device="cuda").manual_seed(m)
    dt = torch.complex128 if cplx else torch.float64
    rhs = torch.randn((m + 1, m + 1), generator=g, device="cuda", dtype=dt)
    kappa = 2j * m if cplx else 2.0 * m
    ref = k.BoxSolver(grid, kappa, "dirichlet-zero").solve(rhs)
    scale = float(ref.abs().max())
    for p in (1, 2, 4, 8):
        u = D.solve_virtual(grid, kappa, rhs, p, mode="carry")
        err = float((u - ref).abs().max()) / scale
        assert err < 1e-13, (p, err)
        for edge in (u[0], u[-1], u[:, 0], u[:, -1]):
            assert bool((edge == 0).all())


def test_slab_carry_16384():
    import torch

    from paper_2404_14864_b200 import dist as D

    m = 16384
    grid = k.CartesianGrid(PI_BOX, m)
    g = torch.Generator(device="cuda").manual_seed(1)
    rhs = torch.randn((m + 1, m + 1), generator=g, device="cuda", dtype=torch.float64)
    ref = k.BoxSolver(grid, 2048.0, "dirichlet-zero").solve(rhs)
    u = D.solve_virtual(grid, 2048.0, rhs, 8, mode="carry")
    assert float((u - ref).abs().max()) / float(ref.abs().max()) < 1e-13
    del u, ref, rhs
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kappa", [200.0, 16j])
def test_slab_carry_richardson(kappa):
    # the slab Richardson solve with the transpose-free column stage: same
    # iterations as the one-GPU device solve, field within rounding
    import torch

    from paper_2404_14864_b200 import dist as D
    from paper_2404_14864_b200.bvp import solve_device

    box = BOX if not isinstance(kappa, complex) else PI_BOX
    ws = k.InterfaceWorkspace(k.build_grid(box, 256, k.StarCurve(1.0, c=0.2, lobes=8)))
    sol = k.StaticPlaneWave(kappa=abs(kappa))
    cps = ws.cps
    interior = ws.geometry.classification.interior
    dt = torch.complex128 if isinstance(kappa, complex) else torch.float64
    X, Y = ws.grid.X, ws.grid.Y
    F = torch.from_numpy(np.where(interior, -(1.0 + kappa) * sol.u(X, Y), 0.0)).to("cuda", dt)
    fg = torch.from_numpy(np.asarray(-(1.0 + kappa) * sol.u(cps.x, cps.y))).to("cuda", dt)
    gb = torch.from_numpy(np.asarray(sol.dirichlet(cps.x, cps.y))).to("cuda", dt)
    ref = solve_device(ws, kappa=kappa, F=F.reshape(-1), f_gamma=fg, g=gb,
                       density=torch.zeros(cps.m, dtype=dt, device="cuda"))
    for p in (2, 4):
        dens = torch.zeros(cps.m, dtype=dt, device="cuda")
        u, tu, tn, it, res, hist = D.richardson_virtual(ws, p, kappa=kappa, F=F, f_gamma=fg, g=gb,
                                                        density=dens, mode="carry")
        assert it == ref.iterations
        err = float((u.reshape(-1) - ref.u.reshape(-1)).abs().max()) / float(ref.u.abs().max())
        assert err < 1e-11, (p, err)
    # the real SlabRichardson at P = 1 in carry mode (IPC buffers, in-kernel exchange)
    solver = D.SlabRichardson(ws, mode="carry")
    dens = torch.zeros(cps.m, dtype=dt, device="cuda")
    m1 = ws.grid.m
    u, tu, tn, it, res, hist = solver.solve(kappa=kappa, F=F[:m1].contiguous(), f_gamma=fg, g=gb,
                                            density=dens)
    assert it == ref.iterations and solver.passes.peers_ok()
    err = float((u.reshape(-1) - ref.u.reshape(-1)[:m1 * (m1 + 1)]).abs().max()) / float(ref.u.abs().max())
    assert err < 1e-11


@pytest.mark.parametrize("m", [64, 256, 1024, 4096, 8192])
@pytest.mark.parametrize("kappa", [2048.0, 262144.0, 512j])
def test_facr_box_solve(m, kappa):
    # one level of cyclic reduction (box_facr.cuh, default where it applies)
    # against the three-pass solve and the oracle
    import torch

    grid = k.CartesianGrid(BOX, m)
    cplx = isinstance(kappa, complex)
    g = torch.Generator(device="cuda").manual_seed(m + 3)
    dt = torch.complex128 if cplx else torch.float64
    rhs = torch.randn((m + 1, m + 1), generator=g, device="cuda", dtype=dt)
    s = k.BoxSolver(grid, kappa, "dirichlet-zero")
    u_f = s.solve(rhs)
    s.plan.set_facr(False)
    try:
        u_3 = s.solve(rhs)
    finally:
        s.plan.set_facr(True)
    scale = float(u_3.abs().max())
    assert float((u_f - u_3).abs().max()) / scale < 1e-12
    for edge in (u_f[0], u_f[-1], u_f[:, 0], u_f[:, -1]):
        assert bool((edge == 0).all())
    if m <= 1024:
        ref = O.box_solve(m, grid.h, kappa, rhs.cpu().numpy())
        assert rel_linf(u_f.cpu().numpy(), ref) < 1e-11


@pytest.mark.parametrize("kappa", [2048.0, 32768.0, 8j])
def test_facr_16384(kappa):
    # M = 16384: real data runs FACR on the one-real-row engine (box_real.cuh,
    # rows_odd_facr_real1); complex data stays on the three-pass solve
    import torch

    m = 16384
    grid = k.CartesianGrid(PI_BOX, m)
    cplx = isinstance(kappa, complex)
    s = k.BoxSolver(grid, kappa, "dirichlet-zero")
    assert s.plan.facr_for(kappa) == (not cplx)
    if cplx:
        return
    g = torch.Generator(device="cuda").manual_seed(5)
    rhs = torch.randn((m + 1, m + 1), generator=g, device="cuda", dtype=torch.float64)
    u_f = s.solve(rhs)
    s.plan.set_facr(False)
    try:
        u_3 = s.solve(rhs)
    finally:
        s.plan.set_facr(True)
    scale = float(u_3.abs().max())
    assert float((u_f - u_3).abs().max()) / scale < 1e-12
    for edge in (u_f[0], u_f[-1], u_f[:, 0], u_f[:, -1]):
        assert bool((edge == 0).all())
    del u_f, u_3, rhs
    torch.cuda.empty_cache()


def test_facr_richardson_same_iterations():
    # the Richardson solve through the FACR box solve (corrections on even and
    # odd rows): same sweeps and field as the three-pass solve
    geo = k.build_grid(BOX, 1024, k.StarCurve(1.0, c=0.2, lobes=8))
    ws = k.InterfaceWorkspace(geo)
    sol = k.StaticPlaneWave(kappa=2048.0)
    cps = ws.cps
    F = np.where(geo.classification.interior, sol.f(geo.grid.X, geo.grid.Y), 0.0)
    prob = k.BvpProblem(kappa=2048.0, F=F, f_gamma=sol.f(cps.x, cps.y), bc_kind="dirichlet",
                        bc_values=sol.dirichlet(cps.x, cps.y))
    a = k.richardson_solve(prob, ws)
    ws.plan.set_facr(False)
    try:
        b = k.richardson_solve(prob, ws)
    finally:
        ws.plan.set_facr(True)
    assert a.iterations == b.iterations
    assert rel_linf(a.u, b.u) < 1e-12


@pytest.fixture
def _three_pass_reference(monkeypatch):
    # bit-identity with the slab passes is defined against the three-pass
    # one-GPU box solve (the FACR form is compared to rounding in
    # test_gpu_tri.py::test_facr_*); plans created here start with FACR off
    from paper_2404_14864_b200 import boxsolve

    monkeypatch.setenv("KFBI_FACR", "0")
    boxsolve._GRID_PLANS.clear()
    yield
    boxsolve._GRID_PLANS.clear()
