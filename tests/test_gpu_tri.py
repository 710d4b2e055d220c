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
