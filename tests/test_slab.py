"""Slab-decomposed box solve (paper_2404_14864_b200/dist.py).

GPU: the P-slab solve (P = 1, 2, 4, 8 virtual ranks on one device, the real
kernels and panel layouts, the all-to-all done by chunk copies) is
bit-identical to BoxSolver.solve, for f64 and c128, up to M = 16384.

CPU (gloo, world_size 2, separate processes): the chunk exchange of the
all-to-all, and the whole rows -> all-to-all -> cols -> all-to-all -> rows
choreography of SlabBoxSolver against the reference box solve, with the three
device passes replaced by a numpy stand-in that follows the documented panel
layouts (include/kfbi_b200.h, kfbi_slab_*) - the host logic a multi-GPU run
exercises, checked where no second GPU exists.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp
from scipy.fft import dst

from conftest import BOX, rel_linf

import paper_2404_14864_b200 as k
from paper_2404_14864_b200 import dist as D
from oracle import kfbi_oracle as O


def test_slab_rows_partition():
    assert D.slab_rows(4096, 1, 0) == (0, 4096)
    assert [D.slab_rows(64, 4, g) for g in range(4)] == [(0, 16), (16, 32), (32, 48), (48, 64)]
    with pytest.raises(k.ConfigError):
        D.slab_rows(64, 3, 0)
    with pytest.raises(k.ConfigError):
        D.slab_rows(64, 2, 2)


# --------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("m,cplx", [(64, False), (256, False), (256, True), (1024, False),
                                    (1024, True), (4096, False)])
def test_virtual_slabs_bit_identical(m, cplx):
    import torch

    grid = k.CartesianGrid(BOX, m)
    g = torch.Generator(device="cuda").manual_seed(m)
    dt = torch.complex128 if cplx else torch.float64
    rhs = torch.randn((m + 1, m + 1), generator=g, device="cuda", dtype=dt)
    kappa = 2j * m if cplx else 3.7
    ref = k.BoxSolver(grid, kappa, "dirichlet-zero").solve(rhs)
    for p in (1, 2, 4, 8):
        u = D.solve_virtual(grid, kappa, rhs, p)
        assert torch.equal(u, ref), (p, float((u - ref).abs().max()))
        # the all-to-alls fused into the pass stores (peer-buffer addressing)
        u = D.solve_virtual(grid, kappa, rhs, p, p2p=True)
        assert torch.equal(u, ref), ("p2p", p, float((u - ref).abs().max()))


@pytest.mark.gpu
def test_slab_solver_single_rank_and_oracle():
    import torch

    m = 512
    grid = k.CartesianGrid(BOX, m)
    rng = np.random.default_rng(5)
    rhs = rng.standard_normal((m + 1, m + 1))
    s = D.SlabBoxSolver(grid, 40.0)
    assert s.nranks == 1 and s.rows == (0, m)
    u = s.solve(torch.from_numpy(rhs[:m]).cuda())
    full = D.gather_rows(u, m).cpu().numpy()
    assert rel_linf(full, O.box_solve(m, grid.h, 40.0, rhs)) < 1e-12
    assert np.all(full[0] == 0) and np.all(full[m] == 0) and np.all(full[:, 0] == 0)


@pytest.mark.gpu
@pytest.mark.parametrize("cplx", [False, True])
def test_p2p_slab_solver_single_rank(cplx):
    """SlabBoxSolver(p2p=True) at P = 1: IPC-allocated buffers, the fused
    passes and the peer-flag barrier, bit-identical to BoxSolver.solve."""
    import torch

    m = 1024
    grid = k.CartesianGrid(BOX, m)
    kappa = 2j * m if cplx else 7.0
    dt = torch.complex128 if cplx else torch.float64
    g = torch.Generator(device="cuda").manual_seed(3)
    s = D.SlabBoxSolver(grid, kappa, p2p=True)
    box = k.BoxSolver(grid, kappa, "dirichlet-zero")
    for it in range(3):
        rhs = torch.randn((m + 1, m + 1), generator=g, device="cuda", dtype=dt)
        rhs[m] = 0
        u = s.solve(rhs[:m])
        ref = box.solve(rhs)
        assert torch.equal(D.gather_rows(u, m), ref), it
    assert s.peers_ok()


@pytest.mark.gpu
def test_p2p_barrier_concurrent_ranks_and_timeout():
    """kfbi_p2p_barrier: two virtual ranks on two streams of one GPU meet;
    a rank whose peer never arrives gives up and reports it."""
    import ctypes as C

    import torch

    from paper_2404_14864_b200 import _native as N

    lib = N.lib()
    flags = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(2)]
    tab = (C.c_void_p * 2)(*[f.data_ptr() for f in flags])
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(2)]
    for epoch in (1, 2, 3):
        for r in (1, 0):
            N.check(lib.kfbi_p2p_barrier(tab, 2, r, epoch, 1 << 26, bad.data_ptr(),
                                         streams[r].cuda_stream))
        torch.cuda.synchronize()
        assert int(bad.item()) == 0
        assert flags[0][:2].tolist() == [epoch, epoch] and flags[1][:2].tolist() == [epoch, epoch]
    # rank 0 alone at epoch 4: times out, does not hang
    N.check(lib.kfbi_p2p_barrier(tab, 2, 0, 4, 1 << 16, bad.data_ptr(), streams[0].cuda_stream))
    torch.cuda.synchronize()
    assert int(bad.item()) == 1
    with pytest.raises(k.ConfigError):
        N.check(lib.kfbi_p2p_barrier(tab, 9, 0, 1, 0, None, None))


@pytest.mark.gpu
def test_virtual_slabs_16384():
    import torch

    m = 16384
    grid = k.CartesianGrid(BOX, m)
    g = torch.Generator(device="cuda").manual_seed(1)
    rhs = torch.randn((m + 1, m + 1), generator=g, device="cuda", dtype=torch.float64)
    ref = k.BoxSolver(grid, 1.0, "dirichlet-zero").solve(rhs)
    u = D.solve_virtual(grid, 1.0, rhs, 8)
    assert torch.equal(u, ref)
    del u
    u = D.solve_virtual(grid, 1.0, rhs, 8, p2p=True)
    assert torch.equal(u, ref)
    # size-independent check: the five-point operator of the solution
    # returns the right-hand side (interior rows of a band); the stencil's
    # own rounding (division by h^2 = 3.4e-8 of a cancelling sum) is ~1e-9
    h = grid.h
    band = slice(8000, 8010)
    uu = u[7999:8011]
    lap = (uu[2:, 1:-1] + uu[:-2, 1:-1] + uu[1:-1, 2:] + uu[1:-1, :-2] - 4 * uu[1:-1, 1:-1]) / h**2
    res = (lap - 1.0 * uu[1:-1, 1:-1]) - rhs[band, 1:-1]
    assert float(res.abs().max() / rhs[band].abs().max()) < 1e-8


# --------------------------------------------------------------------------
# CPU: gloo, two processes
class NumpySlabPlan:
    """Test double of the three kfbi_slab_* device passes, written from the
    documented layouts: panel buffer of rank g = [panel][local row][w] after
    the row pass; [rank block][local panel][rows of that rank][w] for the
    column pass (w = 4 real / 2 complex spectral columns per panel)."""

    def __init__(self, m, h):
        self.m, self.h = m, h
        lam = np.zeros(m + 1)
        p = np.arange(1, m)
        lam[1:m] = (2 * np.cos(p * np.pi / m) - 2) / h**2
        self.lam = lam

    def slab_panel_bytes(self, cplx, nranks):
        return (self.m // nranks) * self.m * (16 if cplx else 8)

    def _w(self, cplx):
        return 2 if cplx else 4

    def slab_rows_fwd(self, cplx, P, g, rhs, panels, sign=1.0, jv=None):
        m, R, w = self.m, self.m // P, self._w(cplx)
        x = rhs.numpy().copy()
        if g == 0:
            x[0] = 0
        spec = np.zeros((R, m), dtype=x.dtype)
        spec[:, 1:m] = dst(x[:, 1:m], type=1, axis=1)
        pv = panels.numpy().view(np.complex128 if cplx else np.float64)
        pv[:] = spec.reshape(R, m // w, w).transpose(1, 0, 2).reshape(-1)

    def slab_cols(self, cplx, P, g, kappa, panels):
        m, R, w = self.m, self.m // P, self._w(cplx)
        npl = m // w // P
        pv = panels.numpy().view(np.complex128 if cplx else np.float64)
        blk = pv.reshape(P, npl, R, w).transpose(1, 0, 2, 3).reshape(npl, m, w)
        cols = blk.transpose(0, 2, 1).reshape(npl * w, m)          # [kx][row]
        out = np.zeros_like(cols)
        kx = g * npl * w + np.arange(npl * w)
        den = self.lam[1:m][None, :] + self.lam[kx][:, None] - kappa
        out[:, 1:m] = dst(dst(cols[:, 1:m], type=1, axis=1) / den / (4.0 * m * m), type=1, axis=1)
        out[kx == 0] = 0
        back = out.reshape(npl, w, m).transpose(0, 2, 1).reshape(npl, P, R, w).transpose(1, 0, 2, 3)
        pv[:] = back.reshape(-1)

    def slab_rows_inv(self, cplx, P, g, panels, u):
        m, R, w = self.m, self.m // P, self._w(cplx)
        pv = panels.numpy().view(np.complex128 if cplx else np.float64)
        spec = pv.reshape(m // w, R, w).transpose(1, 0, 2).reshape(R, m)
        out = np.zeros((R, m + 1), dtype=spec.dtype)
        out[:, 1:m] = dst(spec[:, 1:m], type=1, axis=1)
        if g == 0:
            out[0] = 0
        u.numpy()[:] = out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1) chunk exchange: chunk h of rank g's result came from rank h
        src = torch.tensor([100.0 * rank + h for h in range(world) for _ in range(3)],
                           dtype=torch.float64)
        dst_ = torch.empty_like(src)
        D.exchange_chunks(dst_, src, world)
        out[("x", rank)] = dst_.tolist()
        # 2) the slab solve choreography with the numpy stand-in
        m = 32
        grid = k.CartesianGrid(BOX, m)
        rng = np.random.default_rng(7)
        rhs = rng.standard_normal((m + 1, m + 1))
        s = D.SlabBoxSolver.__new__(D.SlabBoxSolver)
        s.nranks, s.rank, s.group, s.grid, s.kappa = world, rank, None, grid, 2.5
        s.plan = NumpySlabPlan(m, grid.h)
        s.rows = D.slab_rows(m, world, rank)
        s.passes = D.SlabPasses(s.plan, world, rank, None, "cpu")

        class _B:
            torch_device = "cpu"
        s.backend = _B()
        r0, r1 = s.rows
        u = s.solve(torch.from_numpy(rhs[r0:r1].copy()))
        full = D.gather_rows(u, m).numpy()
        out[("u", rank)] = rel_linf(full, O.box_solve(m, grid.h, 2.5, rhs))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_slab_choreography():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    for g in range(world):
        assert out[("x", g)] == [100.0 * h + g for h in range(world) for _ in range(3)]
        assert out[("u", g)] < 1e-12


@pytest.mark.gpu
def test_packed_field_to_host_roundtrip():
    import torch

    geo = k.build_grid(BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8))
    ctx = k.StepContext(geo)
    u = torch.randn(ctx.n_grid, dtype=torch.float64, device="cuda")
    u[~torch.from_numpy(ctx.mask.ravel()).cuda()] = 0.0
    out = torch.empty(ctx.interior_index.numel(), dtype=torch.float64, pin_memory=True)
    ev = ctx.field_to_host(u, out, packed=True)
    ev.synchronize()
    full = ctx.unpack_interior(out.numpy())
    assert np.array_equal(full.ravel(), u.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("m,kappa", [(64, 16.0), (128, 200.0), (128, 16j)])
def test_slab_richardson_virtual_bit_identical(m, kappa):
    # the slab-decomposed Richardson solve (stencil-value all-reduce) equals
    # the one-GPU device solve bit for bit, for 1, 2 and 4 virtual ranks
    import torch

    from paper_2404_14864_b200.bvp import solve_device

    box = BOX if not isinstance(kappa, complex) else (-np.pi, np.pi, -np.pi, np.pi)
    curve = k.StarCurve(1.0, c=0.2, lobes=8) if m == 128 else k.CircleCurve(1.0)
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    sol = k.StaticPlaneWave(kappa=abs(kappa))
    cps = ws.cps
    interior = ws.geometry.classification.interior
    dt = torch.complex128 if isinstance(kappa, complex) else torch.float64
    X, Y = ws.grid.X, ws.grid.Y
    F = torch.from_numpy(np.where(interior, -(1.0 + kappa) * sol.u(X, Y), 0.0)).to("cuda", dt)
    fg = torch.from_numpy(np.asarray(-(1.0 + kappa) * sol.u(cps.x, cps.y))).to("cuda", dt)
    g = torch.from_numpy(np.asarray(sol.dirichlet(cps.x, cps.y))).to("cuda", dt)
    ref = solve_device(ws, kappa=kappa, F=F.reshape(-1), f_gamma=fg, g=g,
                       density=torch.zeros(cps.m, dtype=dt, device="cuda"))
    for p in (1, 2, 4):
        dens = torch.zeros(cps.m, dtype=dt, device="cuda")
        u, tu, tn, it, res, hist = D.richardson_virtual(ws, p, kappa=kappa, F=F, f_gamma=fg, g=g,
                                                        density=dens)
        assert it == ref.iterations
        assert torch.equal(u.reshape(-1), ref.u.reshape(-1)), p
        assert torch.equal(dens, ref.density)
        assert torch.equal(tu, ref.trace_u)
    # the real SlabRichardson at P = 1, transposes fused (p2p buffers + barrier)
    solver = D.SlabRichardson(ws, p2p=True)
    dens = torch.zeros(cps.m, dtype=dt, device="cuda")
    m1 = ws.grid.m
    u, tu, tn, it, res, hist = solver.solve(kappa=kappa, F=F[:m1].contiguous(), f_gamma=fg, g=g,
                                            density=dens)
    assert it == ref.iterations and solver.passes.peers_ok()
    assert torch.equal(u.reshape(-1), ref.u.reshape(-1)[:m1 * (m1 + 1)])
    assert torch.equal(dens, ref.density)


@pytest.fixture(autouse=True)
def _three_pass_reference(monkeypatch):
    # bit-identity with the slab passes is defined against the three-pass
    # one-GPU box solve (the FACR form is compared to rounding in
    # test_gpu_tri.py::test_facr_*); plans created here start with FACR off
    from paper_2404_14864_b200 import boxsolve

    monkeypatch.setenv("KFBI_FACR", "0")
    boxsolve._GRID_PLANS.clear()
    yield
    boxsolve._GRID_PLANS.clear()
