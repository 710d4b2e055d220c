"""Slab-decomposed box solve across the GPUs of one node (the
C5 configuration: one 16384^2 modified-Helmholtz solve split over 2-8 B200).

The dirichlet-zero box solve (BoxSolver.solve, boxsolve.py:46-94) is a DST-I
along x of every row, a DST-I / divide / DST-I along y of every column and
a DST-I along x again.  Rank g of P owns grid rows [g M/P, (g+1) M/P) of the
right-hand side and of the solution, and panels (spectral column strips)
[g n_p/P, (g+1) n_p/P) for the column pass.  One solve is

    rows_fwd (local rows, all columns)  -> all-to-all ->
    cols     (local columns, all rows)  -> all-to-all ->
    rows_inv (local rows, all columns)

The panel buffer layouts are chosen so that both all-to-alls exchange P equal
contiguous chunks (kfbi_slab_* in include/kfbi_b200.h): no pack or unpack
kernels, the collective is ``torch.distributed.all_to_all_single`` over NCCL
(NVLink / NVSwitch).  With P = 1 the exchanges are identities and the solve
is bit-identical to BoxSolver.solve.

With ``p2p=True`` the two all-to-alls are fused into the transforms: the
forward row pass stores each panel chunk straight into the owning rank's
column-pass buffer and the column pass stores each row chunk into the owning
rank's row-pass buffer (device memory of the peers, mapped once with CUDA
IPC), with a peer-flag barrier kernel between the passes instead of a
collective.  The exchange then overlaps the transforms tile by tile.

``solve_virtual`` runs P slabs one after the other on one GPU with the
exchange done by device copies: the same kernels and layouts, used to
validate the decomposition where only one GPU is available.
"""

from __future__ import annotations

from .boxsolve import _grid_plan, _validate
from .errors import ConfigError, GridError


def _dist():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def slab_rows(m, nranks, rank):
    """Grid rows [r0, r1) of rank `rank` (row 0 is the zero ring; row m is not
    stored by any slab)."""
    if nranks < 1 or nranks & (nranks - 1) or not 0 <= rank < nranks:
        raise ConfigError("nranks must be a power of two and 0 <= rank < nranks")
    r = m // nranks
    return rank * r, (rank + 1) * r


def exchange_chunks(dst, src, nranks, group=None):
    """All-to-all of P equal contiguous chunks: chunk g of src goes to rank g,
    chunk h of dst comes from rank h (the transpose of the slab box solve)."""
    if nranks == 1:
        return src
    dist = _dist()
    if dist is None:
        raise ConfigError("slab box solve with nranks > 1 needs an initialised torch.distributed")
    dist.all_to_all_single(dst, src, group=group)
    return dst


class PeerBuffers:
    """One device buffer per rank, addressable by every rank: allocated with
    kfbi_ipc_alloc, handles exchanged once (all_gather_object) and opened with
    kfbi_ipc_open.  ``ptrs[h]`` is rank h's buffer in this process."""

    def __init__(self, nbytes, nranks, rank, group=None):
        import ctypes as C

        from . import _native as N

        self._lib = N.lib()
        self.nranks, self.rank = nranks, rank
        own = C.c_void_p()
        handle = (C.c_char * 64)()
        N.check(self._lib.kfbi_ipc_alloc(int(nbytes), C.byref(own), handle))
        self.own = int(own.value)
        self._opened = []
        if nranks == 1:
            self.ptrs = [self.own]
            return
        dist = _dist()
        if dist is None:
            raise ConfigError("p2p slab solve with nranks > 1 needs an initialised torch.distributed")
        handles = [None] * nranks
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.ptrs = []
        for h, hb in enumerate(handles):
            if h == rank:
                self.ptrs.append(self.own)
                continue
            q = C.c_void_p()
            N.check(self._lib.kfbi_ipc_open(C.create_string_buffer(hb, 64), C.byref(q)))
            self._opened.append(int(q.value))
            self.ptrs.append(int(q.value))

    def close(self):
        for q in self._opened:
            self._lib.kfbi_ipc_close(q)
        self._opened = []
        if self.own:
            self._lib.kfbi_ipc_free(self.own)
            self.own = 0

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


class SlabPasses:
    """The three box-solve passes of one rank with the two transposes
    between them: NCCL all-to-alls (default) or, with p2p=True, fused into
    the pass stores over CUDA-IPC peer buffers with a peer-flag barrier
    kernel between the passes.  Buffers are allocated on first use per dtype
    (the p2p ones collectively: every rank must make its first call)."""

    def __init__(self, plan, nranks, rank, group=None, device=None, p2p=False, mode=None):
        self.plan, self.nranks, self.rank, self.group = plan, nranks, rank, group
        self.device = device
        # "a2a": NCCL all-to-all transposes; "p2p": transposes fused into the
        # pass stores; "carry": no transposes at all, the tridiagonal column
        # stage exchanges three values per column over peer memory
        self.mode = mode or ("p2p" if p2p else "a2a")
        if self.mode not in ("a2a", "p2p", "carry"):
            raise ConfigError(f"unknown slab mode {self.mode!r}")
        self.p2p = self.mode == "p2p"
        self._bufs = {}
        self._epoch = 0
        self._timed_out = None

    def _buffers(self, cplx):
        import torch

        key = bool(cplx)
        if key not in self._bufs:
            nbytes = self.plan.slab_panel_bytes(cplx, self.nranks)
            P, g = self.nranks, self.rank
            if self.mode == "carry":
                agg_b, flag_b = self.plan.slab_tri_bytes(cplx, P)
                own = torch.empty(nbytes // 8, dtype=torch.float64, device=self.device)
                self._bufs[key] = (own, PeerBuffers(agg_b, P, g, self.group),
                                   PeerBuffers(flag_b, P, g, self.group))
                if self._timed_out is None:
                    self._timed_out = torch.zeros(1, dtype=torch.int32, device=self.device)
            elif self.p2p:
                self._bufs[key] = (PeerBuffers(nbytes, P, g, self.group),
                                   PeerBuffers(nbytes, P, g, self.group),
                                   PeerBuffers(8 * 8, P, g, self.group))
                if self._timed_out is None:
                    self._timed_out = torch.zeros(1, dtype=torch.int32, device=self.device)
            else:
                mk = lambda: torch.empty(nbytes // 8, dtype=torch.float64, device=self.device)
                self._bufs[key] = (mk(), mk() if P > 1 else None)
        return self._bufs[key]

    def _barrier(self, flags):
        self._epoch += 1
        self.plan.p2p_barrier(flags.ptrs, self.nranks, self.rank, self._epoch, self._timed_out)

    def peers_ok(self):
        """False if a p2p barrier ever gave up waiting for a peer (syncs)."""
        return self._timed_out is None or int(self._timed_out.item()) == 0

    def run(self, cplx, kappa, rhs, u, sign=1.0, jv=None):
        """u (this rank's rows) = box solve of sign * rhs (+ corrections of jv)."""
        p, P, g = self.plan, self.nranks, self.rank
        if self.mode == "carry":
            own, agg, flags = self._buffers(cplx)
            p.slab_rows_fwd(cplx, P, g, rhs, own, sign=sign, jv=jv)
            self._epoch += 1
            p.slab_cols_tri(cplx, P, g, kappa, own, agg.ptrs, flags.ptrs, self._epoch,
                            self._timed_out)
            p.slab_rows_inv(cplx, P, g, own, u)
            return u
        if self.p2p:
            A, B, F = self._buffers(cplx)
            p.slab_rows_fwd_p2p(cplx, P, g, rhs, A.ptrs, sign=sign, jv=jv)
            self._barrier(F)
            p.slab_cols_p2p(cplx, P, g, kappa, A.own, B.ptrs)
            self._barrier(F)
            p.slab_rows_inv(cplx, P, g, B.own, u)
            return u
        a, b = self._buffers(cplx)
        p.slab_rows_fwd(cplx, P, g, rhs, a, sign=sign, jv=jv)
        t = exchange_chunks(b, a, P, self.group)
        p.slab_cols(cplx, P, g, kappa, t)
        t = exchange_chunks(a, t, P, self.group)
        p.slab_rows_inv(cplx, P, g, t, u)
        return u


class SlabBoxSolver:
    """Slab-decomposed BoxSolver (dirichlet-zero) for the calling rank.

    rhs / u are this rank's rows ``slab_rows(m, nranks, rank)`` as CUDA
    tensors of shape (rows, m + 1), float64 or complex128.  p2p=True fuses
    the transposes into the passes (SlabPasses)."""

    def __init__(self, grid, kappa, bc="dirichlet-zero", nranks=None, rank=None, group=None,
                 backend=None, p2p=False, mode=None):
        _validate(bc, kappa)
        if bc != "dirichlet-zero":
            raise ConfigError("the slab-decomposed box solve supports the dirichlet-zero closure")
        dist = _dist()
        self.nranks = int(nranks if nranks is not None else (dist.get_world_size(group) if dist else 1))
        self.rank = int(rank if rank is not None else (dist.get_rank(group) if dist else 0))
        self.group = group
        self.grid = grid
        self.kappa = complex(kappa) if isinstance(kappa, complex) else float(kappa)
        from .engine import default_backend, make_backend

        self.backend = make_backend(backend) if backend is not None else default_backend()
        self.plan = _grid_plan(grid, self.backend)
        self.rows = slab_rows(grid.m, self.nranks, self.rank)
        self.passes = SlabPasses(self.plan, self.nranks, self.rank, group,
                                 self.backend.torch_device, p2p, mode)

    def peers_ok(self):
        return self.passes.peers_ok()

    def solve(self, rhs):
        import torch

        m = self.grid.m
        r0, r1 = self.rows
        if tuple(rhs.shape) != (r1 - r0, m + 1):
            raise GridError(f"rhs slab shape {tuple(rhs.shape)} != ({r1 - r0}, {m + 1})")
        cplx = rhs.is_complex() or isinstance(self.kappa, complex)
        dt = torch.complex128 if cplx else torch.float64
        rhs = rhs.to(dt).contiguous()
        u = torch.empty_like(rhs)
        return self.passes.run(cplx, self.kappa, rhs, u)


def solve_virtual(grid, kappa, rhs, nranks, backend=None, p2p=False, mode=None):
    """The P-slab solve of a full (m+1)^2 rhs on ONE device: every rank's
    passes run in turn and the all-to-alls are chunk copies (p2p=True: the
    fused passes store into the other virtual ranks' buffers directly).
    Returns the full solution (row m = zero ring)."""
    import torch

    m = grid.m
    solvers = [SlabBoxSolver(grid, kappa, nranks=nranks, rank=g, backend=backend)
               for g in range(nranks)]
    cplx = rhs.is_complex() or isinstance(solvers[0].kappa, complex)
    dt = torch.complex128 if cplx else torch.float64
    rhs = rhs.to(dt)
    plan = solvers[0].plan
    nbytes = plan.slab_panel_bytes(cplx, nranks)
    dev = rhs.device
    send = [torch.empty(nbytes // 8, dtype=torch.float64, device=dev) for _ in range(nranks)]
    recv = [torch.empty_like(x) for x in send]

    def a2a(dst, src):
        c = src[0].numel() // nranks
        for g in range(nranks):
            for h in range(nranks):
                dst[g][h * c:(h + 1) * c].copy_(src[h][g * c:(g + 1) * c])

    if mode == "carry":
        # transpose-free: every rank's own buffer, one column launch for all
        agg_b, flag_b = plan.slab_tri_bytes(cplx, nranks)
        agg = [torch.zeros(max(agg_b // 8, 1), dtype=torch.float64, device=dev) for _ in range(nranks)]
        flg = [torch.zeros(max(flag_b // 8, 1), dtype=torch.int64, device=dev) for _ in range(nranks)]
        for g, s in enumerate(solvers):
            r0, r1 = s.rows
            plan.slab_rows_fwd(cplx, nranks, g, rhs[r0:r1].contiguous(), send[g])
        plan.slab_cols_tri(cplx, nranks, 0, solvers[0].kappa, None, agg, flg, 1,
                           virt_panels=send)
        u = torch.zeros((m + 1, m + 1), dtype=dt, device=dev)
        for g, s in enumerate(solvers):
            r0, r1 = s.rows
            out = torch.empty((r1 - r0, m + 1), dtype=dt, device=dev)
            plan.slab_rows_inv(cplx, nranks, g, send[g], out)
            u[r0:r1] = out
        return u

    if p2p:
        send.clear()
        send.extend(torch.full_like(x, float("nan")) for x in recv)
        recv[:] = [torch.full_like(x, float("nan")) for x in recv]
        for g, s in enumerate(solvers):
            r0, r1 = s.rows
            plan.slab_rows_fwd_p2p(cplx, nranks, g, rhs[r0:r1].contiguous(), recv)
        for g, s in enumerate(solvers):
            plan.slab_cols_p2p(cplx, nranks, g, s.kappa, recv[g], send)
        u = torch.zeros((m + 1, m + 1), dtype=dt, device=dev)
        for g, s in enumerate(solvers):
            r0, r1 = s.rows
            out = torch.empty((r1 - r0, m + 1), dtype=dt, device=dev)
            plan.slab_rows_inv(cplx, nranks, g, send[g], out)
            u[r0:r1] = out
        return u

    for g, s in enumerate(solvers):
        r0, r1 = s.rows
        plan.slab_rows_fwd(cplx, nranks, g, rhs[r0:r1].contiguous(), send[g])
    a2a(recv, send)
    for g, s in enumerate(solvers):
        plan.slab_cols(cplx, nranks, g, s.kappa, recv[g])
    a2a(send, recv)
    u = torch.zeros((m + 1, m + 1), dtype=dt, device=dev)
    for g, s in enumerate(solvers):
        r0, r1 = s.rows
        out = torch.empty((r1 - r0, m + 1), dtype=dt, device=dev)
        plan.slab_rows_inv(cplx, nranks, g, send[g], out)
        u[r0:r1] = out
    return u


def gather_rows(u_slab, m, group=None):
    """Assemble the full (m+1)^2 field on every rank (all_gather of the slabs)."""
    import torch

    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        parts = [u_slab]
    else:
        parts = [torch.empty_like(u_slab) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, u_slab.contiguous(), group=group)
    full = torch.zeros((m + 1, m + 1), dtype=u_slab.dtype, device=u_slab.device)
    full[:m] = torch.cat(parts, 0)
    return full



# ---------------------------------------------------------------------------
# slab-decomposed Richardson solve (bvp.py:276-351), dirichlet-zero box

def _operands(dt, n, F, f_gamma, g, density, m_rows=None):
    """Cast F / f_gamma / g to the solve's dtype (the kernels read raw
    pointers of that element size) and check the in-place density."""
    if density.dtype != dt:
        raise ConfigError(f"density dtype {density.dtype} != the solve's {dt} (updated in place)")
    for name, v in (("f_gamma", f_gamma), ("g", g), ("density", density)):
        if v.numel() != n:
            raise ConfigError(f"{name} has {v.numel()} entries, expected n_ctl = {n}")
    if not density.is_contiguous():
        raise ConfigError("density must be contiguous (updated in place)")
    if m_rows is not None and tuple(F.shape) != m_rows:
        raise GridError(f"F shape {tuple(F.shape)} != {m_rows}")
    return (F.to(dt).contiguous(), f_gamma.to(dt).contiguous(), g.to(dt).contiguous())


def _allreduce_sum(t, nranks, group=None):
    if nranks == 1:
        return t
    dist = _dist()
    if dist is None:
        raise ConfigError("slab Richardson with nranks > 1 needs an initialised torch.distributed")
    dist.all_reduce(t, group=group)
    return t


class SlabRichardson:
    """The Richardson BVP solve of one rank of a slab-decomposed job.

    Rank g holds rows ``slab_rows(m, P, g)`` of F and of the returned field.
    Everything O(n_ctl) (density, jumps, edge values, traces, convergence) is
    replicated and computed identically on every rank; per sweep the ranks
    exchange the box-solve transposes (two all-to-alls) and one all-reduce of
    13 n_ctl stencil values (include/kfbi_b200.h, kfbi_slab_*).  The field,
    density and iteration counts are bit-identical to the one-GPU solve."""

    def __init__(self, workspace, nranks=None, rank=None, group=None, p2p=False, mode=None):
        dist = _dist()
        self.ws = workspace
        self.nranks = int(nranks if nranks is not None else (dist.get_world_size(group) if dist else 1))
        self.rank = int(rank if rank is not None else (dist.get_rank(group) if dist else 0))
        self.group = group
        self.rows = slab_rows(workspace.grid.m, self.nranks, self.rank)
        self.passes = SlabPasses(workspace.plan, self.nranks, self.rank, group,
                                 workspace.backend.torch_device, p2p, mode)

    def solve(self, *, kappa, F, f_gamma, g, density, F_sign=1.0, f_gamma_sign=1.0, gamma=0.8,
              tol=1e-8, max_iter=200, bc_kind="dirichlet"):
        """F: this rank's rows (rows, m+1); f_gamma, g, density: n_ctl device
        vectors (density updated in place).  Returns (u_slab, trace_u,
        trace_un, iterations, residual, history)."""
        import torch

        from .errors import ConvergenceError

        if bc_kind != "dirichlet":
            raise ConfigError("the slab-decomposed solve supports Dirichlet BVPs "
                              "(dirichlet-zero box)")
        ws, P, r = self.ws, self.nranks, self.rank
        plan = ws.plan
        ws.trace_tables()
        cplx = F.is_complex() or isinstance(kappa, complex) and complex(kappa).imag != 0
        dt = torch.complex128 if cplx else torch.float64
        dev = F.device
        n = ws.cps.m
        r0, r1 = self.rows
        F, f_gamma, g = _operands(dt, n, F, f_gamma, g, density, (r1 - r0, ws.grid.m + 1))
        jm = torch.empty(6 * n, dtype=dt, device=dev)
        jv = torch.empty(3 * max(int(ws.geometry.edge_theta.size), 1), dtype=dt, device=dev)
        vals = torch.empty(13 * n, dtype=dt, device=dev)
        tu = torch.empty(n, dtype=dt, device=dev)
        tn = torch.empty_like(tu)
        u = torch.empty_like(F)
        plan.rich_begin(max_iter, tol)
        it = done = 0
        res, hist = 0.0, []
        for _ in range(max_iter):
            plan.jumps(kappa, density, None, f_gamma, jm, f_gamma_sign)
            plan.edge_values(jm, jv)
            self.passes.run(cplx, kappa, F, u, sign=F_sign, jv=jv)
            plan.slab_stencil_values(bc_kind, P, r, u, vals)
            _allreduce_sum(vals, P, self.group)
            plan.slab_update(bc_kind, vals, jm, g, density, tu, tn, gamma)
            it, done, res, hist = plan.rich_state(max_iter)
            if done:
                break
        if done != 1:
            raise ConvergenceError(
                f"Richardson iteration did not reach tol={tol:g} within {max_iter} sweeps "
                f"(last density update {res:.3e})", iterations=max_iter, last_residual=res)
        return u, tu, tn, it, res, hist


def richardson_virtual(workspace, nranks, *, kappa, F, f_gamma, g, density, F_sign=1.0,
                       f_gamma_sign=1.0, gamma=0.8, tol=1e-8, max_iter=200, mode="a2a"):
    """The P-slab Richardson solve on ONE device (every rank's passes in
    turn, the exchanges as chunk copies, the all-reduce as a sum): the same
    kernels and layouts as SlabRichardson.  F: full (m+1)^2 field.  Returns
    (u full, trace_u, trace_un, iterations, residual, history)."""
    import torch

    from .errors import ConvergenceError

    ws, P = workspace, int(nranks)
    plan = ws.plan
    ws.trace_tables()
    m = ws.grid.m
    F = F.reshape(m + 1, m + 1)
    cplx = F.is_complex() or isinstance(kappa, complex) and complex(kappa).imag != 0
    dt = torch.complex128 if cplx else torch.float64
    dev = F.device
    n = ws.cps.m
    F, f_gamma, g = _operands(dt, n, F, f_gamma, g, density)
    rows = [slab_rows(m, P, q) for q in range(P)]
    jm = torch.empty(6 * n, dtype=dt, device=dev)
    jv = torch.empty(3 * max(int(ws.geometry.edge_theta.size), 1), dtype=dt, device=dev)
    vals = torch.empty(13 * n, dtype=dt, device=dev)
    part = torch.empty_like(vals)
    tu = torch.empty(n, dtype=dt, device=dev)
    tn = torch.empty_like(tu)
    nbytes = plan.slab_panel_bytes(cplx, P)
    send = [torch.empty(nbytes // 8, dtype=torch.float64, device=dev) for _ in range(P)]
    recv = [torch.empty_like(x) for x in send]
    Fs = [F[r0:r1].contiguous() for r0, r1 in rows]
    us = [torch.empty_like(f) for f in Fs]

    def a2a(dst, src):
        c = src[0].numel() // P
        for q in range(P):
            for h in range(P):
                dst[q][h * c:(h + 1) * c].copy_(src[h][q * c:(q + 1) * c])

    if mode == "carry":
        agg_b, flag_b = plan.slab_tri_bytes(cplx, P)
        agg = [torch.zeros(max(agg_b // 8, 1), dtype=torch.float64, device=dev) for _ in range(P)]
        flg = [torch.zeros(max(flag_b // 8, 1), dtype=torch.int64, device=dev) for _ in range(P)]
        epoch = 0
    plan.rich_begin(max_iter, tol)
    it = done = 0
    res, hist = 0.0, []
    for _ in range(max_iter):
        plan.jumps(kappa, density, None, f_gamma, jm, f_gamma_sign)
        plan.edge_values(jm, jv)
        for q in range(P):
            plan.slab_rows_fwd(cplx, P, q, Fs[q], send[q], sign=F_sign, jv=jv)
        if mode == "carry":
            epoch += 1
            plan.slab_cols_tri(cplx, P, 0, kappa, None, agg, flg, epoch, virt_panels=send)
        else:
            a2a(recv, send)
            for q in range(P):
                plan.slab_cols(cplx, P, q, kappa, recv[q])
            a2a(send, recv)
        vals.zero_()
        for q in range(P):
            plan.slab_rows_inv(cplx, P, q, send[q], us[q])
            plan.slab_stencil_values("dirichlet", P, q, us[q], part)
            vals += part
        plan.slab_update("dirichlet", vals, jm, g, density, tu, tn, gamma)
        it, done, res, hist = plan.rich_state(max_iter)
        if done:
            break
    if done != 1:
        raise ConvergenceError(f"no convergence in {max_iter} sweeps ({res:.3e})",
                               iterations=max_iter, last_residual=res)
    u = torch.zeros((m + 1, m + 1), dtype=dt, device=dev)
    for (r0, r1), uq in zip(rows, us):
        u[r0:r1] = uq
    return u, tu, tn, it, res, hist
