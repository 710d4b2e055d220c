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


class SlabBoxSolver:
    """Slab-decomposed BoxSolver (dirichlet-zero) for the calling rank.

    rhs / u are this rank's rows ``slab_rows(m, nranks, rank)`` as CUDA
    tensors of shape (rows, m + 1), float64 or complex128."""

    def __init__(self, grid, kappa, bc="dirichlet-zero", nranks=None, rank=None, group=None,
                 backend=None):
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
        self._bufs = {}

    def _panels(self, cplx):
        import torch

        key = bool(cplx)
        if key not in self._bufs:
            nbytes = self.plan.slab_panel_bytes(cplx, self.nranks)
            mk = lambda: torch.empty(nbytes // 8, dtype=torch.float64, device=self.backend.torch_device)
            self._bufs[key] = (mk(), mk() if self.nranks > 1 else None)
        return self._bufs[key]

    def solve(self, rhs):
        import torch

        m = self.grid.m
        r0, r1 = self.rows
        if tuple(rhs.shape) != (r1 - r0, m + 1):
            raise GridError(f"rhs slab shape {tuple(rhs.shape)} != ({r1 - r0}, {m + 1})")
        cplx = rhs.is_complex() or isinstance(self.kappa, complex)
        dt = torch.complex128 if cplx else torch.float64
        rhs = rhs.to(dt).contiguous()
        a, b = self._panels(cplx)
        u = torch.empty_like(rhs)
        p, P, g = self.plan, self.nranks, self.rank
        p.slab_rows_fwd(cplx, P, g, rhs, a)
        t = exchange_chunks(b, a, P, self.group)
        p.slab_cols(cplx, P, g, self.kappa, t)
        t = exchange_chunks(a, t, P, self.group)
        p.slab_rows_inv(cplx, P, g, t, u)
        return u


def solve_virtual(grid, kappa, rhs, nranks, backend=None):
    """The P-slab solve of a full (m+1)^2 rhs on ONE device: every rank's
    passes run in turn and the all-to-alls are chunk copies.  Returns the full
    solution (row m = zero ring)."""
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

