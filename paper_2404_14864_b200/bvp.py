"""Trace extraction and the Richardson solve of the boundary integral
equations (reference `bvp.py`).

`richardson_solve` keeps the whole iteration on the device: each sweep is
jumps -> streamed-W corrections -> box solve (corrections fused into the
row pass) -> extraction + density update + max-norm, and the host only
checks the device convergence flag once per batch of enqueued sweeps.  The
semantics are the reference's (bvp.py:276-351): the returned field is the one
of the converging sweep, the returned density includes that sweep's update,
and tol bounds max|γ(g - trace)|.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, ExtractionError

MAX_STENCIL_COND = 1e12
_TRI_OFFSETS = ((0, 0), (1, 0), (2, 0), (0, 1), (1, 1), (0, 2))


class TraceExtractor:
    """Six-point jump-corrected stencils for every control point
    (bvp.py:34-104).  Tables are built on the host once per workspace."""

    def __init__(self, workspace):
        self.workspace = workspace
        self.stencil_flat, self._ainv, self._jcoef = workspace.trace_tables()
        self.h = workspace.grid.h

    def extract(self, field, jumps, backend=None):
        """(u+, ux+, uy+) at all control points, computed on the device."""
        import torch

        from .device import to_device
        from .interface import _jm_device

        ws = self.workspace
        jm, cplx_j = _jm_device(jumps, ws)
        cplx = cplx_j or (field.is_complex() if isinstance(field, torch.Tensor)
                          else np.iscomplexobj(field))
        dt = np.complex128 if cplx else np.float64
        if cplx and not jm.is_complex():
            jm = jm.to(torch.complex128)
        u = to_device(field, dt, ws.backend)
        n = ws.cps.m
        out = torch.empty(3 * n, dtype=u.dtype, device=u.device)
        ws.plan.extract(u, jm, out)
        o = out.cpu().numpy().reshape(3, n)
        return o[0], o[1], o[2]


def extract_trace(field, jumps, extractor, backend=None):
    return extractor.extract(field, jumps, backend=backend)


class OneSidedExtractor:
    """Interior-only 7-node stencils for Neumann traces (bvp.py:115-228).

    The tables are built on the host exactly as the reference does and
    uploaded to the plan once (InterfaceWorkspace.ensure_onesided); the
    extraction runs on the device (kfbi_extract_onesided)."""

    def __init__(self, workspace):
        self.workspace = workspace
        geo = workspace.geometry
        grid = workspace.grid
        cps = workspace.cps
        interior = geo.classification.interior
        h, m = grid.h, grid.m
        xlo, _, ylo, _ = grid.box
        n = cps.m
        idx = np.zeros((n, 7, 2), dtype=int)
        rows = np.zeros((n, 3, 7))
        fallback = []
        for p in range(n):
            zx, zy = cps.x[p], cps.y[p]
            nx, ny = cps.normal[p]
            offs = _TRI_OFFSETS + (((3, 0),) if abs(nx) >= abs(ny) else ((0, 3),))
            ic = int(np.clip(round((zx - xlo) / h), 0, m))
            jc = int(np.clip(round((zy - ylo) / h), 0, m))
            dirs = sorted(((sx, sy) for sx in (-1, 1) for sy in (-1, 1)),
                          key=lambda s: s[0] * nx + s[1] * ny)
            nodes = self._find_nodes(grid, interior, zx, zy, ic, jc, offs, dirs)
            if nodes is None:
                fallback.append(p)
                continue
            ii, jj = nodes
            xi = (grid.x[ii] - zx) / h
            eta = (grid.y[jj] - zy) / h
            dn = -(xi * nx + eta * ny)
            a = np.stack([np.ones_like(xi), xi, eta, 0.5 * xi**2, xi * eta, 0.5 * eta**2,
                          dn**3 / 6.0], axis=1)
            if np.linalg.cond(a) > MAX_STENCIL_COND:
                fallback.append(p)
                continue
            idx[p, :, 0] = ii
            idx[p, :, 1] = jj
            rows[p] = np.linalg.inv(a)[:3]
        self.stencil_flat = grid.flat_index(idx[:, :, 0], idx[:, :, 1])
        self._rows = rows
        self._fallback = np.array(fallback, dtype=int)
        self._straddling = TraceExtractor(workspace) if fallback else None
        self.h = h

    @staticmethod
    def _find_nodes(grid, interior, zx, zy, ic, jc, offs, dirs):
        m = grid.m
        for w in (2, 3):
            best = None
            for dj in range(-w, w + 1):
                for di in range(-w, w + 1):
                    i, j = ic + di, jc + dj
                    if 0 <= i <= m and 0 <= j <= m and interior[j, i]:
                        d2 = (grid.x[i] - zx) ** 2 + (grid.y[j] - zy) ** 2
                        if best is None or d2 < best[0]:
                            best = (d2, i, j)
            if best is None:
                continue
            _, bi, bj = best
            for sx, sy in dirs:
                ii, jj = [], []
                for dx, dy in offs:
                    i, j = bi + sx * dx, bj + sy * dy
                    if not (0 <= i <= m and 0 <= j <= m and interior[j, i]):
                        break
                    ii.append(i)
                    jj.append(j)
                else:
                    return np.array(ii), np.array(jj)
        return None

    def extract(self, field, jumps, backend=None):
        """(u+, u_x+, u_y+) from the interior-only stencils, the straddling
        six-point stencil at the fallback points (bvp.py:214-228)."""
        import torch

        from .device import to_device
        from .interface import _jm_device

        ws = self.workspace
        ws.ensure_onesided()
        jm, cplx_j = _jm_device(jumps, ws)
        cplx = cplx_j or (field.is_complex() if isinstance(field, torch.Tensor)
                          else np.iscomplexobj(field))
        dt = np.complex128 if cplx else np.float64
        if cplx and not jm.is_complex():
            jm = jm.to(torch.complex128)
        u = to_device(field, dt, ws.backend)
        out = torch.empty(3 * ws.cps.m, dtype=u.dtype, device=u.device)
        ws.plan.extract_onesided(u, jm, out)
        c = out.cpu().numpy().reshape(3, ws.cps.m)
        return c[0], c[1], c[2]


@dataclass
class BvpProblem:
    """Dirichlet or Neumann BVP Δu - κu = f on Ω (bvp.py:231-262)."""

    kappa: complex
    F: np.ndarray
    f_gamma: np.ndarray
    bc_kind: str
    bc_values: np.ndarray
    gamma: float = 0.8
    tol: float = 1e-8
    max_iter: int = 200
    initial_density: np.ndarray = None
    box_bc: str = None

    def __post_init__(self):
        from .boxsolve import BOX_BCS

        if self.bc_kind not in ("dirichlet", "neumann"):
            raise ConfigError(f"unknown boundary condition kind {self.bc_kind!r}")
        if not 0.0 < self.gamma < 1.0:
            raise ConfigError(f"iteration parameter γ must lie strictly in (0,1), got {self.gamma}")
        if not self.tol > 0:
            raise ConfigError(f"tolerance must be positive, got {self.tol}")
        if self.max_iter < 1:
            raise ConfigError(f"max iterations must be ≥ 1, got {self.max_iter}")
        if self.box_bc is None:
            self.box_bc = "dirichlet-zero" if self.bc_kind == "dirichlet" else "neumann-zero"
        # the reference's own test expects this check (test_bvp.py:206-207)
        if self.box_bc not in BOX_BCS:
            raise ConfigError(f"unknown box boundary condition {self.box_bc!r}")


@dataclass
class BvpSolution:
    u: np.ndarray
    density: np.ndarray
    trace_u: np.ndarray
    trace_un: np.ndarray
    iterations: int
    residual: float
    residual_history: list = field(default_factory=list)


@dataclass
class DeviceBvp:
    """Device-resident result of one solve (tensors on the workspace device)."""

    u: object
    density: object
    trace_u: object
    trace_un: object
    iterations: int
    residual: float
    residual_history: list


def solve_device(ws, *, kappa, F, f_gamma, g, density, F_sign=1.0, f_gamma_sign=1.0,
                 gamma=0.8, tol=1e-8, max_iter=200, sweeps_hint=0, u_out=None,
                 use_operator=False, log_slot=-1, bc_kind="dirichlet", box_bc=None,
                 method="richardson", restart=40, field_chunks=False):
    """Richardson solve on device tensors (the inner loop of every time step).

    `density` is updated in place (it carries the warm start); F and f_gamma
    are read with the given signs (the steppers pass -F, -f_gamma,
    timestepping.py:180-190).  `use_operator` runs sweeps >= 2 through the
    workspace's precomputed trace operator (see InterfaceWorkspace
    .ensure_operator); sweep 1 and the returned field use the pipeline."""
    import torch

    cplx = F.is_complex()
    n = ws.cps.m
    if bc_kind == "neumann":
        ws.ensure_onesided()
    u = u_out if u_out is not None else torch.empty_like(F)
    tu = torch.empty(n, dtype=F.dtype, device=F.device)
    tn = torch.empty_like(tu)
    if method == "gmres":
        it, res, hist = ws.plan.gmres(
            kappa=kappa, F=F, F_sign=F_sign, f_gamma=f_gamma, f_gamma_sign=f_gamma_sign, g=g,
            density=density, gamma=gamma, tol=tol, max_iter=max_iter, u=u, trace_u=tu,
            trace_un=tn, restart=restart, use_operator=use_operator, bc_kind=bc_kind,
            box_bc=box_bc)
        return DeviceBvp(u=u, density=density, trace_u=tu, trace_un=tn, iterations=it,
                         residual=res, residual_history=hist)
    if method != "richardson":
        raise ConfigError(f"unknown BIE solver {method!r}; expected 'richardson' or 'gmres'")
    it, res, hist = ws.plan.richardson(
        kappa=kappa, F=F, F_sign=F_sign, f_gamma=f_gamma, f_gamma_sign=f_gamma_sign, g=g,
        density=density, gamma=gamma, tol=tol, max_iter=max_iter, u=u, trace_u=tu,
        trace_un=tn, sweeps_hint=sweeps_hint, use_operator=use_operator, log_slot=log_slot,
        bc_kind=bc_kind, box_bc=box_bc, field_chunks=field_chunks)
    del cplx
    return DeviceBvp(u=u, density=density, trace_u=tu, trace_un=tn, iterations=it,
                     residual=res, residual_history=hist)


def gmres_solve(problem, workspace, backend=None, restart=40):
    """Opt-in restarted GMRES on the same boundary integral equation as
    richardson_solve: the density solves T phi = g - t_F with
    T the trace operator; stops when gamma ||g - trace||_2 <= tol.  The field
    agrees with richardson_solve's to about tol (a different iterate of the
    same fixed point).  `iterations` counts matvecs plus full sweeps."""
    return _solve_problem(problem, workspace, method="gmres", restart=restart)


def richardson_solve(problem, workspace, backend=None, extractor=None):
    """Damped fixed-point iteration on the density (bvp.py:276-351), with
    every sweep on the device.  numpy in, numpy out."""
    dirichlet = problem.bc_kind == "dirichlet"
    want = TraceExtractor if dirichlet else OneSidedExtractor
    if extractor is not None and not isinstance(extractor, want):
        raise ConfigError(f"the device Richardson solve of a {problem.bc_kind} BVP uses the "
                          f"{want.__name__}")
    return _solve_problem(problem, workspace, method="richardson")


def _solve_problem(problem, ws, method, restart=40):
    from .device import to_device

    m_ctl = ws.cps.m
    if np.shape(problem.bc_values) != (m_ctl,):
        raise ConfigError(f"boundary data must have shape ({m_ctl},), got "
                          f"{np.shape(problem.bc_values)}")
    if problem.bc_kind == "dirichlet":
        ws.trace_tables()
    dtype = np.result_type(np.asarray(problem.F).dtype, np.asarray(problem.kappa).dtype,
                           np.asarray(problem.bc_values).dtype)
    cplx = np.issubdtype(dtype, np.complexfloating)
    dt = np.complex128 if cplx else np.float64
    mg = ws.grid.m
    F = to_device(problem.F, dt, ws.backend)
    fg = to_device(problem.f_gamma, dt, ws.backend)
    g = to_device(problem.bc_values, dt, ws.backend)
    dens0 = problem.initial_density if problem.initial_density is not None else np.zeros(m_ctl, dt)
    density = to_device(dens0, dt, ws.backend).clone()
    sol = solve_device(ws, kappa=problem.kappa, F=F, f_gamma=fg, g=g, density=density,
                       gamma=problem.gamma, tol=problem.tol, max_iter=problem.max_iter,
                       bc_kind=problem.bc_kind, box_bc=problem.box_bc, method=method,
                       restart=restart)
    return BvpSolution(
        u=sol.u.cpu().numpy().reshape(mg + 1, mg + 1),
        density=sol.density.cpu().numpy(),
        trace_u=sol.trace_u.cpu().numpy(),
        trace_un=sol.trace_un.cpu().numpy(),
        iterations=sol.iterations,
        residual=sol.residual,
        residual_history=sol.residual_history,
    )
