"""Interface problem: jump relations, corrections at irregular nodes, and the
corrected box solve (reference `interface.py`).

Host side (run once per geometry): control points, the 3x3 jump-system
inverses, the trigonometric interpolation rows W (one row per unique
sign-change edge), the trace-extraction stencils, and their upload to a
device plan.  Device side (every sweep): the jump kernels, the streamed-W
correction kernel and the corrected box solve, all in ``libkfbi_b200.so``.

The functional API (`compute_jumps`, `corrections`, `solve_interface`) takes
and returns numpy arrays like the reference; the device-resident solver path
(`bvp.richardson_solve`, `timestepping.run`) never leaves the GPU per sweep.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ExtractionError, GeometryError, GridError
from .geometry import control_points, derivative_column

TRIG_INTERP_MIN_M = 32
MIN_CONTROL_SPACING = 1.8  # control arc spacing floor, in grid units (interface.py:108)
W_CHUNK_ROWS = 2048


def _trig_rows(query_theta, node_theta):
    """Cardinal trigonometric interpolation rows for an even node count:
    D(x) = sin(m x / 2) cos(x / 2) / (m sin(x / 2)), D(0) = 1, with x wrapped
    to (-pi, pi] (interface.py:38-52).  Evaluated in row chunks with the same
    element-wise expression, so the rows are identical to the reference's."""
    m = node_theta.size
    out = np.empty((query_theta.size, m))
    for s in range(0, query_theta.size, W_CHUNK_ROWS):
        q = query_theta[s:s + W_CHUNK_ROWS]
        x = np.mod(q[:, None] - node_theta[None, :] + np.pi, 2.0 * np.pi) - np.pi
        hit = np.abs(x) < 1e-12
        xs = np.where(hit, 1.0, x)
        rows = np.sin(0.5 * m * xs) * np.cos(0.5 * xs) / (m * np.sin(0.5 * xs))
        out[s:s + W_CHUNK_ROWS] = np.where(hit, 1.0, rows)
    return out


def _cubic_rows(query_theta, node_theta):
    """Periodic cubic-spline interpolation rows (interface.py:55-67)."""
    from scipy.interpolate import CubicSpline

    m = node_theta.size
    knots = np.append(node_theta, 2.0 * np.pi)
    q = np.mod(query_theta, 2.0 * np.pi)
    rows = np.empty((query_theta.size, m))
    for i in range(m):
        e = np.zeros(m + 1)
        e[i] = 1.0
        if i == 0:
            e[-1] = 1.0
        rows[:, i] = CubicSpline(knots, e, bc_type="periodic")(q)
    return rows


def interp_rows(query_theta, node_theta):
    """Interpolation rows from control nodes to query parameters
    (interface.py:70-75): trigonometric for an even count >= 32, else cubic."""
    query_theta = np.atleast_1d(np.asarray(query_theta, dtype=float))
    m = node_theta.size
    if m >= TRIG_INTERP_MIN_M and m % 2 == 0:
        return _trig_rows(query_theta, node_theta)
    return _cubic_rows(query_theta, node_theta)


@dataclass
class InterfaceData:
    """Data of one interface solve (interface.py:78-92)."""

    kappa: complex
    F: np.ndarray
    phi: np.ndarray
    psi: np.ndarray
    f_gamma: np.ndarray


@dataclass
class JumpSet:
    u: np.ndarray
    ux: np.ndarray
    uy: np.ndarray
    uxx: np.ndarray
    uxy: np.ndarray
    uyy: np.ndarray

    def as_matrix(self):
        return np.stack([self.u, self.ux, self.uy, self.uxx, self.uxy, self.uyy], axis=1)


def default_control_count(geometry):
    """Largest even count <= M whose minimum arc spacing stays >= 1.8h
    (interface.py:111-126)."""
    theta = np.linspace(0.0, 2.0 * np.pi, 4096, endpoint=False)
    speed_min = float(np.min(np.hypot(*geometry.curve.velocity(theta).T)))
    cap = speed_min * 2.0 * np.pi / (MIN_CONTROL_SPACING * geometry.grid.h)
    return max(8, min(geometry.grid.m, 2 * int(cap / 2.0)))


def trace_stencils(geometry, cps):
    """Six-point extraction stencils per control point (bvp.py:37-86): the
    four corners of the containing cell plus two outward neighbours of the
    nearest corner; the 6x6 inverses and the jump-shift coefficients."""
    from .bvp import MAX_STENCIL_COND

    grid = geometry.grid
    h = grid.h
    xlo, _, ylo, _ = grid.box
    zx, zy = cps.x, cps.y
    n = cps.m
    ic = np.clip(((zx - xlo) // h).astype(int), 0, grid.m - 1)
    jc = np.clip(((zy - ylo) // h).astype(int), 0, grid.m - 1)
    ci = np.stack([ic, ic + 1, ic, ic + 1], axis=1)
    cj = np.stack([jc, jc, jc + 1, jc + 1], axis=1)
    d2 = (grid.x[ci] - zx[:, None]) ** 2 + (grid.y[cj] - zy[:, None]) ** 2
    near = np.argmin(d2, axis=1)
    ni = ci[np.arange(n), near]
    nj = cj[np.arange(n), near]
    out_i = np.where(ni == ic, ic - 1, ic + 2)
    out_j = np.where(nj == jc, jc - 1, jc + 2)
    si = np.concatenate([ci, np.stack([out_i, ni], axis=1)], axis=1)
    sj = np.concatenate([cj, np.stack([nj, out_j], axis=1)], axis=1)
    if si.min() < 0 or sj.min() < 0 or si.max() > grid.m or sj.max() > grid.m:
        raise ExtractionError("extraction stencil leaves the box; Γ too close to ∂B")
    stencil = grid.flat_index(si, sj)
    dx = grid.x[si] - zx[:, None]
    dy = grid.y[sj] - zy[:, None]
    xi, eta = dx / h, dy / h
    a = np.stack([np.ones_like(xi), xi, eta, 0.5 * xi**2, xi * eta, 0.5 * eta**2], axis=2)
    cond = np.linalg.cond(a)
    if np.any(~np.isfinite(cond)) or cond.max() > MAX_STENCIL_COND:
        raise ExtractionError(f"six-point stencil condition number {cond.max():.3g} exceeds "
                              f"{MAX_STENCIL_COND:.0e}")
    ainv = np.linalg.inv(a)
    exterior = ~geometry.classification.interior.ravel()[stencil]
    rows = np.stack([np.ones_like(dx), dx, dy, 0.5 * dx**2, dx * dy, 0.5 * dy**2], axis=2)
    jcoef = rows * exterior[:, :, None]
    return stencil, ainv, jcoef


class InterfaceWorkspace:
    """Geometry-dependent precomputation shared by every interface solve
    (interface.py:129-168), plus the device plan that holds it on the GPU."""

    def __init__(self, geometry, n_controls=None, backend=None):
        self.geometry = geometry
        self.grid = geometry.grid
        self.records = geometry.records
        self._backend = backend
        m = default_control_count(geometry) if n_controls is None else int(n_controls)
        self.cps = control_points(geometry.curve, m)

        t1, t2 = self.cps.tangent[:, 0], self.cps.tangent[:, 1]
        a = np.empty((m, 3, 3))
        a[:, 0] = np.stack([t1 * t1, 2.0 * t1 * t2, t2 * t2], axis=1)
        a[:, 1] = np.stack([t1 * t2, t2 * t2 - t1 * t1, -t1 * t2], axis=1)
        a[:, 2] = np.stack([np.ones(m), np.zeros(m), np.ones(m)], axis=1)
        if np.any(np.abs(np.linalg.det(a)) < 0.5):
            raise GeometryError("second-derivative jump system is near singular")
        self._inv3 = np.linalg.inv(a)

        # one interpolation row per unique sign-change edge; both records of
        # an edge share theta (grid.py:243-254), so w_records = w_edges[edge].
        # Built lazily on the host (API views, tests); the device plan builds
        # its own copy from the parameters (kfbi_plan_set_geometry)
        self._w_edges = None
        self._box_solvers = {}
        self._plan = None
        self._trace = None
        self._onesided = None
        self._trace_error = None

    # -- host views kept for API compatibility --------------------------------
    @property
    def w_edges(self):
        if self._w_edges is None:
            self._w_edges = interp_rows(self.geometry.edge_theta, self.cps.theta)
        return self._w_edges

    @property
    def device_w(self):
        """W is built on the device when the trigonometric form applies."""
        m = self.cps.m
        return m >= TRIG_INTERP_MIN_M and m % 2 == 0

    @property
    def w_records(self):
        return self.w_edges[self.records.edge]

    @property
    def backend(self):
        if self._backend is None:
            from .engine import default_backend

            self._backend = default_backend()
        elif not hasattr(self._backend, "register"):
            from .engine import make_backend

            self._backend = make_backend(self._backend)
        return self._backend

    def trace_tables(self):
        """(stencil, ainv, jcoef) of the six-point extractor, built once."""
        if self._trace is None and self._trace_error is None:
            try:
                self._trace = trace_stencils(self.geometry, self.cps)
            except ExtractionError as exc:
                self._trace_error = exc
        if self._trace_error is not None:
            raise self._trace_error
        return self._trace

    def device_tables(self):
        rec = self.records
        grid = self.grid
        n = self.cps.m
        try:
            stencil, ainv, jcoef = self.trace_tables()
        except ExtractionError:
            stencil = np.zeros((n, 6), int)
            ainv = np.zeros((n, 6, 6))
            jcoef = np.zeros((n, 6, 6))
        sigma = np.where(rec.owner_interior, -1.0, 1.0) / grid.h**2
        starts = np.append(rec.group_starts, rec.n)
        owners = rec.group_owners
        owner_row = owners // (grid.m + 1)
        row_group = np.searchsorted(owner_row, np.arange(grid.m + 2), side="left")
        return {
            "n_ctl": n,
            "w_edges": None if self.device_w else self.w_edges,
            "edge_theta": self.geometry.edge_theta,
            "ctl_theta": self.cps.theta,
            "edge_axis": self.geometry.edge_axis,
            "rec_edge": rec.edge,
            "rec_d": rec.d,
            "rec_sigma": sigma,
            "group_start": starts,
            "group_node": owners,
            "row_group": row_group,
            "deriv_col": derivative_column(self.cps),
            "speed": self.cps.speed,
            "tangent": self.cps.tangent,
            "normal": self.cps.normal,
            "dtan_ds": self.cps.dtan_ds,
            "inv3": self._inv3,
            "stencil": stencil,
            "ainv_rows": ainv[:, :3, :],
            "jcoef": jcoef,
        }

    @property
    def plan(self):
        """Device plan with this workspace's tables (built on first use)."""
        if self._plan is None:
            from ._plan import Plan

            plan = Plan(self.grid.m, self.grid.h, self.backend)
            plan.set_geometry(self.device_tables())
            self._plan = plan
        return self._plan

    def ensure_operator(self, kappa, cplx, bc_kind="dirichlet", box_bc=None):
        """Build (once per kappa and BVP kind) the explicit trace operator used
        by the operator form of the Richardson sweeps."""
        box_bc = box_bc or ("dirichlet-zero" if bc_kind == "dirichlet" else "neumann-zero")
        if bc_kind == "neumann":
            self.ensure_onesided()
        key = (complex(kappa), bool(cplx), bc_kind, box_bc)
        if getattr(self.plan, "operator_key", None) != key:
            self.plan.build_operator(kappa, cplx, bc_kind, box_bc)

    def onesided(self):
        """The OneSidedExtractor of this workspace (host tables, built once)."""
        if self._onesided is None:
            from .bvp import OneSidedExtractor

            self._onesided = OneSidedExtractor(self)
        return self._onesided

    def ensure_onesided(self):
        """Upload the one-sided extraction tables to the plan (Neumann BVPs)."""
        if not getattr(self.plan, "has_onesided", False):
            ex = self.onesided()
            fb = np.zeros(self.cps.m, np.uint8)
            fb[ex._fallback] = 1
            if len(ex._fallback):
                self.trace_tables()         # the fallback points use the 6-point tables
            self.plan.set_onesided(ex.stencil_flat, ex._rows, fb)

    def box_solver(self, kappa, bc):
        key = (complex(kappa), bc)
        if key not in self._box_solvers:
            from .boxsolve import BoxSolver

            self._box_solvers[key] = BoxSolver(self.grid, kappa, bc, backend=self.backend,
                                               _plan=self.plan)
        return self._box_solvers[key]


# ---------------------------------------------------------------------------
# functional API (numpy in, numpy out; device kernels inside)

def _dtype_of(*arrays_and_scalars):
    return np.result_type(*[np.asarray(a) for a in arrays_and_scalars])


def _dev(ws, a, dtype):
    from .device import to_device

    return to_device(a, dtype, ws.backend)


def _jumps_device(data, ws):
    import torch

    cps = ws.cps
    m = cps.m
    for name, arr in (("phi", data.phi), ("psi", data.psi), ("f_gamma", data.f_gamma)):
        if np.shape(arr) != (m,):
            raise GridError(f"{name} must have shape ({m},), got {np.shape(arr)}")
    dtype = _dtype_of(data.phi, data.psi, data.f_gamma, data.kappa)
    cplx = np.issubdtype(dtype, np.complexfloating)
    dt = np.complex128 if cplx else np.float64
    plan = ws.plan
    jm = torch.empty(6 * m, dtype=torch.complex128 if cplx else torch.float64,
                     device=ws.backend.torch_device)
    plan.jumps(data.kappa, _dev(ws, data.phi, dt), _dev(ws, data.psi, dt),
               _dev(ws, data.f_gamma, dt), jm)
    return jm, cplx


def _jumpset_from_soa(jm_host, m):
    cols = jm_host.reshape(6, m)
    return JumpSet(*(cols[k].copy() for k in range(6)))


def compute_jumps(data, workspace, backend=None):
    """Jumps of u and its first/second derivatives at the control points
    (interface.py:171-203), computed on the device."""
    jm, _ = _jumps_device(data, workspace)
    return _jumpset_from_soa(jm.cpu().numpy(), workspace.cps.m)


def _jm_device(jumps, ws):
    """JumpSet -> device SoA [6][n]."""
    mat = jumps.as_matrix()
    cplx = np.iscomplexobj(mat)
    dt = np.complex128 if cplx else np.float64
    return _dev(ws, np.ascontiguousarray(mat.T), dt), cplx


def corrections(jumps, workspace, backend=None):
    """Right-hand-side corrections at irregular nodes (interface.py:206-238),
    computed on the device from the streamed interpolation rows."""
    import torch

    jm, cplx = _jm_device(jumps, workspace)
    m = workspace.grid.m
    c = torch.empty((m + 1) * (m + 1), dtype=jm.dtype, device=jm.device)
    workspace.plan.corrections(jm, c)
    return c.cpu().numpy().reshape(m + 1, m + 1)


def jump_at_point(jumps, theta, workspace):
    """All six jumps interpolated to parameter(s) theta (host utility,
    interface.py:241-247)."""
    out = interp_rows(theta, workspace.cps.theta) @ jumps.as_matrix()
    if np.isscalar(theta) or np.ndim(theta) == 0:
        return tuple(out[0])
    return out


def solve_interface(data, workspace, box_bc, backend=None):
    """Δu - κu = F with jumps (phi, psi) across Γ and a homogeneous box
    closure (interface.py:250-261): jumps, corrections and the box solve run
    back to back on the device."""
    import torch

    from .boxsolve import BOX_BCS
    from .errors import ConfigError

    if box_bc not in BOX_BCS:
        raise ConfigError(f"unknown box boundary condition {box_bc!r}; expected one of {BOX_BCS}")
    if box_bc == "neumann-zero" and complex(data.kappa) == 0:
        raise ConfigError("neumann-zero box with κ = 0 is singular (constant null mode)")
    ws = workspace
    jm, cplx = _jumps_device(data, ws)
    cplx = cplx or np.iscomplexobj(np.asarray(data.F))
    dt = np.complex128 if cplx else np.float64
    if cplx and not jm.is_complex():
        jm = jm.to(torch.complex128)
    m = ws.grid.m
    F = _dev(ws, data.F, dt)
    u = torch.empty_like(F)
    ws.plan.interface_solve(data.kappa, F, jm, u, box_bc)
    return u.cpu().numpy().reshape(m + 1, m + 1)
