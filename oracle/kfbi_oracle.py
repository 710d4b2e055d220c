"""CPU oracle for the KFBI hot path — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's per-time-step solve (the
reference package `/root/reference/pkg/src/kfbi` is pure Python; its native
arithmetic comes from scipy 1.18.1's ducc0 DST/DCT, numpy 2.3.5's pocketfft
and OpenBLAS 0.3.30, the versions recorded in tests/golden/*.npz).  Each
function cites the reference file:line it follows.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module, and only as the checker / the timed CPU baseline.  The product
package never imports it.

Parity pinning: tests/test_oracle.py checks this module against the golden
vectors produced by the unmodified reference (tests/golden/make_golden.py):
box solves, jumps, corrections, extraction, Richardson solves and full runs.

Inputs are plain arrays (a `Tables` bundle), so the oracle does not depend on
the product's code; `tables_from_workspace` reads them off any object with
the reference's InterfaceWorkspace attribute names.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
from scipy.fft import dct, dst, idct, idst

WORKERS = int(os.environ.get("KFBI_ORACLE_WORKERS", "1"))


# ---------------------------------------------------------------------------
# setup tables

@dataclass
class Tables:
    m: int
    h: float
    mask: np.ndarray            # (M+1, M+1) bool interior
    X: np.ndarray
    Y: np.ndarray
    # control points
    ctl_x: np.ndarray
    ctl_y: np.ndarray
    theta: np.ndarray
    dtheta: float
    tangent: np.ndarray
    normal: np.ndarray
    dtan_ds: np.ndarray
    speed: np.ndarray
    inv3: np.ndarray
    # records
    w_records: np.ndarray       # (n_rec, n_ctl)
    rec_d: np.ndarray
    rec_axis: np.ndarray
    rec_owner_interior: np.ndarray
    group_starts: np.ndarray
    group_owners: np.ndarray
    # six-point extractor
    stencil: np.ndarray
    ainv: np.ndarray
    jcoef: np.ndarray
    # one-sided extractor (Neumann; bvp.py:115-212), optional
    os_stencil: np.ndarray = None
    os_rows: np.ndarray = None
    os_fallback: np.ndarray = None


def tables_from_workspace(ws, onesided=False):
    grid, cps, rec = ws.grid, ws.cps, ws.records
    stencil, ainv, jcoef = ws.trace_tables()
    os_tabs = {}
    if onesided:
        ox = ws.onesided()
        os_tabs = dict(os_stencil=ox.stencil_flat, os_rows=ox._rows, os_fallback=ox._fallback)
    return Tables(
        m=grid.m, h=grid.h, mask=ws.geometry.classification.interior, X=grid.X, Y=grid.Y,
        ctl_x=cps.x, ctl_y=cps.y, theta=cps.theta, dtheta=cps.dtheta, tangent=cps.tangent,
        normal=cps.normal, dtan_ds=cps.dtan_ds, speed=cps.speed, inv3=ws._inv3,
        w_records=ws.w_records, rec_d=rec.d, rec_axis=rec.axis,
        rec_owner_interior=rec.owner_interior, group_starts=rec.group_starts,
        group_owners=rec.group_owners, stencil=stencil, ainv=ainv, jcoef=jcoef, **os_tabs)


# ---------------------------------------------------------------------------
# box solve — boxsolve.py:38-44 (eigenvalues), :46-94 (dirichlet-zero solve)

def eigen_denominators(m, h, kappa, bc="dirichlet-zero"):
    p = np.arange(1, m) if bc == "dirichlet-zero" else np.arange(0, m + 1)
    lam = (2.0 * np.cos(p * np.pi / m) - 2.0) / h**2
    return lam[:, None] + lam[None, :] - kappa


def box_solve(m, h, kappa, rhs, denom=None, bc="dirichlet-zero"):
    """(Δ_h - κ) u = rhs.  dirichlet-zero: u = 0 on the box ring, DST-I rows,
    DST-I columns, divide, inverse columns, inverse rows (boxsolve.py:58-93);
    neumann-zero: the same with DCT-I over the whole grid (mirror ghost)."""
    if denom is None:
        denom = eigen_denominators(m, h, kappa, bc)
    dtype = np.result_type(rhs.dtype, np.asarray(kappa).dtype)
    if bc == "neumann-zero":
        w = np.array(rhs, dtype=dtype)
        w = dct(w, type=1, axis=1, workers=WORKERS)
        w = dct(w, type=1, axis=0, workers=WORKERS)
        w /= denom
        w = idct(w, type=1, axis=0, workers=WORKERS)
        return idct(w, type=1, axis=1, workers=WORKERS)
    w = np.array(rhs[1:m, 1:m], dtype=dtype)
    w = dst(w, type=1, axis=1, workers=WORKERS)
    w = dst(w, type=1, axis=0, workers=WORKERS)
    w /= denom
    w = idst(w, type=1, axis=0, workers=WORKERS)
    w = idst(w, type=1, axis=1, workers=WORKERS)
    u = np.zeros((m + 1, m + 1), dtype=dtype)
    u[1:m, 1:m] = w
    return u


# ---------------------------------------------------------------------------
# boundary calculus — geometry.py:415-444

def _spectral_dtheta(values, dtheta):
    m = values.shape[-1]
    k = np.fft.fftfreq(m) * m
    if m % 2 == 0:
        k[m // 2] = 0.0
    dv = np.fft.ifft(np.fft.fft(values) * (1j * k * (2.0 * np.pi / (m * dtheta))))
    return dv.real if np.isrealobj(values) else dv


def arc_derivatives(values, t):
    d1 = _spectral_dtheta(values, t.dtheta) / t.speed
    d2 = _spectral_dtheta(d1, t.dtheta) / t.speed
    return d1, d2


# ---------------------------------------------------------------------------
# jumps — interface.py:171-203 ; returns JM (n_ctl, 6): u ux uy uxx uxy uyy

def jumps(t, kappa, phi, psi, f_gamma):
    phi_s, phi_ss = arc_derivatives(phi, t)
    psi_s, _ = arc_derivatives(psi, t)
    t1, t2 = t.tangent[:, 0], t.tangent[:, 1]
    dt1, dt2 = t.dtan_ds[:, 0], t.dtan_ds[:, 1]
    dtype = np.result_type(phi, psi, f_gamma, np.asarray(kappa))
    ju = np.asarray(phi, dtype=dtype)
    jx = t1 * phi_s + t2 * psi
    jy = t2 * phi_s - t1 * psi
    r = np.empty((phi.size, 3), dtype=dtype)
    r[:, 0] = phi_ss - dt1 * jx - dt2 * jy
    r[:, 1] = psi_s - dt2 * jx + dt1 * jy
    r[:, 2] = f_gamma + kappa * ju
    j2 = np.einsum("pij,pj->pi", t.inv3, r)
    return np.stack([ju, jx.astype(dtype), jy.astype(dtype), j2[:, 0], j2[:, 1], j2[:, 2]], axis=1)


# ---------------------------------------------------------------------------
# corrections — interface.py:206-238

def corrections(t, jm):
    j = t.w_records @ jm
    horiz = t.rec_axis == 0
    j1 = np.where(horiz, j[:, 1], j[:, 2])
    j2 = np.where(horiz, j[:, 3], j[:, 5])
    sigma = np.where(t.rec_owner_interior, -1.0, 1.0) / t.h**2
    vals = sigma * (j[:, 0] + j1 * t.rec_d + 0.5 * j2 * t.rec_d**2)
    c = np.zeros((t.m + 1) ** 2, dtype=jm.dtype)
    if vals.size:
        c[t.group_owners] = np.add.reduceat(vals, t.group_starts)
    return c.reshape(t.m + 1, t.m + 1)


# ---------------------------------------------------------------------------
# six-point extraction — bvp.py:88-104

def extract(t, field, jm):
    flat = field.ravel()
    vals = flat[t.stencil] + np.einsum("pnk,pk->pn", t.jcoef, jm)
    coeffs = np.einsum("pij,pj->pi", t.ainv, vals)
    return coeffs[:, 0], coeffs[:, 1] / t.h, coeffs[:, 2] / t.h


# one-sided extraction — bvp.py:214-228 (Neumann)
def extract_onesided(t, field, jm):
    flat = field.ravel()
    dtype = np.result_type(flat.dtype, float)
    coeffs = np.einsum("pin,pn->pi", t.os_rows, flat[t.os_stencil]).astype(dtype)
    fb = t.os_fallback
    if len(fb):
        su, sx, sy = extract(t, field, jm)
        coeffs[fb, 0] = su[fb]
        coeffs[fb, 1] = sx[fb] * t.h
        coeffs[fb, 2] = sy[fb] * t.h
    return coeffs[:, 0], coeffs[:, 1] / t.h, coeffs[:, 2] / t.h


# ---------------------------------------------------------------------------
# Richardson — bvp.py:276-351 (Dirichlet)

@dataclass
class Solution:
    u: np.ndarray
    density: np.ndarray
    trace_u: np.ndarray
    trace_un: np.ndarray
    iterations: int
    residual: float
    history: list = field(default_factory=list)


class NotConverged(Exception):
    def __init__(self, iterations, last_residual):
        super().__init__(f"no convergence in {iterations} sweeps ({last_residual:.3e})")
        self.iterations = iterations
        self.last_residual = last_residual


def richardson(t, kappa, F, f_gamma, g, density0=None, gamma=0.8, tol=1e-8, max_iter=200,
               max_sweeps=None, bc_kind="dirichlet"):
    """Damped fixed point φ <- φ + γ(g - u+[φ]) (Dirichlet) or
    ψ <- ψ + γ(g - ∂ₙu+[ψ]) (Neumann: neumann-zero box, one-sided
    extraction).  Returns the field of the converging sweep and the density
    after its update.  `max_sweeps` stops early (timing samples) without
    raising."""
    dirichlet = bc_kind == "dirichlet"
    box_bc = "dirichlet-zero" if dirichlet else "neumann-zero"
    dtype = np.result_type(F.dtype, np.asarray(kappa).dtype, np.asarray(g).dtype)
    n = t.theta.size
    density = (np.array(density0, dtype=dtype) if density0 is not None
               else np.zeros(n, dtype=dtype))
    zero = np.zeros(n, dtype=dtype)
    g = np.asarray(g, dtype=dtype)
    denom = eigen_denominators(t.m, t.h, kappa, box_bc)
    history = []
    for it in range(1, max_iter + 1):
        if dirichlet:
            jm = jumps(t, kappa, density, zero, f_gamma)
        else:
            jm = jumps(t, kappa, zero, density, f_gamma)
        c = corrections(t, jm)
        u = box_solve(t.m, t.h, kappa, F + c, denom, box_bc)
        tu, tx, ty = (extract if dirichlet else extract_onesided)(t, u, jm)
        tun = tx * t.normal[:, 0] + ty * t.normal[:, 1]
        update = gamma * (g - (tu if dirichlet else tun))
        density += update
        res = float(np.max(np.abs(update)))
        history.append(res)
        if res <= tol or (max_sweeps is not None and it >= max_sweeps):
            return Solution(u, density, tu, tun, it, res, history)
    raise NotConverged(max_iter, history[-1])


# ---------------------------------------------------------------------------
# steppers — timestepping.py:178-515 (Dirichlet)

def interior_field(t, fn):
    vals = np.asarray(fn(t.X, t.Y))
    return np.where(t.mask, vals, np.zeros((), dtype=vals.dtype))


def nonlinear_phase(values, v, w, half_tau, tol=1e-12, max_iter=50):
    """Vectorised damped Newton of timestepping.py:317-368."""
    us = np.asarray(values, dtype=complex)
    if us.size == 0:
        return us
    c = half_tau
    rhs = us - 1j * c * (v + w * np.abs(us) ** 2) * us
    r1, r2 = rhs.real.copy(), rhs.imag.copy()

    def resid(a, b):
        nv = v + w * (a * a + b * b)
        return a - c * nv * b - r1, b + c * nv * a - r2

    a, b = us.real.copy(), us.imag.copy()
    g1, g2 = resid(a, b)
    res = np.maximum(np.abs(g1), np.abs(g2))
    for _ in range(max_iter):
        active = res > tol
        if not np.any(active):
            break
        nv = v + w * (a * a + b * b)
        j11 = 1.0 - 2.0 * c * w * a * b
        j12 = -c * nv - 2.0 * c * w * b * b
        j21 = c * nv + 2.0 * c * w * a * a
        j22 = 1.0 + 2.0 * c * w * a * b
        det = j11 * j22 - j12 * j21
        da = (j22 * g1 - j12 * g2) / det
        db = (j11 * g2 - j21 * g1) / det
        step = np.where(active, 1.0, 0.0)
        for _h in range(30):
            an, bn = a - step * da, b - step * db
            g1, g2 = resid(an, bn)
            rn = np.maximum(np.abs(g1), np.abs(g2))
            worse = active & (rn > res)
            if not np.any(worse):
                break
            step = np.where(worse, 0.5 * step, step)
        a, b, res = an, bn, rn
    if np.any(res > tol):
        raise NotConverged(max_iter, float(res.max()))
    return a + 1j * b


@dataclass
class Spec:
    equation: str
    g: callable
    u0: callable
    lap_u0: callable
    tau: float
    t_final: float
    c: float = 1.0
    theta: float = 0.25
    w: float = 1.0
    potential: callable = None
    splitting: str = "strang"
    v0: callable = None
    lap_v0: callable = None
    gamma: float = 0.8
    tol: float = 1e-8
    max_iter: int = 200
    bc_kind: str = "dirichlet"

    def n_steps(self):
        return int(round(self.t_final / self.tau))


class Stepper:
    """Rolling state of one evolution (timestepping.py:119-136, 203-450)."""

    def __init__(self, t, spec, max_sweeps=None):
        self.t, self.spec = t, spec
        self.max_sweeps = max_sweeps
        self.iterations = []
        self.n = 0
        self.time = 0.0
        self.density = None
        zx, zy = t.ctl_x, t.ctl_y
        s = spec
        if s.equation == "heat":
            a = 2.0 * s.c / s.tau
            self.u = interior_field(t, s.u0)
            self.F = a * self.u + interior_field(t, s.lap_u0)
            self.fg = a * s.u0(zx, zy) + s.lap_u0(zx, zy)
        elif s.equation == "wave":
            tau, th = s.tau, s.theta
            kw = 1.0 / (th * tau**2)
            coef = (1.0 - 2.0 * th) / th
            u0 = interior_field(t, s.u0)
            lu0 = interior_field(t, s.lap_u0)
            u1 = u0 + tau * interior_field(t, s.v0) + 0.5 * tau**2 * lu0
            lu1 = lu0 + tau * interior_field(t, s.lap_v0)
            self.u, self.u_prev = u1, u0
            self.F_prev = kw * u1 - lu1
            self.F = (2.0 * u1 - u0) * kw + coef * lu1 + lu0
            gu0, glu0 = s.u0(zx, zy), s.lap_u0(zx, zy)
            gu1 = gu0 + tau * s.v0(zx, zy) + 0.5 * tau**2 * glu0
            glu1 = glu0 + tau * s.lap_v0(zx, zy)
            self.fg_prev = kw * gu1 - glu1
            self.fg = (2.0 * gu1 - gu0) * kw + coef * glu1 + glu0
            self.trace = gu1
            self.n, self.time = 1, tau
        else:
            self.u = interior_field(t, s.u0).astype(complex)
            self.carry = None
            self.carry_gamma = None

    def _solve(self, kappa, F, fg, g):
        sol = richardson(self.t, kappa, -F, -fg, g, self.density, self.spec.gamma, self.spec.tol,
                         self.spec.max_iter, max_sweeps=self.max_sweeps,
                         bc_kind=self.spec.bc_kind)
        self.density = sol.density
        self.iterations.append(sol.iterations)
        return sol

    def _g(self, time):
        """Boundary data at the controls (timestepping.py:166-170)."""
        t, s = self.t, self.spec
        if s.bc_kind == "neumann":
            return np.asarray(s.g(t.ctl_x, t.ctl_y, time, t.normal))
        return np.asarray(s.g(t.ctl_x, t.ctl_y, time))

    def step(self):
        t, s = self.t, self.spec
        zx, zy = t.ctl_x, t.ctl_y
        t_next = self.time + s.tau
        neumann = s.bc_kind == "neumann"
        if s.equation == "heat":
            kappa = 2.0 * s.c / s.tau
            g = self._g(t_next)
            sol = self._solve(kappa, self.F, self.fg, g)
            u_next = np.where(t.mask, sol.u, 0.0)
            a = 4.0 * s.c / s.tau
            self.F = a * u_next - self.F
            trace = sol.trace_u if neumann else g          # timestepping.py:230
            self.fg = a * trace - self.fg
            self.u = u_next
        elif s.equation == "wave":
            tau, th = s.tau, s.theta
            kw = 1.0 / (th * tau**2)
            coef = (1.0 - 2.0 * th) / th
            sol = self._solve(kw, self.F, self.fg, self._g(t_next))
            g_next = sol.trace_u if neumann else self._g(t_next)   # timestepping.py:299
            un = np.where(t.mask, sol.u, 0.0)
            uc = self.u
            F_new = (2.0 * un - uc) * kw + coef * (kw * un - self.F) + (kw * uc - self.F_prev)
            fg_new = ((2.0 * g_next - self.trace) * kw + coef * (kw * g_next - self.fg)
                      + (kw * self.trace - self.fg_prev))
            self.u_prev, self.u = uc, un
            self.F_prev, self.F = self.F, F_new
            self.fg_prev, self.fg = self.fg, fg_new
            self.trace = g_next
        else:
            godunov = s.splitting == "godunov"
            kappa = (1j if godunov else 2j) / s.tau
            if godunov:
                ustar = self.u.astype(complex)
                ustar_g = s.g(zx, zy, self.time).astype(complex)
            elif self.carry is None:
                ustar = self.u - 0.5j * s.tau * interior_field(t, s.lap_u0).astype(complex)
                ustar_g = (np.asarray(s.u0(zx, zy), dtype=complex)
                           - 0.5j * s.tau * np.asarray(s.lap_u0(zx, zy)))
            else:
                ustar = 2.0 * self.u - self.carry
                ustar_g = 2.0 * s.g(zx, zy, self.time).astype(complex) - self.carry_gamma
            v_grid = np.where(t.mask, s.potential(t.X, t.Y), 0.0)
            v_g = s.potential(zx, zy)
            carry = nonlinear_phase(ustar.ravel(), v_grid.ravel(), s.w, 0.5 * s.tau)
            carry = np.where(t.mask, carry.reshape(ustar.shape), 0.0)
            carry_g = nonlinear_phase(ustar_g, v_g, s.w, 0.5 * s.tau)
            sol = self._solve(kappa, kappa * carry, kappa * carry_g, s.g(zx, zy, t_next))
            self.u = np.where(t.mask, sol.u, 0.0)
            if not godunov:
                self.carry, self.carry_gamma = carry, carry_g
        self.n += 1
        self.time = t_next
        return self


def run(t, spec, max_sweeps=None):
    st = Stepper(t, spec, max_sweeps=max_sweeps)
    while st.n < spec.n_steps():
        st.step()
    return st
