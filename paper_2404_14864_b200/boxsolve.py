"""Fast box solver for the five-point (Δ_h - κ)u = rhs (reference
`boxsolve.py`), on the device.

The dirichlet-zero closure diagonalises in the tensor-product sine basis with
eigenvalues (2cos(p pi/M) - 2)/h^2, p = 1..M-1 (boxsolve.py:1-9, 38-44).  The
solve is three sm_100a passes (rows DST-I, fused columns DST-I / scale /
DST-I, rows DST-I) in ``libkfbi_b200.so``; see csrc/box_reg.cuh.  The
neumann-zero closure is the same three passes with DCT-I (csrc/box_neu.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, GridError

BOX_BCS = ("dirichlet-zero", "neumann-zero")

_GRID_PLANS = {}


def _grid_plan(grid, backend):
    from ._plan import Plan

    key = (grid.m, grid.h, backend.device, id(backend))
    plan = _GRID_PLANS.get(key)
    if plan is None:
        plan = Plan(grid.m, grid.h, backend)
        _GRID_PLANS[key] = plan
    return plan


def _validate(bc, kappa):
    if bc not in BOX_BCS:
        raise ConfigError(f"unknown box boundary condition {bc!r}; expected one of {BOX_BCS}")
    if bc == "neumann-zero" and complex(kappa) == 0:
        raise ConfigError("neumann-zero box with κ = 0 is singular (constant null mode)")


class BoxSolver:
    """Box solver for one (grid, κ, closure) (boxsolve.py:25-94)."""

    def __init__(self, grid, kappa, bc, backend=None, _plan=None):
        _validate(bc, kappa)
        kappa = complex(kappa) if np.iscomplexobj(kappa) or isinstance(kappa, complex) else float(kappa)
        self.grid = grid
        self.kappa = kappa
        self.bc = bc
        from .engine import default_backend, make_backend

        self.backend = make_backend(backend) if backend is not None else default_backend()
        self._plan = _plan

    @property
    def plan(self):
        if self._plan is None:
            self._plan = _grid_plan(self.grid, self.backend)
        return self._plan

    @property
    def denom(self):
        """Eigenvalue denominators lam_p + lam_q - κ (host view for API
        compatibility; the device recomputes them from the 1-D table)."""
        m, h = self.grid.m, self.grid.h
        p = np.arange(1, m) if self.bc == "dirichlet-zero" else np.arange(0, m + 1)
        lam = (2.0 * np.cos(p * np.pi / m) - 2.0) / h**2
        return lam[:, None] + lam[None, :] - self.kappa

    def solve(self, rhs):
        """Full (M+1, M+1) solution.  dirichlet-zero reads rhs at interior
        nodes only and returns an exact zero ring; neumann-zero reads rhs
        everywhere (mirror ghost, DCT-I).  numpy in -> numpy out; a CUDA
        tensor in -> CUDA tensor out (no host round trip)."""
        import torch

        m = self.grid.m
        if tuple(rhs.shape) != (m + 1, m + 1):
            raise GridError(f"rhs shape {tuple(rhs.shape)} does not match grid ({m + 1}, {m + 1})")
        is_tensor = isinstance(rhs, torch.Tensor)
        rdt = np.complex128 if (rhs.is_complex() if is_tensor else np.iscomplexobj(rhs)) else np.float64
        out_dtype = np.result_type(rdt, np.asarray(self.kappa).dtype)
        from .device import to_device

        r = to_device(rhs, out_dtype, self.backend)
        u = torch.empty_like(r)
        self.plan.box_solve(r, u, self.kappa, self.bc)
        if is_tensor:
            return u.reshape(m + 1, m + 1)
        return u.cpu().numpy().reshape(m + 1, m + 1)


@dataclass
class BoxProblem:
    grid: object
    kappa: complex
    bc: str
    rhs: np.ndarray

    def __post_init__(self):
        _validate(self.bc, self.kappa)


def solve_box(problem, backend=None):
    return BoxSolver(problem.grid, problem.kappa, problem.bc, backend=backend).solve(problem.rhs)


def apply_box_operator(grid, u, kappa, bc):
    """Five-point (Δ_h - κ)u at the solve nodes (boxsolve.py:120-140).  A
    host verification utility (the residual oracle of the tests), not part of
    the solve."""
    m, h = grid.m, grid.h
    out = np.zeros_like(u, dtype=np.result_type(u.dtype, np.asarray(kappa).dtype))
    if bc == "dirichlet-zero":
        c = u[1:m, 1:m]
        out[1:m, 1:m] = (u[1:m, 2:] + u[1:m, :-2] + u[2:, 1:m] + u[:-2, 1:m] - 4.0 * c) / h**2 - kappa * c
    elif bc == "neumann-zero":
        e = np.pad(u, 1, mode="reflect")
        out[:, :] = (e[1:-1, 2:] + e[1:-1, :-2] + e[2:, 1:-1] + e[:-2, 1:-1]
                     - 4.0 * e[1:-1, 1:-1]) / h**2 - kappa * u
    else:
        raise ConfigError(f"unknown box boundary condition {bc!r}")
    return out
