import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
BOX = (-1.5, 1.5, -1.5, 1.5)
PI_BOX = (-np.pi, np.pi, -np.pi, np.pi)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running checks")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_CACHE = {}


def golden(name):
    if name not in _CACHE:
        _CACHE[name] = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return _CACHE[name]


def setup_cases():
    import paper_2404_14864_b200 as k

    return {
        "disc32": (BOX, 32, k.CircleCurve(1.0)),
        "star64": (BOX, 64, k.StarCurve(1.0, c=0.2, lobes=3)),
        "flower128": (BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8)),
        "ellipse128": (BOX, 128, k.EllipseCurve(1.2, 0.8)),
        "pistar128": (PI_BOX, 128, k.StarCurve(1.5, c=0.2, lobes=3)),
    }


def box_rhs(m, seed, complex_rhs):
    rng = np.random.default_rng(seed)
    rhs = rng.standard_normal((m + 1, m + 1))
    if complex_rhs:
        rhs = rhs + 1j * rng.standard_normal((m + 1, m + 1))
    return rhs


# (tag, m, kappa, bc, seed, complex_rhs) — mirrors tests/golden/make_golden.py
BOX_CASES = [
    ("d16_k3p7", 16, 3.7, "dirichlet-zero", 101, False),
    ("d32_k3p7", 32, 3.7, "dirichlet-zero", 102, False),
    ("d128_k2048", 128, 2048.0, "dirichlet-zero", 103, False),
    ("d128_k0", 128, 0.0, "dirichlet-zero", 104, False),
    ("d64_kc", 64, 256j, "dirichlet-zero", 105, True),
    ("d32_kc_realrhs", 32, 2j, "dirichlet-zero", 106, False),
    ("n16_k3p7", 16, 3.7, "neumann-zero", 107, False),
    ("n64_k200", 64, 200.0, "neumann-zero", 108, False),
    ("n32_kc", 32, 256j, "neumann-zero", 109, True),
]


def run_cases():
    """Full-run golden cases (make_golden.run_cases), as ProblemSpec kwargs."""
    import paper_2404_14864_b200 as k

    heat = k.HeatPlaneDecay(c=1.0)
    wave = k.WaveStanding(phase=0.0)
    schr = k.SchrodingerPhaseRotation()
    return {
        "c1_heat_flower128": (BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8), dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=0.01, t_final=1.0, c=1.0)),
        "heat_flower64": (BOX, 64, k.StarCurve(1.0, c=0.2, lobes=5), dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=0.25, t_final=1.0, c=1.0)),
        "wave_ellipse128": (BOX, 128, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=0.125,
            t_final=1.0, theta=0.25)),
        "wave_ellipse64_th05": (BOX, 64, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=0.25,
            t_final=1.0, theta=0.5)),
        "schr_star128": (PI_BOX, 128, k.StarCurve(1.5, c=0.2, lobes=3), dict(
            equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
            lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=0.125,
            t_final=1.0)),
        "godunov_star64": (PI_BOX, 64, k.StarCurve(1.5, c=0.2, lobes=3), dict(
            equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
            lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=0.25,
            t_final=1.0, splitting="godunov")),
    }


def oracle_spec(kw):
    """ProblemSpec kwargs -> oracle Spec."""
    from oracle import kfbi_oracle as O

    keys = ("equation", "g", "u0", "lap_u0", "tau", "t_final", "c", "theta", "w", "potential",
            "splitting", "v0", "lap_v0", "bc_kind")
    return O.Spec(**{k: kw[k] for k in keys if k in kw})


def rel_linf(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (scale if scale > 0 else 1.0))


def neumann_run_cases():
    """Neumann full-run golden cases (make_golden.gen_neumann)."""
    import paper_2404_14864_b200 as k

    heat = k.HeatPlaneDecay(c=1.0)
    wave = k.WaveStanding(phase=0.0)
    return {
        "heat_flower64": (BOX, 64, k.StarCurve(1.0, c=0.2, lobes=5), dict(
            equation="heat", bc_kind="neumann", g=heat.neumann, u0=heat.u0,
            lap_u0=heat.lap_u0, tau=0.25, t_final=1.0, c=1.0)),
        "wave_ellipse64": (BOX, 64, k.EllipseCurve(1.2, 0.8), dict(
            equation="wave", bc_kind="neumann", g=wave.neumann, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, tau=0.25,
            t_final=1.0, theta=0.25)),
    }


NEUMANN_RICH_CASES = {
    "disc64_k16": (BOX, 64, "disc", 16.0),
    "flower128_k200": (BOX, 128, "flower8", 200.0),
}


def curve_of(tag):
    import paper_2404_14864_b200 as k

    return {"disc": k.CircleCurve(1.0), "flower8": k.StarCurve(1.0, c=0.2, lobes=8)}[tag]
