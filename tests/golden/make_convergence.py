"""Golden convergence tables (SURVEY §6.3 / BASELINE config C4) from the
UNMODIFIED reference: e_inf, e_2 and the per-step Richardson iteration counts
of the three equations at M = 64, 128, 256 (and 512 for heat), with the
convergence rule tau = 0.25 * 64 / M, T = 1, Dirichlet data.

    python tests/golden/make_convergence.py      # writes convergence.npz
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import BOX, PI_BOX, load_reference  # noqa: E402


def cases(k):
    heat, wave, schr = k.HeatPlaneDecay(1.0), k.WaveStanding(0.0), k.SchrodingerPhaseRotation()
    return {
        "heat": (BOX, k.StarCurve(1.0, c=0.2, lobes=5), heat, dict(
            equation="heat", bc_kind="dirichlet", g=heat.dirichlet, u0=heat.u0,
            lap_u0=heat.lap_u0, c=1.0)),
        "wave": (BOX, k.EllipseCurve(1.2, 0.8), wave, dict(
            equation="wave", bc_kind="dirichlet", g=wave.dirichlet, u0=wave.u0,
            lap_u0=wave.lap_u0, v0=wave.v0, lap_v0=wave.lap_v0, theta=0.25)),
        "schrodinger": (PI_BOX, k.StarCurve(1.5, c=0.2, lobes=3), schr, dict(
            equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
            lap_u0=schr.lap_u0, potential=schr.potential, w=1.0)),
    }


SIZES = {"heat": (64, 128, 256, 512), "wave": (64, 128, 256), "schrodinger": (64, 128, 256)}


def main():
    k = load_reference()
    out = {}
    for eq, (box, curve, sol, kw) in cases(k).items():
        for m in SIZES[eq]:
            tau = 0.25 * 64 / m
            t0 = time.time()
            geo = k.build_grid(box, m, curve)
            res = k.run(k.ProblemSpec(tau=tau, t_final=1.0, **kw), geo)
            e_inf, e_2 = k.compute_errors(res.state.u, lambda x, y: sol.u(x, y, 1.0), geo.grid,
                                          geo.classification)
            p = f"{eq}_{m}__"
            out[p + "e_inf"] = np.array(e_inf)
            out[p + "e_2"] = np.array(e_2)
            out[p + "iterations"] = np.array(res.iterations)
            print(eq, m, f"e_inf={e_inf:.6e} e_2={e_2:.6e} iters={sum(res.iterations)} "
                  f"({time.time() - t0:.1f}s)", flush=True)
    import scipy

    out["stamp"] = np.array(f"kfbi {k.__version__}; numpy {np.__version__}; scipy {scipy.__version__}")
    np.savez_compressed(os.path.join(HERE, "convergence.npz"), **out)


if __name__ == "__main__":
    main()
