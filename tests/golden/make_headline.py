"""Golden fixtures for the benched configurations (BASELINE.json metric and
configs[2]): short windows of the 4096² heat / wave / Schrödinger runs that
bench.py times, and C3 (Schrödinger, Strang, star3, 2048², τ = 1/128).

The full 4096² fields cannot be run by the oracle inside the GPU test budget
(minutes per step on the host), so this script runs the CPU oracle
(`oracle/kfbi_oracle.py`, itself pinned bit for bit to the unmodified
reference by tests/test_oracle.py) HERE and stores, per case:

  iterations   Richardson sweeps of every step (must be identical)
  u_sub        the final field on every 16th grid row / column
  u_irr        the final field at every irregular node (the correction sites)
  u_rows       two full grid rows (through the centre and through the
               boundary band) and two full columns
  density      the final density at the control points
  norm_inf     max |u| over the whole final field

The host tables come from the package's setup (bit-identical to the
reference's, tests/test_setup.py).  Re-run with

    python tests/golden/make_headline.py [case ...]      (~15 min on 8 cores)
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

STRIDE = 16


def cases():
    import bench
    import paper_2404_14864_b200 as k

    out = {}
    wl = bench.workload(4096)
    for eq in ("heat", "wave", "schrodinger"):
        box, curve, kw = wl[eq]
        kw = dict(kw, t_final=3 * kw["tau"])
        out[f"{eq}4096"] = (box, 4096, curve, kw)
    schr = k.SchrodingerPhaseRotation()
    pibox = (-np.pi, np.pi, -np.pi, np.pi)
    out["c3_schrodinger2048"] = (pibox, 2048, k.StarCurve(1.5, c=0.2, lobes=3), dict(
        equation="schrodinger", bc_kind="dirichlet", g=schr.dirichlet, u0=schr.u0,
        lap_u0=schr.lap_u0, potential=schr.potential, w=1.0, tau=1 / 128, t_final=2 / 128))
    return out


def sample_rows(m):
    """Full rows / columns stored besides the stride sample: the centre and
    one through the boundary band (a quarter of the box from the edge)."""
    return [m // 2, m // 4 + 3]


def record(ws, st, m):
    u = np.asarray(st.u)
    owners = np.asarray(ws.records.group_owners)
    rows = sample_rows(m)
    return {
        "iterations": np.asarray(st.iterations, np.int64),
        "u_sub": u[::STRIDE, ::STRIDE].copy(),
        "u_irr": u.reshape(-1)[owners].copy(),
        "irr_index": owners.astype(np.int64),
        "u_rows": np.stack([u[r] for r in rows]),
        "u_cols": np.stack([u[:, r] for r in rows]),
        "density": np.asarray(st.density).copy(),
        "norm_inf": np.array(np.max(np.abs(u))),
    }


def main(names):
    import paper_2404_14864_b200 as k
    from oracle import kfbi_oracle as O
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import oracle_spec

    allc = cases()
    for name in names or list(allc):
        box, m, curve, kw = allc[name]
        t0 = time.time()
        geo = k.build_grid(box, m, curve)
        ws = k.InterfaceWorkspace(geo)
        tabs = O.tables_from_workspace(ws)
        st = O.run(tabs, oracle_spec(kw))
        rec = record(ws, st, m)
        import scipy

        rec["stamp"] = np.array(f"oracle/kfbi_oracle.py, numpy {np.__version__}, scipy {scipy.__version__}")
        np.savez_compressed(os.path.join(HERE, f"headline_{name}.npz"), **rec)
        print(f"{name}: iterations {st.iterations} ({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
