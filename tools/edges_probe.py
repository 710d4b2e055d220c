"""Time the W-row edge values (kfbi_edge_values, interp "w") per geometry and
compare with a saved result: run once with KFBI_EDGES_SMEM=0 (per-warp form,
saves gpurun_out/edges_ref_*.npy) and once with the default (staged form).

    KFBI_EDGES_SMEM=0 python tools/edges_probe.py save ; python tools/edges_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_14864_b200 as k  # noqa: E402

save = len(sys.argv) > 1 and sys.argv[1] == "save"
tag = "per-warp" if os.environ.get("KFBI_EDGES_SMEM") == "0" else "staged"
out = "/tmp/edges_probe"
os.makedirs(out, exist_ok=True)
cases = []
for m in (1024, 4096):
    wl = bench.workload(m)
    for eq in ("heat", "wave", "schrodinger"):
        box, curve, kw = wl[eq]
        cases.append((f"{eq}{m}", box, m, curve, eq == "schrodinger"))
for name, box, m, curve, cplx in cases:
    ws = k.InterfaceWorkspace(k.build_grid(box, m, curve))
    plan = ws.plan
    plan.set_interp("w")
    n = ws.cps.m
    g = torch.Generator(device="cuda").manual_seed(1)
    dt = torch.complex128 if cplx else torch.float64
    jm = torch.randn((6, n), generator=g, device="cuda", dtype=dt)
    jv = torch.zeros(3 * 400000, device="cuda", dtype=dt)
    plan.edge_values(jm, jv)
    torch.cuda.synchronize()
    import time
    reps = 100
    t0 = time.perf_counter()
    for _ in range(reps):
        plan.edge_values(jm, jv)
    torch.cuda.synchronize()
    us = (time.perf_counter() - t0) / reps * 1e6
    res = jv.cpu().numpy()
    path = os.path.join(out, f"edges_ref_{name}.npy")
    msg = ""
    if save:
        np.save(path, res)
    elif os.path.exists(path):
        ref = np.load(path)
        sc = np.max(np.abs(ref)) or 1.0
        msg = f"max |diff| / max = {np.max(np.abs(res - ref)) / sc:.2e}"
    wbytes = 8 * n * (res.size // 3)
    print(f"[{tag}] {name:16s} n_ctl {n:5d} {us:8.1f} us  {msg}", flush=True)
