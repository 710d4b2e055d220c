"""Error norms and field dumps of a run (reference report.py:37-62).

Only the two numeric helpers of the reference's report module are mirrored
(the CLI, TOML configs, manifests and figures are the reference's host
harness, out of scope — DESIGN.md §8).  `compute_errors` accepts numpy arrays
(the reference's arithmetic, bit-identical) or CUDA tensors (the norms are
reduced on the device, only two scalars come back).  `dump_field` writes the
reference's CSV format, text-identical, without its per-line Python loop.
"""

from __future__ import annotations

import numpy as np


def compute_errors(u_numeric, u_exact, grid, classification):
    """(‖e‖∞, ‖e‖₂) over interior nodes; complex errors use the modulus
    (report.py:37-44)."""
    mask = classification.interior
    exact = u_exact(grid.X[mask], grid.Y[mask])
    if hasattr(u_numeric, "is_cuda") and u_numeric.is_cuda:
        import torch

        dev = u_numeric.device
        idx = torch.from_numpy(np.flatnonzero(mask.ravel())).to(dev)
        diff = u_numeric.reshape(-1)[idx] - torch.as_tensor(np.asarray(exact), device=dev)
        a = diff.abs()
        if a.numel() == 0:
            return 0.0, 0.0
        return float(a.max()), float(torch.sqrt(torch.sum(a * a)) / grid.m)
    diff = np.asarray(u_numeric)[mask] - exact
    abs_diff = np.abs(diff)
    e_inf = float(abs_diff.max()) if abs_diff.size else 0.0
    e_2 = float(np.sqrt(np.sum(abs_diff**2)) / grid.m)
    return e_inf, e_2


def dump_field(u, grid, classification, path, m=None, t=None, equation=None):
    """CSV dump of the interior nodes: x, y, value[, imag] (report.py:47-62),
    the same text as the reference's line-by-line writer."""
    if hasattr(u, "cpu"):
        u = u.cpu().numpy().reshape(grid.m + 1, grid.m + 1)
    mask = classification.interior
    xs, ys, vals = grid.X[mask], grid.Y[mask], np.asarray(u)[mask]
    is_complex = np.iscomplexobj(vals)
    meta = f"# M={grid.m if m is None else m} t={t} equation={equation}\n"
    header = "x,y,value,imag\n" if is_complex else "x,y,value\n"
    cols = [xs, ys, vals.real, vals.imag] if is_complex else [xs, ys, vals]
    fmt = ",".join(["%.17g"] * len(cols))
    with open(path, "w") as fh:
        fh.write(meta)
        fh.write(header)
        if xs.size:
            np.savetxt(fh, np.column_stack(cols), fmt=fmt, delimiter=",")
    return path
