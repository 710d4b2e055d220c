"""Host <-> device plumbing (torch is the allocator and stream provider)."""

from __future__ import annotations

import numpy as np


def torch_dtype(np_dtype):
    import torch

    return torch.complex128 if np.issubdtype(np.dtype(np_dtype), np.complexfloating) else torch.float64


def to_device(a, np_dtype, backend):
    """Contiguous flat device copy of an array-like (torch tensors are moved /
    cast without a host round trip)."""
    import torch

    td = torch_dtype(np_dtype)
    if isinstance(a, torch.Tensor):
        return a.to(device=backend.torch_device, dtype=td).contiguous().reshape(-1)
    arr = np.ascontiguousarray(np.asarray(a), dtype=np_dtype).reshape(-1)
    return torch.from_numpy(arr).to(backend.torch_device)


def to_host(t, shape=None):
    out = t.detach().cpu().numpy()
    return out.reshape(shape) if shape is not None else out


def mask_device(mask, backend):
    import torch

    arr = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8)).reshape(-1)
    return torch.from_numpy(arr).to(backend.torch_device)
