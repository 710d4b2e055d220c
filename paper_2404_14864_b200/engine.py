"""Backend selection and per-kernel accounting (reference `engine.py`).

The reference routes every array sweep through ``Backend.dispatch(spec,
item_fn)`` with numpy closures executed on host threads (engine.py:84-169).
Here the sweeps are sm_100a kernels behind the C ABI, so the backend is a
device handle plus the same accounting surface: ``timings[name]`` (seconds,
from CUDA events around each launch) and ``calls[name]`` keyed by the nine
reference kernel names (engine.py:23-35).

Selectors: ``None`` / ``"cuda"`` -> current CUDA device, ``"cuda:<k>"`` ->
device k.  ``"serial"`` and ``"workers:<k>"`` name the reference's CPU
executors, which this package does not contain; they raise ConfigError (as
does ``"gpu"``, which the reference tests reject, test_engine.py:142-144).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

from .errors import ConfigError

KERNEL_NAMES = frozenset(
    {
        "classify-nodes",
        "edge-intersections",
        "jumps-and-corrections",
        "transform-rows",
        "transform-cols",
        "diagonal-scale",
        "extract-traces",
        "density-update",
        "rhs-update",
    }
)

DEFAULT_CHUNK_SIZE = 256


@dataclass(frozen=True)
class KernelSpec:
    """A named sweep over n_items (kept for API compatibility; the device
    grid shapes are chosen by the kernels themselves)."""

    name: str
    n_items: int
    chunk_size: int = DEFAULT_CHUNK_SIZE

    def __post_init__(self):
        if self.name not in KERNEL_NAMES:
            raise ConfigError(f"unknown kernel name '{self.name}'")
        if self.n_items < 0:
            raise ConfigError("kernel item count must be non-negative")
        if self.chunk_size < 1:
            raise ConfigError("kernel chunk size must be >= 1")

    @property
    def n_chunks(self):
        return (self.n_items + self.chunk_size - 1) // self.chunk_size

    def chunk_bounds(self):
        return [(k * self.chunk_size, min((k + 1) * self.chunk_size, self.n_items))
                for k in range(self.n_chunks)]


@dataclass
class Backend:
    timings: dict = field(default_factory=dict)
    calls: dict = field(default_factory=dict)

    @property
    def kind(self):  # pragma: no cover - interface
        raise NotImplementedError

    def reset_timings(self):
        self.timings.clear()
        self.calls.clear()

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


class CudaBackend(Backend):
    """One CUDA device.  Plans (device tables + scratch) register themselves
    so that ``collect()`` can fold their event timings into ``timings``."""

    def __init__(self, device=None, timing=True):
        super().__init__()
        import torch

        if not torch.cuda.is_available():
            raise ConfigError("the cuda backend needs a CUDA device (none visible)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.timing = bool(timing)
        self._plans = weakref.WeakSet()

    @property
    def kind(self):
        return f"cuda:{self.device}"

    @property
    def torch_device(self):
        import torch

        return torch.device("cuda", self.device)

    def stream_handle(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def register(self, plan):
        self._plans.add(plan)
        plan.set_timing(self.timing)

    def collect(self):
        """Fold device timings of every registered plan into timings/calls."""
        tot_ms, tot_calls = {}, {}
        for plan in list(self._plans):
            ms, calls = plan.kernel_times()
            for k, v in ms.items():
                tot_ms[k] = tot_ms.get(k, 0.0) + v
            for k, v in calls.items():
                tot_calls[k] = tot_calls.get(k, 0) + v
        self.timings.clear()
        self.calls.clear()
        for k in tot_calls:
            if tot_calls[k]:
                self.timings[k] = tot_ms[k] / 1e3
                self.calls[k] = tot_calls[k]
        return self.timings

    def reset_timings(self):
        for plan in list(self._plans):
            plan.reset_kernel_times()
        super().reset_timings()

    def dispatch(self, spec, item_fn):
        raise ConfigError(
            "the cuda backend runs the solver's device kernels; it does not execute "
            "host closures (use the reference package for CPU dispatch)")


_DEFAULT = {}


def make_backend(selector=None):
    """'cuda' | 'cuda:<device>' | an existing Backend (passed through)."""
    if isinstance(selector, Backend):
        return selector
    if selector is None or selector == "cuda":
        key = None
    elif isinstance(selector, str) and selector.startswith("cuda:"):
        try:
            key = int(selector.split(":", 1)[1])
        except ValueError:
            raise ConfigError(f"bad device index in backend selector '{selector}'")
    else:
        raise ConfigError(
            f"unknown backend '{selector}' (expected 'cuda' or 'cuda:<device>'; the CPU "
            "executors 'serial' / 'workers:<k>' belong to the reference package)")
    return CudaBackend(key)


def default_backend():
    """Process-wide default CudaBackend for calls made without a backend."""
    import torch

    dev = torch.cuda.current_device() if torch.cuda.is_available() else None
    if dev not in _DEFAULT:
        _DEFAULT[dev] = CudaBackend(dev)
    return _DEFAULT[dev]
