"""Device-container helpers: torch CUDA tensors hold memory, the C ABI computes."""

from __future__ import annotations

import numpy as np


def torch():
    import torch as _t
    return _t


def is_device_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def to_device(x, dtype=None):
    """float64 (or dtype) contiguous CUDA tensor from numpy / list / tensor."""
    t = torch()
    dt = t.float64 if dtype is None else dtype
    if isinstance(x, t.Tensor):
        return x.to(device="cuda", dtype=dt).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64 if dt == t.float64 else None))
    return t.from_numpy(arr).to(device="cuda", dtype=dt, non_blocking=False).contiguous()


def empty(shape, dtype=None):
    t = torch()
    return t.empty(shape, dtype=t.float64 if dtype is None else dtype, device="cuda")


def zeros(shape, dtype=None):
    t = torch()
    return t.zeros(shape, dtype=t.float64 if dtype is None else dtype, device="cuda")


def host_f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))
