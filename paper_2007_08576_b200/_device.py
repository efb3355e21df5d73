"""Device-memory plumbing: numpy <-> torch CUDA tensors, raw pointers, the stream.

torch is used only to own device allocations and to name the current CUDA stream; every
computation on these buffers runs in libdeformtrack_b200.so.
"""

from __future__ import annotations

import numpy as np
import torch

_TORCH_DTYPES = {
    np.dtype(np.float64): torch.float64,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.bool_): torch.uint8,
}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "deformtrack_b200 needs a CUDA device (sm_100a); there is no CPU fallback"
        )
    return torch.device("cuda", torch.cuda.current_device())


def to_device(a, dtype=None) -> torch.Tensor:
    """Contiguous copy of a host array on the current CUDA device."""
    dev = require_cuda()
    arr = np.asarray(a)
    if dtype is not None:
        arr = arr.astype(dtype, copy=False)
    if arr.dtype == np.bool_:
        arr = arr.astype(np.uint8)
    arr = np.ascontiguousarray(arr)
    return torch.from_numpy(arr).to(dev, non_blocking=False)


def empty(shape, dtype=np.float64) -> torch.Tensor:
    dev = require_cuda()
    return torch.empty(tuple(int(s) for s in shape), dtype=_TORCH_DTYPES[np.dtype(dtype)], device=dev)


def zeros(shape, dtype=np.float64) -> torch.Tensor:
    dev = require_cuda()
    return torch.zeros(tuple(int(s) for s in shape), dtype=_TORCH_DTYPES[np.dtype(dtype)], device=dev)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() > 0 else None


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_host(t: torch.Tensor) -> np.ndarray:
    torch.cuda.current_stream().synchronize()
    return t.detach().cpu().numpy()


def sync() -> None:
    torch.cuda.current_stream().synchronize()
