"""Device plumbing: torch supplies device memory and the CUDA stream; all
compute runs in libctap.so.  There is no CPU fallback."""

from __future__ import annotations

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1309_2451_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def to_device_c128(a) -> torch.Tensor:
    """Contiguous complex128 CUDA tensor (uploads numpy, keeps CUDA tensors)."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=torch.complex128)
    else:
        arr = np.ascontiguousarray(a, dtype=np.complex128)
        t = torch.from_numpy(arr).to(dev)
    return t.contiguous()


def to_device_f64(a) -> torch.Tensor:
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=torch.float64)
    else:
        arr = np.ascontiguousarray(a, dtype=np.float64)
        t = torch.from_numpy(arr).to(dev)
    return t.contiguous()


def pinned_like(shape, dtype=torch.complex128) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def to_host(t: torch.Tensor) -> np.ndarray:
    """D2H into pinned memory; returns a writable numpy view."""
    host = pinned_like(tuple(t.shape), t.dtype)
    host.copy_(t)
    return host.numpy()
