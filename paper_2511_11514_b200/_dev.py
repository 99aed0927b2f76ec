"""Device plumbing: torch owns memory and streams, the C ABI does the math.

Host arrays (numpy float64) are uploaded once per call, kernels run on the
current torch stream, and results come back as fresh numpy arrays, matching
the reference's ownership rules (inputs never mutated, outputs fresh).
"""

from __future__ import annotations

import contextlib
import ctypes
import os

import numpy as np
import torch

from . import _lib

# NVTX ranges around the planner's phases (FCB_NVTX=1), for ncu --nvtx
# filtering (e.g. --nvtx-include "flow/"); off by default (host cost per range)
NVTX = os.environ.get("FCB_NVTX", "0") != "0"


def nvtx_push(name: str) -> None:
    if NVTX:
        torch.cuda.nvtx.range_push(name)


def nvtx_pop() -> None:
    if NVTX:
        torch.cuda.nvtx.range_pop()


@contextlib.contextmanager
def nvtx(name: str):
    if not NVTX:
        yield
        return
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError(
            "flowcover-b200 runs on a CUDA device (sm_100a); no GPU is visible"
        )
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t: torch.Tensor | None) -> ctypes.c_void_p | None:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def f64(a, device: torch.device | None = None) -> torch.Tensor:
    """Upload a host array (or pass through a device tensor) as contiguous float64."""
    dev = device or require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.float64).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to(dev, non_blocking=False)


def empty(shape, dtype=torch.float64, device: torch.device | None = None) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device or require_cuda())


def zeros(shape, dtype=torch.float64, device: torch.device | None = None) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device or require_cuda())


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


class Workspace:
    """Grow-only scratch buffer per (device, tag).

    Calls are stream ordered, so consecutive calls on one stream may share a
    buffer; tags separate buffers that must stay alive together.
    """

    _pool: dict[tuple[int, str], torch.Tensor] = {}

    @classmethod
    def get(cls, nbytes: int, tag: str = "default") -> torch.Tensor:
        dev = require_cuda()
        key = (dev.index, tag)
        buf = cls._pool.get(key)
        if buf is None or buf.numel() < nbytes:
            size = max(int(nbytes * 1.25), 1 << 20)
            buf = torch.empty(size, dtype=torch.uint8, device=dev)
            cls._pool[key] = buf
        return buf

    @classmethod
    def clear(cls) -> None:
        cls._pool.clear()
