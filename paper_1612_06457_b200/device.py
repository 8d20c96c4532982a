"""Device plumbing: torch tensors as HBM buffers, current-stream handles,
cube descriptors and per-(device, stream) workspaces for the C ABI.

torch is used only for memory, streams and ``torch.distributed``; every
arithmetic step of the path runs in ``lib/libundertext_b200.so``.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib

TORCH_TO_UT = {
    torch.uint8: _lib.UT_U8,
    torch.uint16: _lib.UT_U16,
    torch.float16: _lib.UT_F16,
    torch.float32: _lib.UT_F32,
    torch.float64: _lib.UT_F64,
}
NUMPY_TO_TORCH = {
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.uint16): torch.uint16,
    np.dtype(np.float16): torch.float16,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def to_device(arr, device, dtype=None) -> torch.Tensor:
    """Host numpy (or tensor) -> contiguous device tensor."""
    if isinstance(arr, torch.Tensor):
        t = arr
    else:
        a = np.ascontiguousarray(arr)
        if not a.flags.writeable:
            a = a.copy()
        t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device, non_blocking=False).contiguous()


def cube_desc(planes: torch.Tensor, row0: int = 0) -> _lib.Cube:
    """ut_cube for a (B, rows, cols) tensor view (strides in elements)."""
    if planes.dim() != 3:
        raise ValueError("planes must be (bands, rows, cols)")
    if planes.dtype not in TORCH_TO_UT:
        raise TypeError(f"unsupported sample dtype {planes.dtype}")
    b, rows, cols = planes.shape
    sb, sr, sc = planes.stride()
    if sc != 1:
        raise ValueError("columns must be contiguous")
    return _lib.Cube(planes.data_ptr(), TORCH_TO_UT[planes.dtype], b, rows, cols, sb, sr, row0)


class _Workspaces(threading.local):
    def __init__(self):
        self.bufs = {}


_ws = _Workspaces()


def workspace(name: str, nbytes: int, device: torch.device) -> torch.Tensor:
    """A cached uint8 scratch buffer, one per (name, device, stream, thread)."""
    key = (name, device.index, stream_handle(device))
    buf = _ws.bufs.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws.bufs[key] = buf
    return buf
