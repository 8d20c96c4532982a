"""The uint8/uint16 code mapping (/root/reference/pkg/src/undertext/quantize.py).

``linear_to_codes`` (:36-46) runs on the device (``ut_linear_to_codes``) with
the reference arithmetic in fp64: floor(clip((v - lo) * (top / (hi - lo)),
0, top) + 0.5) -- ties away from zero, clip before rounding.
``round_half_away``, ``max_code`` and ``code_dtype`` are host utilities.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from . import device as dev


def round_half_away(values):
    """Nearest integer, ties away from zero (quantize.py:13-21)."""
    v = np.asarray(values, dtype=np.float64)
    return np.sign(v) * np.floor(np.abs(v) + 0.5)


def max_code(depth: int) -> int:
    if depth not in (8, 16):
        raise ValueError(f"unsupported bit depth {depth}; expected 8 or 16")
    return (1 << depth) - 1


def code_dtype(depth: int):
    return np.uint8 if depth == 8 else np.uint16


def _torch_code_dtype(depth: int):
    return torch.uint8 if depth == 8 else torch.uint16


def linear_to_codes(values, lo: float, hi: float, depth: int) -> np.ndarray:
    """Map [lo, hi] linearly onto [0, max_code(depth)] and quantize on the device."""
    if not np.isfinite(lo) or not np.isfinite(hi) or lo >= hi:
        raise ValueError(f"invalid rescale range [{lo}, {hi}]")
    max_code(depth)
    arr = np.asarray(values, dtype=np.float64)
    device = dev.require_cuda()
    v_d = dev.to_device(arr.reshape(-1), device)
    lohi = torch.tensor([float(lo), float(hi)], dtype=torch.float64, device=device)
    codes = torch.empty(arr.size, dtype=_torch_code_dtype(depth), device=device)
    _lib.check(_lib.lib().ut_linear_to_codes(v_d.data_ptr(), _lib.UT_F64, arr.size,
                                             lohi.data_ptr(), depth, codes.data_ptr(),
                                             dev.stream_handle()), "ut_linear_to_codes")
    return codes.cpu().numpy().reshape(arr.shape)
