"""Score planes and the full-range stretch.

Mirrors ``ScorePlane`` and ``rescale_full`` of
/root/reference/pkg/src/undertext/rendering.py (:39-60, :119-130).  A host
ScorePlane (float64 numpy, finite-checked) is rescaled on the device by
``ut_plane_minmax`` + ``ut_linear_to_codes``; a ``DeviceScorePlane`` (one fp32
plane of the projector's output, with the min/max the projector already
reduced) is rescaled by ``ut_stretch`` without another reduction pass.
The other rescale modes, composites and codecs are outside the hot path.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import DataError, UndertextWarning
from .quantize import _torch_code_dtype, code_dtype, max_code


@dataclass(frozen=True)
class ScorePlane:
    """One projected plane of floating-point scores, shape (height, width)."""

    values: np.ndarray

    def __post_init__(self):
        values = np.asarray(self.values, dtype=np.float64)
        if values.ndim != 2:
            raise DataError(f"score plane must be 2-D, got shape {values.shape}")
        if not np.isfinite(values).all():
            raise DataError("score plane contains NaN or Inf")
        values.setflags(write=False)
        object.__setattr__(self, "values", values)

    @property
    def height(self) -> int:
        return int(self.values.shape[0])

    @property
    def width(self) -> int:
        return int(self.values.shape[1])


@dataclass(frozen=True)
class DeviceScorePlane:
    """Plane ``index`` of a projector output resident in HBM.

    ``scores`` is the (K, H, W) float32 tensor, ``minmax`` the (2K,) record
    [-min_0.., max_0..] written by ``ut_project_minmax`` (all-reduced across row
    shards when sharded).
    """

    scores: torch.Tensor = field(repr=False)
    minmax: torch.Tensor = field(repr=False)
    index: int = 0

    @property
    def values(self) -> torch.Tensor:
        return self.scores[self.index]

    @property
    def height(self) -> int:
        return int(self.scores.shape[1])

    @property
    def width(self) -> int:
        return int(self.scores.shape[2])

    def range(self) -> tuple[float, float]:
        k = self.scores.shape[0]
        mm = self.minmax.cpu().numpy()
        return -float(mm[self.index]), float(mm[k + self.index])

    def to_host(self) -> ScorePlane:
        return ScorePlane(self.values.double().cpu().numpy())


def _zeros_warning(reason: str) -> None:
    warnings.warn(f"{reason}; rendering all zeros", UndertextWarning, stacklevel=3)


def stretch_planes(scores: torch.Tensor, minmax: torch.Tensor, depth: int = 8,
                   first: int = 0, count: int | None = None, out: torch.Tensor | None = None):
    """K5 over planes [first, first+count) of a (K, H, W) projector output."""
    max_code(depth)
    k_total = scores.shape[0]
    count = k_total - first if count is None else count
    npix = scores.shape[1] * scores.shape[2]
    if out is None:
        out = torch.empty((count, scores.shape[1], scores.shape[2]),
                          dtype=_torch_code_dtype(depth), device=scores.device)
    _lib.check(_lib.lib().ut_stretch(scores[first].data_ptr(), minmax[first:].data_ptr(), count,
                                     k_total, npix, depth, out.data_ptr(), dev.stream_handle()),
               "ut_stretch")
    return out


def rescale_full(plane, depth: int = 8):
    """Map the plane's min to 0 and its max to the top code (rendering.py:124-130).

    Host ScorePlane (or array) -> numpy codes, warning + zeros on a constant
    plane; DeviceScorePlane -> device codes (no host sync).
    """
    if isinstance(plane, DeviceScorePlane):
        with torch.cuda.device(plane.scores.device):
            return stretch_planes(plane.scores, plane.minmax, depth, plane.index, 1)[0]
    if not isinstance(plane, ScorePlane):
        plane = ScorePlane(plane)
    max_code(depth)
    device = dev.require_cuda()
    v = plane.values
    v_d = dev.to_device(v.reshape(-1), device)
    ws = dev.workspace("plane_minmax", _lib.lib().ut_plane_minmax_ws(), device)
    lohi = torch.empty(2, dtype=torch.float64, device=device)
    flag = torch.empty(1, dtype=torch.int32, device=device)
    codes = torch.empty(v.size, dtype=_torch_code_dtype(depth), device=device)
    L = _lib.lib()
    s = dev.stream_handle()
    _lib.check(L.ut_plane_minmax(v_d.data_ptr(), _lib.UT_F64, v.size, lohi.data_ptr(),
                                 flag.data_ptr(), ws.data_ptr(), ws.numel(), s), "ut_plane_minmax")
    _lib.check(L.ut_linear_to_codes(v_d.data_ptr(), _lib.UT_F64, v.size, lohi.data_ptr(), depth,
                                    codes.data_ptr(), s), "ut_linear_to_codes")
    host = codes.cpu().numpy().reshape(v.shape)
    lo, hi = lohi.cpu().numpy()
    if lo == hi:
        _zeros_warning("constant score plane")
        return np.zeros(v.shape, dtype=code_dtype(depth))
    return host
