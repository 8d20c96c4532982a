"""Score planes and the full-range stretch.

Mirrors ``ScorePlane`` and ``rescale_full`` of
/root/reference/pkg/src/undertext/rendering.py (:39-60, :119-130).  A host
ScorePlane (float64 numpy, finite-checked) is rescaled on the device by
``ut_plane_minmax`` + ``ut_linear_to_codes``; a ``DeviceScorePlane`` (one fp32
plane of the projector's output, with the min/max the projector already
reduced) is rescaled by ``ut_stretch`` without another reduction pass.
The training-range and percentile modes (:133-179) use the same
``ut_linear_to_codes``; the percentile window comes from an exact radix select
on the device (``ut_plane_select``).  ``compose_rgb`` (:206-225) interleaves
three code planes on the device (``ut_compose_rgb``); files are written by
``image_io.save_image`` (device PNG / TIFF encoders).
"""

from __future__ import annotations

import ctypes as C
import math
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import DataError, UndertextWarning
from .quantize import _torch_code_dtype, code_dtype, max_code


MODE_FULL_RANGE = "full"            # rendering.py:31-36
MODE_TRAINING_RANGE = "training"
MODE_PERCENTILE = "percentile"
RESCALE_MODES = (MODE_FULL_RANGE, MODE_TRAINING_RANGE, MODE_PERCENTILE)
PERCENTILE_CHOICES = (0.01, 0.1, 1.0, 5.0)


@dataclass(frozen=True)
class RenderSpec:
    """How to quantize score planes: mode, optional percentile, bit depth
    (rendering.py:63-93)."""

    mode: str = MODE_FULL_RANGE
    percentile_p: float | None = None
    out_depth: int = 8
    one_tail: bool = False

    def __post_init__(self):
        if self.mode not in RESCALE_MODES:
            raise DataError(f"unknown rescale mode {self.mode!r}")
        if self.out_depth not in (8, 16):
            raise DataError(f"bit depth must be 8 or 16, got {self.out_depth}")
        if self.mode == MODE_PERCENTILE:
            if self.percentile_p not in PERCENTILE_CHOICES:
                raise DataError(f"percentile must be one of {PERCENTILE_CHOICES}, "
                                f"got {self.percentile_p!r}")
        elif self.percentile_p is not None:
            raise DataError(f"percentile given but mode is {self.mode!r}")

    def suffix(self) -> str:
        if self.mode == MODE_PERCENTILE:
            p = self.percentile_p
            text = str(int(p)) if float(p).is_integer() else str(p).replace(".", "_")
            return f"_p{text}"
        return f"_{self.mode}"


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


def host_plane(plane) -> ScorePlane:
    """A host ScorePlane from ours, the reference's ScorePlane (rendering.py:39-60;
    duck-typed on ``values``) or a bare 2-D array."""
    if isinstance(plane, ScorePlane):
        return plane
    values = getattr(plane, "values", plane)
    if isinstance(values, torch.Tensor):
        values = values.double().cpu().numpy()
    return ScorePlane(values)


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
    plane = host_plane(plane)
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


# ---------------------------------------------------------------- other modes

def _plane_on_device(plane):
    """(values tensor on the device, UT dtype, shape, is_host) of a plane."""
    if isinstance(plane, DeviceScorePlane):
        v = plane.values
        if not v.is_contiguous():
            v = v.contiguous()
        return v, dev.TORCH_TO_UT[v.dtype], tuple(v.shape), False
    plane = host_plane(plane)
    device = dev.require_cuda()
    v = dev.to_device(plane.values, device)
    return v, _lib.UT_F64, plane.values.shape, True


def _codes(v, dtype, shape, lohi, depth, host):
    codes = torch.empty(int(np.prod(shape)), dtype=_torch_code_dtype(depth), device=v.device)
    _lib.check(_lib.lib().ut_linear_to_codes(v.data_ptr(), dtype, codes.numel(), lohi.data_ptr(),
                                             depth, codes.data_ptr(), dev.stream_handle()),
               "ut_linear_to_codes")
    codes = codes.view(shape)
    return codes.cpu().numpy() if host else codes


def _zeros(shape, depth, host, device):
    if host:
        return np.zeros(shape, dtype=code_dtype(depth))
    return torch.zeros(shape, dtype=_torch_code_dtype(depth), device=device)


def rescale_training_range(plane, model, k: int, depth: int = 8):
    """Map the training-score span of component k onto the code range
    (rendering.py:133-152); values outside clamp to 0 / the top code."""
    if model.training_scores is None:
        raise DataError("model has no training scores (unsupervised fit); use full-range")
    if not (0 <= k < model.training_scores.shape[0]):
        raise DataError(f"component {k} out of range")
    max_code(depth)
    row = model.training_scores[k]
    lo, hi = float(row.min()), float(row.max())
    v, dtype, shape, host = _plane_on_device(plane)
    if lo == hi:
        _zeros_warning(f"training scores constant for component {k}")
        return _zeros(shape, depth, host, v.device)
    lohi = torch.tensor([lo, hi], dtype=torch.float64).to(v.device)
    return _codes(v, dtype, shape, lohi, depth, host)


def nearest_rank_percentile(sorted_values, p: float) -> float:
    """Element ceil(p/100 n) (1-based) of an ascending sample
    (rendering.py:146-152; host helper, as in the reference)."""
    n = len(sorted_values)
    rank = max(1, math.ceil(p / 100.0 * n))
    return float(sorted_values[rank - 1])


def rescale_percentile(plane, p: float, depth: int = 8, one_tail: bool = False):
    """Clip the darkest and brightest p percent, then map linearly
    (rendering.py:155-179).  lo / hi are the nearest-rank p-th and (100-p)-th
    percentiles, found on the device by an exact radix select."""
    if p not in PERCENTILE_CHOICES:
        raise DataError(f"percentile must be one of {PERCENTILE_CHOICES}, got {p!r}")
    max_code(depth)
    v, dtype, shape, host = _plane_on_device(plane)
    n = int(np.prod(shape))
    r_lo = 1 if one_tail else max(1, math.ceil(p / 100.0 * n))
    r_hi = max(1, math.ceil((100.0 - p) / 100.0 * n))
    ranks = (C.c_int64 * 2)(r_lo, r_hi)
    lohi = torch.empty(2, dtype=torch.float64, device=v.device)
    L = _lib.lib()
    ws = dev.workspace("plane_select", L.ut_plane_select_ws(), v.device)
    _lib.check(L.ut_plane_select(v.data_ptr(), dtype, n, ranks, lohi.data_ptr(), ws.data_ptr(),
                                 ws.numel(), dev.stream_handle()), "ut_plane_select")
    lo, hi = lohi.cpu().numpy()
    if lo == hi:
        _zeros_warning(f"percentile window empty at p={p}")
        return _zeros(shape, depth, host, v.device)
    return _codes(v, dtype, shape, lohi, depth, host)


def rescale(plane, spec: RenderSpec, model=None, k: int | None = None):
    """Apply the rescale mode named by ``spec`` to one plane (rendering.py:182-195)."""
    if spec.mode == MODE_FULL_RANGE:
        return rescale_full(plane, spec.out_depth)
    if spec.mode == MODE_TRAINING_RANGE:
        if model is None or k is None:
            raise DataError("training-range rescale needs the fitted model and plane index")
        return rescale_training_range(plane, model, k, spec.out_depth)
    return rescale_percentile(plane, spec.percentile_p, spec.out_depth, spec.one_tail)


# ---------------------------------------------------------------- composites

@dataclass(frozen=True)
class CompositeRecipe:
    """Which rendered planes land in R, G, B, with an optional channel swap
    (a pair of channel indices, 0=R 1=G 2=B, exchanged after assignment)
    (rendering.py:96-116)."""

    red: int
    green: int
    blue: int
    swap: tuple[int, int] | None = None

    def __post_init__(self):
        if self.swap is not None:
            a, b = self.swap
            if not {a, b} <= {0, 1, 2} or a == b:
                raise DataError(f"swap must name two distinct channels, got {self.swap}")

    def suffix(self) -> str:
        text = f"_R{self.red}G{self.green}B{self.blue}"
        if self.swap is not None:
            text += f"_swap{self.swap[0]}{self.swap[1]}"
        return text


def _code_depth(img, name: str = "image") -> int:
    dt = img.dtype
    if dt in (np.uint8, torch.uint8):
        return 8
    if dt in (np.uint16, torch.uint16):
        return 16
    raise DataError(f"{name} must be uint8 or uint16, got {dt}")


def compose_rgb(planes: list, recipe: CompositeRecipe):
    """Stack three rendered planes into an RGB image per the recipe
    (rendering.py:206-225).  Recipe indices select from ``planes`` (repeats
    allowed); the optional swap exchanges two finished channels afterwards.
    Device planes -> device (H, W, 3) tensor; host arrays -> numpy."""
    for idx in (recipe.red, recipe.green, recipe.blue):
        if not (0 <= idx < len(planes)):
            raise DataError(f"recipe index {idx} outside plane set of {len(planes)}")
    channels = [planes[recipe.red], planes[recipe.green], planes[recipe.blue]]
    depths = {_code_depth(c) for c in channels}
    shapes = {tuple(c.shape) for c in channels}
    if len(shapes) != 1 or len(depths) != 1:
        raise DataError("composite channels must share dimensions and bit depth")
    if any(len(c.shape) != 2 for c in channels):
        raise DataError("composite channels must be grayscale")
    if recipe.swap is not None:
        a, b = recipe.swap
        channels[a], channels[b] = channels[b], channels[a]
    host = not isinstance(channels[0], torch.Tensor)
    device = dev.require_cuda() if host else channels[0].device
    chans = [dev.to_device(c, device) if (host or not c.is_cuda or not c.is_contiguous())
             else c for c in channels]
    h, w = chans[0].shape
    depth = depths.pop()
    out = torch.empty((h, w, 3), dtype=_torch_code_dtype(depth), device=device)
    with torch.cuda.device(device):
        _lib.check(_lib.lib().ut_compose_rgb(chans[0].data_ptr(), chans[1].data_ptr(),
                                             chans[2].data_ptr(), depth, h * w, out.data_ptr(),
                                             dev.stream_handle()), "ut_compose_rgb")
    return out.cpu().numpy() if host else out
