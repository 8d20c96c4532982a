"""Spectral cubes on the host and in HBM.

``SpectralStack`` mirrors the reference container
(/root/reference/pkg/src/undertext/stack.py:22-98): B co-registered planes,
(B, H, W) band-sequential, read-only, with per-band metadata.  ``DeviceStack``
is the same cube resident in HBM (a torch tensor), optionally a row shard
``[row0, row0 + rows)`` of a taller image; it is what the fast path consumes.
A host stack is staged to HBM once and the device copy is cached for the
lifetime of its (immutable) plane array, so the reference's usual call
sequence -- assemble_matrix, fit, project_stack on one stack -- pays one H2D.
"""

from __future__ import annotations

import ctypes as C
import threading
import warnings
import weakref
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import device as dev
from .errors import DataError


@dataclass(frozen=True)
class BandMeta:
    """Acquisition metadata for one band (stack.py:22-36)."""

    band_id: int
    wavelength_nm: float
    illumination: str
    filter: str | None = None

    def __post_init__(self):
        if self.wavelength_nm <= 0:
            raise DataError(f"band {self.band_id}: wavelength must be positive, "
                            f"got {self.wavelength_nm}")


def default_bands(n: int) -> tuple[BandMeta, ...]:
    return tuple(BandMeta(i, 400.0 + i, "synthetic") for i in range(n))


@dataclass(frozen=True)
class SpectralStack:
    """Host cube, validated like the reference (stack.py:53-71)."""

    bands: tuple[BandMeta, ...]
    planes: np.ndarray = field(repr=False)
    bit_depth: int
    normalized: bool = False

    def __post_init__(self):
        if self.bit_depth not in (8, 16):
            raise DataError(f"bit depth must be 8 or 16, got {self.bit_depth}")
        if self.planes.ndim != 3 or self.planes.shape[0] != len(self.bands):
            raise DataError(f"planes shape {self.planes.shape} does not match "
                            f"{len(self.bands)} bands")
        if len(self.bands) < 1:
            raise DataError("a stack needs at least one band")
        ids = [b.band_id for b in self.bands]
        if len(set(ids)) != len(ids):
            raise DataError(f"duplicate band ids in stack: {ids}")
        if self.planes.size and float(self.planes.max()) >= (1 << self.bit_depth):
            raise DataError(f"sample value {self.planes.max()} exceeds "
                            f"{self.bit_depth}-bit range")
        self.planes.setflags(write=False)

    @property
    def band_count(self) -> int:
        return len(self.bands)

    @property
    def width(self) -> int:
        return int(self.planes.shape[2])

    @property
    def height(self) -> int:
        return int(self.planes.shape[1])

    def band_by_id(self, band_id: int) -> np.ndarray:
        """Plane for a band id; DataError for unknown ids (stack.py:84-89)."""
        return _band_by_id(self, band_id)

    def pixel_vector(self, x: int, y: int) -> np.ndarray:
        """The B samples at (x, y) in band order, as float64 (stack.py:91-97)."""
        _check_pixel(self, x, y)
        return self.planes[:, y, x].astype(np.float64)


def _band_by_id(stack, band_id: int):
    for i, meta in enumerate(stack.bands):
        if meta.band_id == band_id:
            return stack.planes[i]
    raise DataError(f"unknown band id {band_id}")


def _check_pixel(stack, x: int, y: int) -> None:
    if not (0 <= x < stack.width and 0 <= y < stack.height):
        raise DataError(f"pixel ({x}, {y}) outside {stack.width}x{stack.height} stack")


@dataclass(frozen=True)
class DeviceStack:
    """A cube (or row shard) resident in HBM.

    ``planes`` is a (B, rows, W) CUDA tensor of uint8/uint16/float16/float32/
    float64 samples; ``row0`` is the global index of local row 0 and
    ``full_height`` the global image height (== rows when unsharded).
    """

    bands: tuple[BandMeta, ...]
    planes: torch.Tensor = field(repr=False)
    bit_depth: int = 8
    normalized: bool = True
    row0: int = 0
    full_height: int | None = None

    def __post_init__(self):
        if not self.planes.is_cuda:
            raise DataError("DeviceStack planes must be a CUDA tensor")
        if self.planes.dim() != 3 or self.planes.shape[0] != len(self.bands):
            raise DataError(f"planes shape {tuple(self.planes.shape)} does not match "
                            f"{len(self.bands)} bands")
        if self.planes.dtype not in dev.TORCH_TO_UT:
            raise DataError(f"unsupported sample dtype {self.planes.dtype}")
        if self.full_height is None:
            object.__setattr__(self, "full_height", int(self.planes.shape[1]) + self.row0)

    @property
    def band_count(self) -> int:
        return len(self.bands)

    @property
    def width(self) -> int:
        return int(self.planes.shape[2])

    @property
    def height(self) -> int:
        """Local rows (the reference's stack.height for an unsharded stack)."""
        return int(self.planes.shape[1])

    @property
    def pixels(self) -> int:
        return self.height * self.width

    def cube(self):
        return dev.cube_desc(self.planes, self.row0)

    def band_by_id(self, band_id: int) -> torch.Tensor:
        """The (rows, W) device plane of a band id (stack.py:84-89)."""
        return _band_by_id(self, band_id)

    def pixel_vector(self, x: int, y: int) -> np.ndarray:
        """Host float64 samples at (x, local row y) in band order (stack.py:91-97)."""
        _check_pixel(self, x, y)
        return self.planes[:, y, x].double().cpu().numpy()

    @classmethod
    def from_host(cls, stack: SpectralStack, device=None) -> "DeviceStack":
        device = device or dev.require_cuda()
        with warnings.catch_warnings():  # read-only planes: only ever copied to the device
            warnings.simplefilter("ignore", UserWarning)
            t = torch.from_numpy(np.ascontiguousarray(stack.planes))
        return cls(stack.bands, t.to(device), stack.bit_depth, stack.normalized)


_cache_lock = threading.Lock()
_device_copies: dict[int, tuple[weakref.ref, DeviceStack]] = {}


def is_host_stack(stack) -> bool:
    """A host cube in the reference's shape: ours or the reference's own
    SpectralStack (stack.py:39-71) -- duck-typed on its fields."""
    return isinstance(stack, SpectralStack) or (
        isinstance(getattr(stack, "planes", None), np.ndarray) and hasattr(stack, "bands")
        and hasattr(stack, "bit_depth") and hasattr(stack, "normalized"))


def on_device(stack) -> DeviceStack:
    """The HBM copy of a stack (identity for a DeviceStack; cached H2D otherwise)."""
    if isinstance(stack, DeviceStack):
        return stack
    if not is_host_stack(stack):
        raise DataError(f"expected a SpectralStack or DeviceStack, got {type(stack).__name__}")
    device = dev.require_cuda()
    key = id(stack.planes)
    with _cache_lock:
        hit = _device_copies.get(key)
        if hit is not None and hit[0]() is stack.planes and \
                hit[1].planes.device == device and hit[1].normalized == stack.normalized:
            return hit[1]
    ds = DeviceStack.from_host(stack, device)
    _register_device_copy(stack, ds)
    return ds


def _register_device_copy(stack: SpectralStack, ds: DeviceStack) -> None:
    """Remember ``ds`` as the HBM copy of the host stack's (immutable) planes."""
    key = id(stack.planes)
    with _cache_lock:
        ref = weakref.ref(stack.planes, lambda _r, k=key: _device_copies.pop(k, None)) \
            if _weakrefable(stack.planes) else (lambda: None)
        _device_copies[key] = (ref, ds)


def _weakrefable(a) -> bool:
    try:
        weakref.ref(a)
        return True
    except TypeError:
        return False


def normalize_stack(stack, scope: str = "per-band"):
    """Min-max map samples onto [0, 255], rounded ties away (stack.py:180-213).

    ``scope="per-band"`` maps each band by its own min/max, ``"global"`` by the
    cube's.  A constant band (stack) maps to zeros with a warning; an already
    normalized stack is refused.  Host SpectralStack -> host SpectralStack
    (uint8, normalized); DeviceStack -> DeviceStack in HBM.  Both passes run on
    the GPU (``ut_normalize_stack``); codes are bit-identical to numpy's.
    """
    import warnings

    from . import _lib
    from .errors import UndertextWarning

    if not (isinstance(stack, DeviceStack) or is_host_stack(stack)):
        raise DataError(f"expected a SpectralStack or DeviceStack, got {type(stack).__name__}")
    if stack.normalized:
        raise DataError("stack is already normalized")
    if scope not in ("per-band", "global"):
        raise DataError(f"unknown normalization scope {scope!r}")
    host = not isinstance(stack, DeviceStack)
    ds = DeviceStack.from_host(stack) if host else stack
    device = ds.planes.device
    b = ds.band_count
    with torch.cuda.device(device):
        out = torch.empty((b, ds.height, ds.width), dtype=torch.uint8, device=device)
        lohi = torch.empty(2 * b, dtype=torch.float64, device=device)
        const = torch.empty(b, dtype=torch.int32, device=device)
        L = _lib.lib()
        ws = dev.workspace("normalize", L.ut_normalize_ws(), device)
        cube = ds.cube()
        _lib.check(L.ut_normalize_stack(C.byref(cube), 0 if scope == "per-band" else 1,
                                        out.data_ptr(), lohi.data_ptr(), const.data_ptr(),
                                        ws.data_ptr(), ws.numel(), dev.stream_handle()),
                   "ut_normalize_stack")
        flags = const.cpu().numpy()
        lo = lohi.cpu().numpy()[0::2]
    for i in np.flatnonzero(flags):
        warnings.warn(f"band {ds.bands[i].band_id} is constant (value {int(lo[i])}); "
                      f"normalized to all zeros", UndertextWarning, stacklevel=2)
    if host:
        return SpectralStack(stack.bands, out.cpu().numpy(), 8, normalized=True)
    return DeviceStack(ds.bands, out, 8, True, ds.row0, ds.full_height)


# ------------------------------------------------------------------ load_stack

def _parse_manifest_line(line: str, lineno: int, base: Path):
    """``path,wavelength_nm,illumination[,filter]`` (stack.py:101-116)."""
    parts = [p.strip() for p in line.split(",")]
    if len(parts) not in (3, 4):
        raise DataError(f"manifest line {lineno}: expected "
                        f"'path,wavelength_nm,illumination[,filter]', got {line!r}")
    path = base / parts[0]
    try:
        wavelength = float(parts[1])
    except ValueError:
        raise DataError(f"manifest line {lineno}: bad wavelength {parts[1]!r}") from None
    filt = parts[3] if len(parts) == 4 else None
    return path, wavelength, parts[2], filt


def load_device_stack(manifest) -> DeviceStack:
    """The bands named by a manifest, decoded into one HBM cube (TIFF and PNG
    bands decode on the device; see image_io.read_image_device)."""
    from .image_io import _Unsupported, decode_batch, read_image_device

    manifest = Path(manifest)
    if not manifest.is_file():
        raise DataError(f"manifest not found: {manifest}")
    entries = []
    for lineno, raw in enumerate(manifest.read_text(encoding="utf-8").splitlines(), 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        entries.append(_parse_manifest_line(line, lineno, manifest.parent))
    if not entries:
        raise DataError(f"manifest {manifest} lists no bands")
    for band_id, (path, _w, _i, _f) in enumerate(entries):
        if not path.is_file():
            raise DataError(f"band {band_id}: image file not found: {path}")
    # all bands in one batched device decode when every file is a TIFF / PNG the
    # device decoders parse
    imgs = None
    try:
        datas = [path.read_bytes() for path, *_ in entries]
        imgs = decode_batch(datas)
    except (_Unsupported, DataError, OSError):
        imgs = None
    metas, planes = [], []
    shape, depth = None, None
    for band_id, (path, wavelength, illum, filt) in enumerate(entries):
        if imgs is not None:
            img = imgs[band_id]
        else:
            try:
                img, _ = read_image_device(path)
            except DataError:
                raise DataError(f"band {band_id}: could not decode {path}") from None
        if img.dim() != 2:
            raise DataError(f"band {band_id}: {path} has {img.shape[2]} channels; "
                            f"stacks are built from single-channel images")
        if img.dtype == torch.uint8:
            band_depth = 8
        elif img.dtype == torch.uint16:
            band_depth = 16
        else:
            raise DataError(f"band {band_id}: {path} has unsupported sample type {img.dtype}")
        if shape is None:
            shape, depth = tuple(img.shape), band_depth
        else:
            if tuple(img.shape) != shape:
                raise DataError(f"band {band_id}: size {img.shape[1]}x{img.shape[0]} does not "
                                f"match band 0 ({shape[1]}x{shape[0]})")
            if band_depth != depth:
                raise DataError(f"band {band_id}: {band_depth}-bit plane in a {depth}-bit stack")
        metas.append(BandMeta(band_id, wavelength, illum, filt))
        planes.append(img)
    return DeviceStack(tuple(metas), torch.stack(planes), depth, False)


def load_stack(manifest) -> SpectralStack:
    """Load a stack from a manifest file (stack.py:119-177): one band per line,
    ``relative/path.tif,wavelength_nm,illumination[,filter]``, ``#`` comments,
    paths relative to the manifest, band ids in manifest order; every band a
    single-channel image of one shared size and bit depth.  The bands are
    decoded on the device; the returned host stack keeps that HBM copy
    registered, so the fit / projection that follows pays no upload."""
    ds = load_device_stack(manifest)
    host = SpectralStack(ds.bands, ds.planes.cpu().numpy(), ds.bit_depth, False)
    _register_device_copy(host, ds)
    return host


def crop(stack, x0: int, y0: int, width: int, height: int):
    """Crop all bands identically to the given rectangle (stack.py:216-225);
    a DeviceStack is cropped in HBM."""
    if width <= 0 or height <= 0:
        raise DataError(f"crop rectangle has zero area: {width}x{height}")
    if x0 < 0 or y0 < 0 or x0 + width > stack.width or y0 + height > stack.height:
        raise DataError(f"crop ({x0},{y0},{width},{height}) outside "
                        f"{stack.width}x{stack.height} stack")
    planes = stack.planes[:, y0:y0 + height, x0:x0 + width]
    if isinstance(stack, DeviceStack):
        return DeviceStack(stack.bands, planes.contiguous(), stack.bit_depth, stack.normalized)
    return SpectralStack(tuple(stack.bands), planes.copy(), stack.bit_depth, stack.normalized)
