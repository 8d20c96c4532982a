"""Image files from device code planes: PNG and TIFF encoders on the B200.

Mirrors ``save_image`` of /root/reference/pkg/src/undertext/rendering.py
(:303-331): grayscale (H, W) or RGB (H, W, 3) uint8 / uint16 codes, format by
suffix (.png / .tif / .tiff), TIFF compression 'none' or 'deflate', PNG always
compressed, RGB channel order R, G, B in memory; same DataError messages.
The reference calls cv2.imwrite; here ``ut_encode_png`` / ``ut_encode_tiff``
(csrc/codec.cu) do the row filtering / prediction, deflate, Adler-32 and chunk
CRCs on the device, and the host only adds the fixed headers (PNG signature,
IHDR, IEND; TIFF header and IFD) around the device bytes and writes the file.
Files decode with any PNG / TIFF reader (cv2, libpng, libtiff, zlib) and are
byte-deterministic.
"""

from __future__ import annotations

import struct
import zlib
from pathlib import Path

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import DataError

_TIFF_COMPRESSION = {"none": 1, "deflate": 8}   # rendering.py:300
_PNG_SIGNATURE = b"\x89PNG\r\n\x1a\n"
_STRIP_TARGET = 1 << 18                          # bytes per TIFF strip (~256 KB)


def check_image(img) -> tuple[int, int]:
    """(depth, channels) of a code image, with the reference's checks and
    messages (rendering.py:196-201, :311-318); no data is touched."""
    if isinstance(img, torch.Tensor):
        if img.dtype not in (torch.uint8, torch.uint16):
            raise DataError(f"image must be uint8 or uint16, got {img.dtype}")
        depth = 8 if img.dtype == torch.uint8 else 16
    else:
        dt = np.asarray(img).dtype
        if dt not in (np.uint8, np.uint16):
            raise DataError(f"image must be uint8 or uint16, got {dt}")
        depth = 8 if dt == np.uint8 else 16
    shape = tuple(img.shape)
    if len(shape) == 3:
        if shape[2] != 3:
            raise DataError(f"color image must have 3 channels, got {shape[2]}")
        return depth, 3
    if len(shape) == 2:
        return depth, 1
    raise DataError(f"image must be 2-D or 3-D, got shape {shape}")


def _image_on_device(img):
    """(device tensor (H, W, C), depth, channels) of a checked code image."""
    depth, channels = check_image(img)
    shape = tuple(img.shape)
    t = img if isinstance(img, torch.Tensor) else None
    if t is None:
        t = dev.to_device(np.ascontiguousarray(img), dev.require_cuda())
    elif not t.is_cuda:
        t = dev.to_device(t, dev.require_cuda())
    t = t.contiguous()
    if t.numel() == 0:
        raise DataError(f"image must be non-empty, got shape {shape}")
    return t.view(shape[0], shape[1], channels), depth, channels


def _chunk(kind: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + kind + data + struct.pack(">I", zlib.crc32(kind + data))


def encode_png(img) -> bytes:
    """PNG file bytes of a code image (device or host array)."""
    t, depth, ch = _image_on_device(img)
    rows, cols = int(t.shape[0]), int(t.shape[1])
    L = _lib.lib()
    with torch.cuda.device(t.device):
        cap = L.ut_encode_bound(rows, cols, ch, depth, 0, 1)
        ws = dev.workspace("encode", L.ut_encode_ws(rows, cols, ch, depth, 0, 1), t.device)
        out = torch.empty(cap, dtype=torch.uint8, device=t.device)
        n = torch.zeros(1, dtype=torch.int64, device=t.device)
        _lib.check(L.ut_encode_png(t.data_ptr(), rows, cols, ch, depth, out.data_ptr(), cap,
                                   n.data_ptr(), ws.data_ptr(), ws.numel(), dev.stream_handle()),
                   "ut_encode_png")
        idat = out[: int(n.item())].cpu().numpy().tobytes()
    ihdr = struct.pack(">IIBBBBB", cols, rows, depth, 2 if ch == 3 else 0, 0, 0, 0)
    return _PNG_SIGNATURE + _chunk(b"IHDR", ihdr) + idat + _chunk(b"IEND", b"")


def _rows_per_strip(rows: int, row_bytes: int) -> int:
    return max(1, min(rows, _STRIP_TARGET // max(1, row_bytes)))


def encode_tiff(img, compression: str = "none") -> bytes:
    """Baseline little-endian TIFF of a code image: one IFD, strips of about
    256 KB, compression 1 (raw) or 8 (zlib deflate with horizontal
    differencing, Predictor 2)."""
    if compression not in _TIFF_COMPRESSION:
        raise DataError(f"TIFF compression must be 'none' or 'deflate', got {compression!r}")
    code = _TIFF_COMPRESSION[compression]
    t, depth, ch = _image_on_device(img)
    rows, cols = int(t.shape[0]), int(t.shape[1])
    rb = cols * ch * depth // 8
    rps = _rows_per_strip(rows, rb)
    nstrips = -(-rows // rps)
    L = _lib.lib()
    with torch.cuda.device(t.device):
        cap = max(L.ut_encode_bound(rows, cols, ch, depth, 1, rps), rows * rb)
        ws_bytes = L.ut_encode_ws(rows, cols, ch, depth, 1, rps) if code == 8 else 0
        ws = dev.workspace("encode", ws_bytes, t.device)
        out = torch.empty(cap, dtype=torch.uint8, device=t.device)
        n = torch.zeros(1, dtype=torch.int64, device=t.device)
        sizes = torch.zeros(nstrips, dtype=torch.int64, device=t.device)
        _lib.check(L.ut_encode_tiff(t.data_ptr(), rows, cols, ch, depth, code, rps, out.data_ptr(),
                                    cap, sizes.data_ptr(), n.data_ptr(), ws.data_ptr(),
                                    ws.numel(), dev.stream_handle()), "ut_encode_tiff")
        body = out[: int(n.item())].cpu().numpy().tobytes()
        strip_bytes = sizes.cpu().numpy().astype(np.int64)
    return _tiff_file(body, strip_bytes, rows, cols, ch, depth, code, rps)


def _tiff_file(body: bytes, strip_bytes, rows, cols, ch, depth, code, rps) -> bytes:
    nstrips = len(strip_bytes)
    head = 8
    ifd_at = head + len(body)
    ifd_at += ifd_at & 1                        # IFD on a word boundary
    entries = []                                # (tag, type, count, value-or-bytes)
    SHORT, LONG = 3, 4
    entries.append((256, LONG, 1, cols))
    entries.append((257, LONG, 1, rows))
    entries.append((258, SHORT, ch, [depth] * ch))
    entries.append((259, SHORT, 1, code))
    entries.append((262, SHORT, 1, 2 if ch == 3 else 1))
    offsets = head + np.concatenate([[0], np.cumsum(strip_bytes)[:-1]]).astype(np.int64)
    entries.append((273, LONG, nstrips, [int(v) for v in offsets]))
    entries.append((277, SHORT, 1, ch))
    entries.append((278, LONG, 1, rps))
    entries.append((279, LONG, nstrips, [int(v) for v in strip_bytes]))
    entries.append((284, SHORT, 1, 1))
    if code == 8:
        entries.append((317, SHORT, 1, 2))
    n = len(entries)
    extra_at = ifd_at + 2 + 12 * n + 4
    ifd = struct.pack("<H", n)
    extra = b""
    for tag, typ, count, val in entries:
        vals = val if isinstance(val, list) else [val]
        fmt = "<" + ("H" if typ == SHORT else "I") * count
        raw = struct.pack(fmt, *vals)
        if len(raw) <= 4:
            ifd += struct.pack("<HHI", tag, typ, count) + raw.ljust(4, b"\0")
        else:
            ifd += struct.pack("<HHII", tag, typ, count, extra_at + len(extra))
            extra += raw
            extra += b"\0" * (len(extra) & 1)
    ifd += struct.pack("<I", 0)
    total = extra_at + len(extra)
    if total >= 1 << 32:
        raise DataError("image too large for a classic TIFF (4 GiB)")
    header = b"II*\0" + struct.pack("<I", ifd_at)
    pad = b"\0" * (ifd_at - head - len(body))
    return header + body + pad + ifd + extra


def save_image(img, path: str | Path, compression: str = "none") -> None:
    """Write a grayscale or RGB code image as TIFF or PNG (rendering.py:303-331).

    ``img`` may be a host array or a device tensor (e.g. rendered codes still
    in HBM); the encode runs on the device either way."""
    path = Path(path)
    check_image(img)
    suffix = path.suffix.lower()
    if suffix in (".tif", ".tiff"):
        if compression not in _TIFF_COMPRESSION:
            raise DataError(f"TIFF compression must be 'none' or 'deflate', got {compression!r}")
        data = encode_tiff(img, compression)
    elif suffix == ".png":
        data = encode_png(img)
    else:
        raise DataError(f"unsupported image format {suffix!r} (use .tif/.tiff/.png)")
    path.parent.mkdir(parents=True, exist_ok=True)
    try:
        path.write_bytes(data)
    except OSError as e:
        raise DataError(f"failed to write image {path}: {e}") from None
