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


# ------------------------------------------------------------------ decode

_TIFF_TYPES = {1: ("B", 1), 3: ("H", 2), 4: ("I", 4), 16: ("Q", 8)}


class _Unsupported(Exception):
    """A file layout the device decoder does not handle (the caller uses cv2)."""


def _tiff_layout(data: bytes) -> dict:
    """Parse the first IFD of a classic TIFF (host, header bytes only)."""
    if len(data) < 8 or data[:2] not in (b"II", b"MM"):
        raise _Unsupported("not a TIFF")
    bo = "<" if data[:2] == b"II" else ">"
    magic, ifd = struct.unpack(bo + "HI", data[2:8])
    if magic != 42:
        raise _Unsupported("not a classic TIFF")
    (n,) = struct.unpack(bo + "H", data[ifd:ifd + 2])
    tags = {}
    for i in range(n):
        tag, typ, count = struct.unpack(bo + "HHI", data[ifd + 2 + 12 * i:ifd + 10 + 12 * i])
        if typ not in _TIFF_TYPES:
            continue
        code, size = _TIFF_TYPES[typ]
        raw_at = ifd + 10 + 12 * i
        if size * count > 4:
            (raw_at,) = struct.unpack(bo + "I", data[raw_at:raw_at + 4])
        tags[tag] = list(struct.unpack(bo + code * count, data[raw_at:raw_at + size * count]))
    get = lambda t, d=None: tags.get(t, [d])  # noqa: E731
    lay = {
        "bo": bo, "width": get(256)[0], "height": get(257)[0], "bps": get(258, 1),
        "compression": get(259, 1)[0], "photometric": get(262, 1)[0], "spp": get(277, 1)[0],
        "rps": get(278, 2 ** 32 - 1)[0], "planar": get(284, 1)[0], "predictor": get(317, 1)[0],
        "format": get(339, 1)[0], "offsets": tags.get(273), "counts": tags.get(279),
    }
    if 322 in tags or lay["offsets"] is None or lay["counts"] is None:
        raise _Unsupported("tiled or strip-less TIFF")
    if lay["compression"] not in (1, 8, 32946) or lay["predictor"] not in (1, 2):
        raise _Unsupported(f"compression {lay['compression']} / predictor {lay['predictor']}")
    if len(set(lay["bps"])) != 1 or lay["bps"][0] not in (8, 16) or lay["format"] != 1:
        raise _Unsupported("sample type")
    if lay["spp"] not in (1, 3) or (lay["spp"] == 3 and lay["planar"] != 1):
        raise _Unsupported("sample layout")
    if lay["photometric"] not in ((1,) if lay["spp"] == 1 else (2,)):
        raise _Unsupported(f"photometric {lay['photometric']}")
    return lay


def _tiff_plan(data: bytes) -> dict:
    """Geometry and strip tables of a device-decodable TIFF (host)."""
    lay = _tiff_layout(data)
    h, w, ch = int(lay["height"]), int(lay["width"]), int(lay["spp"])
    depth = int(lay["bps"][0])
    rb = w * ch * depth // 8
    rps = min(int(lay["rps"]), h)
    nstrips = -(-h // rps)
    offs = np.asarray(lay["offsets"], dtype=np.int64)
    counts = np.asarray(lay["counts"], dtype=np.int64)
    if len(offs) != nstrips or len(counts) != nstrips:
        raise DataError(f"TIFF lists {len(offs)} strips, expected {nstrips}")
    if int((offs + counts).max()) > len(data):
        raise DataError("TIFF strip runs past the end of the file")
    out_len = np.full(nstrips, rps * rb, dtype=np.int64)
    out_len[-1] = (h - (nstrips - 1) * rps) * rb
    return {"h": h, "w": w, "ch": ch, "depth": depth, "bytes": h * rb, "offs": offs,
            "counts": counts, "out_off": np.arange(nstrips, dtype=np.int64) * rps * rb,
            "out_len": out_len, "code": 1 if lay["compression"] == 1 else 8,
            "predictor": int(lay["predictor"]), "swap": int(lay["bo"] == ">" and depth == 16)}


def decode_tiff_batch(datas: list, device=None) -> list:
    """Device planes of several stripped TIFFs (raw or deflate, Predictor 1 / 2,
    either byte order) with one staging copy and one decode launch per
    compression kind, so every strip of every file decodes in parallel.
    Raises _Unsupported if any file has another layout."""
    plans = [_tiff_plan(d) for d in datas]
    device = device or dev.require_cuda()
    file_base = np.cumsum([0] + [len(d) for d in datas])
    # each image starts on a 256-byte boundary (16-bit views need no copy)
    out_base = np.cumsum([0] + [-(-pl["bytes"] // 256) * 256 for pl in plans])
    with torch.cuda.device(device):
        host = torch.empty(int(file_base[-1]), dtype=torch.uint8, pin_memory=True)
        hv = host.numpy()
        for d, b0 in zip(datas, file_base):
            hv[b0:b0 + len(d)] = np.frombuffer(d, dtype=np.uint8)
        src = host.to(device, non_blocking=True)
        out = torch.empty(int(out_base[-1]) + 16, dtype=torch.uint8, device=device)
        L = _lib.lib()
        s = dev.stream_handle()
        statuses = []
        for code in (1, 8):
            sel = [i for i, pl in enumerate(plans) if pl["code"] == code]
            if not sel:
                continue
            cat = lambda key, base: np.concatenate(  # noqa: E731
                [plans[i][key] + (base[i] if base is not None else 0) for i in sel])
            tables = torch.from_numpy(np.stack([cat("offs", file_base), cat("counts", None),
                                                cat("out_off", out_base),
                                                cat("out_len", None)])).to(device)
            n = tables.shape[1]
            status = torch.empty(n, dtype=torch.int32, device=device)
            _lib.check(L.ut_decode_strips(src.data_ptr(), tables[0].data_ptr(),
                                          tables[1].data_ptr(), n, code, out.data_ptr(),
                                          tables[2].data_ptr(), tables[3].data_ptr(),
                                          status.data_ptr(), s), "ut_decode_strips")
            statuses.append(status)
        images = []
        for pl, o0 in zip(plans, out_base):
            dtype = torch.uint8 if pl["depth"] == 8 else torch.uint16
            flat = out[int(o0):int(o0) + pl["bytes"]]
            img = flat.view(dtype)
            _lib.check(L.ut_unpredict(img.data_ptr(), pl["depth"], pl["h"], pl["w"], pl["ch"],
                                      pl["predictor"], pl["swap"], s), "ut_unpredict")
            images.append(img.view(pl["h"], pl["w"], pl["ch"]) if pl["ch"] == 3
                          else img.view(pl["h"], pl["w"]))
        bad = sum(int((st != 0).sum().item()) for st in statuses)
    if bad:
        raise DataError(f"TIFF data has {bad} undecodable strip(s)")
    return images


def decode_tiff(data: bytes, device=None) -> torch.Tensor:
    """Device (H, W[, 3]) uint8 / uint16 planes of one stripped TIFF."""
    return decode_tiff_batch([data], device)[0]


def read_image_device(path: str | Path, device=None):
    """(device tensor, decoded-on-device flag) for an image file: stripped
    TIFFs decode on the B200; other files (PNG, LZW / tiled TIFF, ...) go
    through cv2.imread on the host exactly as the reference reads them, then
    to the device.  DataError if the file cannot be read."""
    path = Path(path)
    try:
        data = path.read_bytes()
    except OSError:
        raise DataError(f"cannot read image {path}") from None
    try:
        return decode_tiff(data, device), True
    except _Unsupported:
        pass
    import cv2  # the reference's decoder, for layouts the device path does not parse

    img = cv2.imdecode(np.frombuffer(data, dtype=np.uint8), cv2.IMREAD_UNCHANGED)
    if img is None:
        raise DataError(f"cannot read image {path}")
    if img.ndim == 3 and img.shape[2] == 3:
        img = img[:, :, ::-1]  # BGR -> RGB
    return dev.to_device(np.ascontiguousarray(img), device or dev.require_cuda()), False


def load_image(path: str | Path) -> np.ndarray:
    """Read a TIFF or PNG back as uint8/uint16, RGB channel order
    (rendering.py:334-343)."""
    t, _ = read_image_device(path)
    if t.dim() == 3 and t.shape[2] != 3:
        raise DataError(f"{path}: expected 3 channels, got {t.shape[2]}")
    img = t.cpu().numpy()
    check_image(img)
    return np.ascontiguousarray(img)
