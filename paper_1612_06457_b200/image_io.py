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
import threading
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


class PendingEncode:
    """An encode enqueued on the device: ``parts()`` waits for it and returns the
    file's byte pieces (host), so a caller can keep several images in flight and
    write finished files while the next ones encode."""

    def __init__(self, finish):
        self._finish = finish
        self._parts = None

    def parts(self) -> list:
        if self._parts is None:
            self._parts = self._finish()
            self._finish = None
        return self._parts

    def bytes(self) -> bytes:
        return b"".join(bytes(p) for p in self.parts())


def encode_png_start(img) -> PendingEncode:
    """Enqueue the PNG encode of a code image (device or host array)."""
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
        done = torch.cuda.Event()
        done.record()
    ihdr = struct.pack(">IIBBBBB", cols, rows, depth, 2 if ch == 3 else 0, 0, 0, 0)

    def finish():   # may run on another thread: wait for the encode, then read back
        done.synchronize()
        with torch.cuda.device(out.device):
            idat = out[: int(n.item())].cpu().numpy()
        return [_PNG_SIGNATURE + _chunk(b"IHDR", ihdr), memoryview(idat), _chunk(b"IEND", b"")]

    return PendingEncode(finish)


def encode_png(img) -> bytes:
    """PNG file bytes of a code image (device or host array)."""
    return encode_png_start(img).bytes()


def _rows_per_strip(rows: int, row_bytes: int) -> int:
    return max(1, min(rows, _STRIP_TARGET // max(1, row_bytes)))


def encode_tiff_start(img, compression: str = "none") -> PendingEncode:
    """Enqueue the TIFF encode of a code image: one IFD, strips of about 256 KB,
    compression 1 (raw) or 8 (zlib deflate with horizontal differencing,
    Predictor 2)."""
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
        done = torch.cuda.Event()
        done.record()

    def finish():   # may run on another thread: wait for the encode, then read back
        done.synchronize()
        with torch.cuda.device(out.device):
            body = out[: int(n.item())].cpu().numpy().tobytes()
            strip_bytes = sizes.cpu().numpy().astype(np.int64)
        return [_tiff_file(body, strip_bytes, rows, cols, ch, depth, code, rps)]

    return PendingEncode(finish)


def encode_tiff(img, compression: str = "none") -> bytes:
    """Baseline little-endian TIFF of a code image (see encode_tiff_start)."""
    return encode_tiff_start(img, compression).bytes()


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


def save_image_start(img, path: str | Path, compression: str = "none"):
    """Check the arguments of save_image and enqueue the encode; returns a
    function that waits for the device and writes the file."""
    path = Path(path)
    check_image(img)
    suffix = path.suffix.lower()
    if suffix in (".tif", ".tiff"):
        if compression not in _TIFF_COMPRESSION:
            raise DataError(f"TIFF compression must be 'none' or 'deflate', got {compression!r}")
        pending = encode_tiff_start(img, compression)
    elif suffix == ".png":
        pending = encode_png_start(img)
    else:
        raise DataError(f"unsupported image format {suffix!r} (use .tif/.tiff/.png)")

    def write():
        parts = pending.parts()
        path.parent.mkdir(parents=True, exist_ok=True)
        try:
            with open(path, "wb") as f:
                for part in parts:
                    f.write(part)
        except OSError as e:
            raise DataError(f"failed to write image {path}: {e}") from None

    return write


def save_image(img, path: str | Path, compression: str = "none") -> None:
    """Write a grayscale or RGB code image as TIFF or PNG (rendering.py:303-331).

    ``img`` may be a host array or a device tensor (e.g. rendered codes still
    in HBM); the encode runs on the device either way."""
    save_image_start(img, path, compression)()


# ------------------------------------------------------------------ decode

_TIFF_TYPES = {1: ("B", 1), 3: ("H", 2), 4: ("I", 4), 16: ("Q", 8)}
_TIFF_CODES = {1: 1, 5: 5, 8: 8, 32946: 8}      # Compression tag -> decoder (raw, LZW, zlib)


# the most a stream can expand: raw 1:1, deflate 1032:1 (RFC 1951: 258 bytes per 2 bits),
# TIFF LZW 12-bit codes of strings up to a strip long (bounded here by 4096:1)
_MAX_EXPANSION = {1: 1, 8: 1032, 5: 4096}
_MAX_IMAGE_BYTES = 1 << 35


class _Unsupported(Exception):
    """A file layout the device decoders do not handle (the caller uses cv2)."""


def _align(n: int, a: int = 256) -> int:
    return -(-int(n) // a) * a


def _tiff_layout(data: bytes) -> dict:
    """Parse the first IFD of a classic TIFF (host, header bytes only)."""
    if len(data) < 8 or data[:2] not in (b"II", b"MM"):
        raise _Unsupported("not a TIFF")
    bo = "<" if data[:2] == b"II" else ">"
    magic, ifd = struct.unpack(bo + "HI", data[2:8])
    if magic != 42:
        raise _Unsupported("not a classic TIFF")
    if ifd + 2 > len(data):
        raise DataError("TIFF directory runs past the end of the file")
    (n,) = struct.unpack(bo + "H", data[ifd:ifd + 2])
    if ifd + 2 + 12 * n > len(data):
        raise DataError("TIFF directory runs past the end of the file")
    tags = {}
    for i in range(n):
        tag, typ, count = struct.unpack(bo + "HHI", data[ifd + 2 + 12 * i:ifd + 10 + 12 * i])
        if typ not in _TIFF_TYPES:
            continue
        code, size = _TIFF_TYPES[typ]
        raw_at = ifd + 10 + 12 * i
        if size * count > 4:
            (raw_at,) = struct.unpack(bo + "I", data[raw_at:raw_at + 4])
        if raw_at + size * count > len(data):
            raise DataError(f"TIFF tag {tag} runs past the end of the file")
        tags[tag] = list(struct.unpack(bo + code * count, data[raw_at:raw_at + size * count]))
    get = lambda t, d=None: tags.get(t) or [d]  # noqa: E731
    lay = {
        "bo": bo, "width": get(256)[0], "height": get(257)[0], "bps": get(258, 1),
        "compression": get(259, 1)[0], "photometric": get(262, 1)[0], "spp": get(277, 1)[0],
        "rps": get(278, 2 ** 32 - 1)[0], "planar": get(284, 1)[0], "predictor": get(317, 1)[0],
        "format": get(339, 1)[0], "offsets": tags.get(273), "counts": tags.get(279),
        "tile_w": get(322)[0], "tile_h": get(323)[0],
        "tile_offsets": tags.get(324), "tile_counts": tags.get(325),
    }
    lay["tiled"] = lay["tile_w"] is not None
    if lay["tiled"]:
        if lay["tile_h"] is None or lay["tile_offsets"] is None or lay["tile_counts"] is None:
            raise _Unsupported("incomplete tile tags")
    elif lay["offsets"] is None or lay["counts"] is None:
        raise _Unsupported("strip-less TIFF")
    if lay["compression"] not in _TIFF_CODES or lay["predictor"] not in (1, 2):
        raise _Unsupported(f"compression {lay['compression']} / predictor {lay['predictor']}")
    if len(set(lay["bps"])) != 1 or lay["bps"][0] not in (8, 16) or lay["format"] != 1:
        raise _Unsupported("sample type")
    if lay["spp"] not in (1, 3) or (lay["spp"] == 3 and lay["planar"] != 1):
        raise _Unsupported("sample layout")
    if lay["photometric"] not in ((1,) if lay["spp"] == 1 else (2,)):
        raise _Unsupported(f"photometric {lay['photometric']}")
    return lay


def _tiff_plan(data: bytes) -> dict:
    """Geometry and stream tables of a device-decodable TIFF (host).  Streams
    are the strips, or the tiles (decoded into a scratch area behind the image
    and scattered into its rows afterwards)."""
    lay = _tiff_layout(data)
    h, w, ch = int(lay["height"] or 0), int(lay["width"] or 0), int(lay["spp"])
    if h <= 0 or w <= 0:
        raise DataError("TIFF has an empty image")
    depth = int(lay["bps"][0])
    px = ch * depth // 8
    rb = w * px
    if h * rb > _MAX_IMAGE_BYTES:
        raise DataError(f"image of {h * rb} bytes is larger than the decoder accepts")
    plan = {"kind": "tiff", "payload": data, "h": h, "w": w, "ch": ch, "depth": depth,
            "bytes": h * rb, "code": _TIFF_CODES[lay["compression"]],
            "predictor": int(lay["predictor"]), "swap": int(lay["bo"] == ">" and depth == 16),
            "tiled": bool(lay["tiled"])}
    if lay["tiled"]:
        tw, th = int(lay["tile_w"]), int(lay["tile_h"])
        if tw <= 0 or th <= 0:
            raise DataError("TIFF tile size must be positive")
        across, down = -(-w // tw), -(-h // th)
        n = across * down
        offs = np.asarray(lay["tile_offsets"], dtype=np.int64)
        counts = np.asarray(lay["tile_counts"], dtype=np.int64)
        if len(offs) != n or len(counts) != n:
            raise DataError(f"TIFF lists {len(offs)} tiles, expected {n}")
        tile_bytes = th * tw * px
        if tile_bytes > max(1 << 26, 16 * h * rb):   # a 64 MB tile for a small image: refuse the scratch
            raise DataError("TIFF tile size does not fit the image")
        scratch0 = _align(h * rb)
        plan.update(tile_w=tw, tile_h=th, across=across, ntiles=n, scratch=scratch0,
                    out_off=scratch0 + np.arange(n, dtype=np.int64) * tile_bytes,
                    out_len=np.full(n, tile_bytes, dtype=np.int64),
                    region=scratch0 + _align(n * tile_bytes))
    else:
        rps = min(int(lay["rps"]), h)
        if rps <= 0:
            raise DataError("TIFF RowsPerStrip must be positive")
        n = -(-h // rps)
        offs = np.asarray(lay["offsets"], dtype=np.int64)
        counts = np.asarray(lay["counts"], dtype=np.int64)
        if len(offs) != n or len(counts) != n:
            raise DataError(f"TIFF lists {len(offs)} strips, expected {n}")
        out_len = np.full(n, rps * rb, dtype=np.int64)
        out_len[-1] = (h - (n - 1) * rps) * rb
        plan.update(out_off=np.arange(n, dtype=np.int64) * rps * rb, out_len=out_len,
                    region=_align(h * rb))
    if int((offs + counts).max()) > len(data):
        raise DataError("TIFF strip runs past the end of the file")
    plan.update(offs=offs, counts=counts)
    return plan


def _png_plan(data: bytes) -> dict:
    """Geometry of a device-decodable PNG (host: chunk walk only).  Grayscale or
    RGB, 8 or 16 bits, not interlaced, no transparency chunk; the payload staged
    to the device is the IDAT chunks' zlib stream."""
    if data[:8] != _PNG_SIGNATURE:
        raise _Unsupported("not a PNG")
    at, ihdr, idat, seen_end = 8, None, [], False
    while at + 12 <= len(data):
        (n,) = struct.unpack(">I", data[at:at + 4])
        kind = data[at + 4:at + 8]
        body_at = at + 8
        if body_at + n + 4 > len(data):
            raise DataError("PNG chunk runs past the end of the file")
        if kind in (b"IHDR", b"IDAT"):   # critical chunks: CRC checked, as libpng does
            (crc,) = struct.unpack(">I", data[body_at + n:body_at + n + 4])
            if zlib.crc32(data[at + 4:body_at + n]) != crc:
                raise DataError(f"PNG {kind.decode()} chunk fails its CRC")
        if kind == b"IHDR":
            if n != 13:
                raise DataError("PNG IHDR chunk has the wrong length")
            ihdr = struct.unpack(">IIBBBBB", data[body_at:body_at + 13])
        elif kind == b"IDAT":
            idat.append(data[body_at:body_at + n])
        elif kind in (b"tRNS", b"PLTE"):
            raise _Unsupported("palette / transparency")
        elif kind == b"IEND":
            seen_end = True
            break
        at = body_at + n + 4
    if ihdr is None or not idat or not seen_end:
        raise DataError("PNG has no IHDR / IDAT / IEND chunk")
    w, h, depth, color, comp, filt, interlace = ihdr
    if color not in (0, 2) or depth not in (8, 16) or interlace != 0 or comp != 0 or filt != 0:
        raise _Unsupported(f"PNG colour type {color}, depth {depth}, interlace {interlace}")
    if w <= 0 or h <= 0:
        raise DataError("PNG has an empty image")
    ch = 3 if color == 2 else 1
    rb = w * ch * depth // 8
    work0 = _align(h * rb)
    return {"kind": "png", "payload": b"".join(idat), "h": h, "w": w, "ch": ch, "depth": depth,
            "bytes": h * rb, "code": 8, "work": work0, "region": work0 + _align(h * (rb + 1)),
            "offs": np.zeros(1, dtype=np.int64), "counts": np.asarray([sum(map(len, idat))], dtype=np.int64),
            "out_off": np.asarray([work0], dtype=np.int64),
            "out_len": np.asarray([h * (rb + 1)], dtype=np.int64)}


_STAGING: dict = {}
_STAGING_LOCK = threading.Lock()   # one decode fills / copies out of the staging buffer at a time


def _pinned_staging(nbytes: int) -> torch.Tensor:
    """A cached, grow-only pinned host buffer for the compressed bytes (pinning
    memory costs more than decoding a small stack; the buffer is reused once the
    previous copy out of it has completed)."""
    buf, busy = _STAGING.get("buf"), _STAGING.get("busy")
    if busy is not None:
        busy.synchronize()            # the last H2D out of the buffer
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        _STAGING["buf"] = buf
    return buf[:nbytes]


def _plan(data: bytes) -> dict:
    plan = _png_plan(data) if data[:8] == _PNG_SIGNATURE else _tiff_plan(data)
    if plan["bytes"] > _MAX_IMAGE_BYTES:
        raise DataError(f"image of {plan['bytes']} bytes is larger than the decoder accepts")
    limit = plan["counts"] * _MAX_EXPANSION[plan["code"]] + 64
    if plan["code"] == 1 and plan["kind"] == "tiff":
        limit = plan["counts"]
    if np.any(plan["out_len"] > limit):
        raise DataError("image data is too short for the image size in its header")
    return plan


def decode_batch(datas: list, device=None) -> list:
    """Device planes of several image files -- TIFFs (strips or tiles; raw, LZW
    or deflate; Predictor 1 / 2; either byte order) and PNGs (grayscale / RGB,
    8 / 16 bit) -- with one staging copy and one decode launch per compression
    kind, so every stream of every file decodes in parallel (a PNG is one
    stream).  Raises _Unsupported if any file has another layout."""
    plans = [_plan(d) for d in datas]
    device = device or dev.require_cuda()
    file_base = np.cumsum([0] + [_align(len(pl["payload"]), 16) for pl in plans])
    out_base = np.cumsum([0] + [pl["region"] for pl in plans])
    with torch.cuda.device(device):
        with _STAGING_LOCK:
            host = _pinned_staging(int(file_base[-1]) + 16)
            hv = host.numpy()
            for pl, b0 in zip(plans, file_base):
                hv[b0:b0 + len(pl["payload"])] = np.frombuffer(pl["payload"], dtype=np.uint8)
            src = host.to(device, non_blocking=True)
            _STAGING["busy"] = torch.cuda.Event()
            _STAGING["busy"].record()
        out = torch.empty(int(out_base[-1]) + 16, dtype=torch.uint8, device=device)
        L = _lib.lib()
        s = dev.stream_handle()
        statuses = []
        for code in (1, 5, 8):
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
            largest = int(max(int(plans[i]["out_len"].max()) for i in sel))
            _lib.check(L.ut_decode_streams(src.data_ptr(), tables[0].data_ptr(),
                                           tables[1].data_ptr(), n, code, out.data_ptr(),
                                           tables[2].data_ptr(), tables[3].data_ptr(), largest,
                                           status.data_ptr(), s), "ut_decode_streams")
            statuses.append(status)
        _raise_on_bad_streams(statuses)   # before the filters / predictors run over damaged rows
        pngs = [i for i, pl in enumerate(plans) if pl["kind"] == "png"]
        if pngs:
            table = torch.from_numpy(np.asarray(
                [[out_base[i] + plans[i]["work"], out_base[i], plans[i]["h"], plans[i]["w"],
                  plans[i]["ch"], plans[i]["depth"]] for i in pngs], dtype=np.int64)).to(device)
            status = torch.empty(len(pngs), dtype=torch.int32, device=device)
            _lib.check(L.ut_png_unfilter(out.data_ptr(), table.data_ptr(), len(pngs),
                                         out.data_ptr(), status.data_ptr(), s), "ut_png_unfilter")
            statuses.append(status)
        images = []
        for pl, o0 in zip(plans, out_base):
            o0 = int(o0)
            dtype = torch.uint8 if pl["depth"] == 8 else torch.uint16
            img = out[o0:o0 + pl["bytes"]].view(dtype)
            if pl["kind"] == "tiff" and pl["tiled"]:
                # byte order and Predictor 2 are per tile row: undo them on the tiles
                t0 = o0 + pl["scratch"]
                tiles = out[t0:t0 + pl["ntiles"] * pl["tile_h"] * pl["tile_w"] * pl["ch"] * pl["depth"] // 8]
                _lib.check(L.ut_unpredict(tiles.data_ptr(), pl["depth"], pl["ntiles"] * pl["tile_h"],
                                          pl["tile_w"], pl["ch"], pl["predictor"], pl["swap"], s),
                           "ut_unpredict")
                px = pl["ch"] * pl["depth"] // 8
                _lib.check(L.ut_untile(tiles.data_ptr(), img.data_ptr(), pl["h"], pl["w"] * px,
                                       pl["tile_h"], pl["tile_w"] * px, pl["across"], pl["ntiles"], s),
                           "ut_untile")
            elif pl["kind"] == "tiff":
                _lib.check(L.ut_unpredict(img.data_ptr(), pl["depth"], pl["h"], pl["w"], pl["ch"],
                                          pl["predictor"], pl["swap"], s), "ut_unpredict")
            images.append(img.view(pl["h"], pl["w"], pl["ch"]) if pl["ch"] == 3
                          else img.view(pl["h"], pl["w"]))
        _raise_on_bad_streams(statuses[-1:] if pngs else [])
    return images


def _raise_on_bad_streams(statuses: list) -> None:
    codes = torch.cat([st[st != 0] for st in statuses]).cpu().tolist() if statuses else []
    if codes:
        names = {1: "malformed", 2: "too short", 3: "too long", 4: "checksum", 5: "header"}
        kinds = sorted({names.get(int(c), str(c)) for c in codes})
        raise DataError(f"image data has {len(codes)} undecodable stream(s) ({', '.join(kinds)})")


def decode_tiff_batch(datas: list, device=None) -> list:
    """Device planes of several TIFFs (see decode_batch)."""
    for d in datas:
        if d[:8] == _PNG_SIGNATURE:
            raise _Unsupported("not a TIFF")
    return decode_batch(datas, device)


def decode_tiff(data: bytes, device=None) -> torch.Tensor:
    """Device (H, W[, 3]) uint8 / uint16 planes of one TIFF."""
    return decode_tiff_batch([data], device)[0]


def decode_png(data: bytes, device=None) -> torch.Tensor:
    """Device (H, W[, 3]) uint8 / uint16 planes of one PNG."""
    if data[:8] != _PNG_SIGNATURE:
        raise _Unsupported("not a PNG")
    return decode_batch([data], device)[0]


def read_image_device(path: str | Path, device=None):
    """(device tensor, decoded-on-device flag) for an image file: TIFFs (strips
    or tiles; raw / LZW / deflate) and PNGs (grayscale / RGB, 8 / 16 bit) decode
    on the B200; other layouts (palette, interlaced, alpha, JPEG-in-TIFF, ...)
    go through cv2.imread on the host exactly as the reference reads them, then
    to the device.  DataError if the file cannot be read."""
    path = Path(path)
    try:
        data = path.read_bytes()
    except OSError:
        raise DataError(f"cannot read image {path}") from None
    try:
        return decode_batch([data], device)[0], True
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
