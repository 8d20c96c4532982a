"""Host framing of the device encoders (image_io.py), checked on CPU with the
reference's codec library: the TIFF header/IFD around raw strips and the PNG
signature/IHDR/IEND around IDAT data decode to the input (the device part --
filters, deflate, CRCs -- is covered by tests/test_gpu_codec.py)."""

import struct
import zlib

import numpy as np
import pytest

cv2 = pytest.importorskip("cv2")

from paper_1612_06457_b200 import image_io  # noqa: E402
from paper_1612_06457_b200.errors import DataError  # noqa: E402


@pytest.mark.parametrize("shape,dtype", [((20, 30), np.uint8), ((1000, 300), np.uint16),
                                         ((33, 17, 3), np.uint8)])
def test_tiff_framing_raw_strips(tmp_path, shape, dtype):
    rng = np.random.default_rng(1)
    img = rng.integers(0, np.iinfo(dtype).max, size=shape).astype(dtype)
    ch = 3 if img.ndim == 3 else 1
    depth = 8 * img.itemsize
    rb = shape[1] * ch * img.itemsize
    rps = image_io._rows_per_strip(shape[0], rb)
    nstrips = -(-shape[0] // rps)
    sizes = np.full(nstrips, rps * rb, dtype=np.int64)
    sizes[-1] = (shape[0] - (nstrips - 1) * rps) * rb
    data = image_io._tiff_file(img.tobytes(), sizes, shape[0], shape[1], ch, depth, 1, rps)
    path = tmp_path / "x.tif"
    path.write_bytes(data)
    got = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    if ch == 3:
        got = got[:, :, ::-1]
    assert np.array_equal(got, img)


def test_tiff_framing_deflate_strips(tmp_path):
    """Strips as independent zlib streams over Predictor-2 samples."""
    rng = np.random.default_rng(2)
    img = rng.integers(0, 60000, size=(700, 400)).astype(np.uint16)
    rb = 400 * 2
    rps = image_io._rows_per_strip(700, rb)
    pred = img.copy()
    pred[:, 1:] = img[:, 1:] - img[:, :-1]
    strips = [zlib.compress(pred[r:r + rps].tobytes()) for r in range(0, 700, rps)]
    data = image_io._tiff_file(b"".join(strips), np.array([len(s) for s in strips]), 700, 400,
                               1, 16, 8, rps)
    path = tmp_path / "x.tif"
    path.write_bytes(data)
    assert np.array_equal(cv2.imread(str(path), cv2.IMREAD_UNCHANGED), img)


def test_png_framing(tmp_path):
    img = np.arange(15 * 15, dtype=np.uint8).reshape(15, 15)
    raw = b"".join(b"\0" + img[r].tobytes() for r in range(15))
    idat = image_io._chunk(b"IDAT", zlib.compress(raw))
    ihdr = struct.pack(">IIBBBBB", 15, 15, 8, 0, 0, 0, 0)
    data = image_io._PNG_SIGNATURE + image_io._chunk(b"IHDR", ihdr) + idat + \
        image_io._chunk(b"IEND", b"")
    path = tmp_path / "x.png"
    path.write_bytes(data)
    assert np.array_equal(cv2.imread(str(path), cv2.IMREAD_UNCHANGED), img)


def test_check_image_messages():
    with pytest.raises(DataError, match="uint8 or uint16"):
        image_io.check_image(np.zeros((2, 2), dtype=np.int32))
    with pytest.raises(DataError, match="3 channels"):
        image_io.check_image(np.zeros((2, 2, 2), dtype=np.uint8))
    with pytest.raises(DataError, match="2-D or 3-D"):
        image_io.check_image(np.zeros((2,), dtype=np.uint8))
    assert image_io.check_image(np.zeros((2, 2, 3), dtype=np.uint16)) == (16, 3)


def test_render_names_and_recipe_validation(tmp_path):
    import paper_1612_06457_b200 as ut
    assert ut.CompositeRecipe(0, 1, 2).suffix() == "_R0G1B2"
    assert ut.CompositeRecipe(0, 1, 2, swap=(1, 2)).suffix() == "_R0G1B2_swap12"
    with pytest.raises(DataError):
        ut.CompositeRecipe(0, 1, 2, swap=(1, 1))
    with pytest.raises(DataError):
        ut.CompositeRecipe(0, 1, 2, swap=(0, 3))
    spec = ut.RenderSpec("percentile", 0.1)
    assert ut.plane_filename("run", 3, spec, "png") == "run_plane03_p0_1.png"
    assert ut.composite_filename("run", ut.CompositeRecipe(2, 1, 0)) == "run_R2G1B0.png"
    with pytest.raises(DataError, match="format"):
        ut.render_planes(None, None, [spec], tmp_path, fmt="jpg")
    with pytest.raises(DataError, match="spec"):
        ut.render_planes(None, None, [], tmp_path)


def test_manifest_errors_before_any_decode(tmp_path):
    """load_stack's manifest checks (test_stack.py:86-113) need no device."""
    import paper_1612_06457_b200 as ut

    def manifest(lines):
        p = tmp_path / "m.txt"
        p.write_text("\n".join(lines) + "\n", encoding="utf-8")
        return p

    with pytest.raises(DataError, match="gone.tif"):
        ut.load_stack(manifest(["gone.tif,365,uv"]))
    with pytest.raises(DataError, match="line 2"):
        ut.load_stack(manifest(["# header", "not enough fields"]))
    with pytest.raises(DataError):
        ut.load_stack(manifest(["# nothing"]))
    with pytest.raises(DataError, match="manifest not found"):
        ut.load_stack(tmp_path / "absent.txt")


def test_tiff_layout_parse():
    """Host IFD parsing of a device-style TIFF (framing only)."""
    img = np.arange(6 * 5, dtype=np.uint16).reshape(6, 5)
    data = image_io._tiff_file(img.tobytes(), np.array([img.nbytes]), 6, 5, 1, 16, 1, 6)
    lay = image_io._tiff_layout(data)
    assert (lay["width"], lay["height"], lay["bps"], lay["compression"]) == (5, 6, [16], 1)
    assert lay["offsets"] == [8] and lay["counts"] == [img.nbytes]
    with pytest.raises(image_io._Unsupported):
        image_io._tiff_layout(b"\x89PNG\r\n\x1a\n")


def _png_bytes(w, h, depth, color, interlace=0, extra=(), idat_parts=2, drop_iend=False):
    rb = w * {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}[color] * depth // 8
    raw = b"".join(b"\0" + bytes(rb) for _ in range(h))
    z = zlib.compress(raw)
    chunk = lambda k, d: struct.pack(">I", len(d)) + k + d + struct.pack(">I", zlib.crc32(k + d))  # noqa: E731
    cut = max(1, len(z) // idat_parts)
    body = b"".join(chunk(b"IDAT", z[i:i + cut]) for i in range(0, len(z), cut))
    out = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, color, 0, 0, interlace))
    out += b"".join(chunk(k, d) for k, d in extra) + body
    return out if drop_iend else out + chunk(b"IEND", b""), z


def test_png_plan_host_parsing():
    """Host chunk walk of the PNG decoder (image_io._png_plan): geometry, the
    IDAT payloads joined into one zlib stream, and which layouts are left to cv2."""
    data, z = _png_bytes(7, 5, 16, 2, extra=[(b"tEXt", b"k\0v")], idat_parts=3)
    plan = image_io._png_plan(data)
    assert (plan["h"], plan["w"], plan["ch"], plan["depth"]) == (5, 7, 3, 16)
    assert plan["payload"] == z and plan["code"] == 8
    assert plan["bytes"] == 5 * 7 * 6 and int(plan["out_len"][0]) == 5 * (7 * 6 + 1)
    assert int(plan["out_off"][0]) >= plan["bytes"] and plan["region"] >= plan["out_off"][0] + plan["out_len"][0]
    for kwargs in ({"color": 6}, {"color": 4}, {"color": 3, "extra": [(b"PLTE", bytes(6))]},
                   {"color": 0, "interlace": 1}, {"color": 0, "extra": [(b"tRNS", b"\0\0")]}):
        args = {"w": 4, "h": 4, "depth": 8, "color": 0}
        args.update(kwargs)
        with pytest.raises(image_io._Unsupported):
            image_io._png_plan(_png_bytes(**args)[0])
    with pytest.raises(image_io._Unsupported):
        image_io._png_plan(b"II*\0" + bytes(16))
    with pytest.raises(DataError):
        image_io._png_plan(_png_bytes(4, 4, 8, 0, drop_iend=True)[0])
    with pytest.raises(DataError):
        image_io._png_plan(data[:60])
    bad = bytearray(data)
    bad[bad.index(b"IDAT") + 6] ^= 0x40          # payload bit flip: the chunk CRC catches it
    with pytest.raises(DataError, match="CRC"):
        image_io._png_plan(bytes(bad))


def _ifd_tiff(entries, body=b""):
    ifd_at = 8 + len(body)
    extra_at = ifd_at + 2 + 12 * len(entries) + 4
    ifd, extra = struct.pack("<H", len(entries)), b""
    for tag, typ, vals in entries:
        raw = struct.pack("<" + ("H" if typ == 3 else "I") * len(vals), *vals)
        if len(raw) <= 4:
            ifd += struct.pack("<HHI", tag, typ, len(vals)) + raw.ljust(4, b"\0")
        else:
            ifd += struct.pack("<HHII", tag, typ, len(vals), extra_at + len(extra))
            extra += raw
    return b"II*\0" + struct.pack("<I", ifd_at) + body + ifd + struct.pack("<I", 0) + extra


def test_tiff_plan_tiles_and_lzw():
    """Host IFD parsing for tiled and LZW TIFFs (image_io._tiff_plan): tiles decode
    into a scratch area behind the image; degenerate tags are DataErrors."""
    body = bytes(4 * 16 * 16 * 2)
    tiled = [(256, 4, [20]), (257, 4, [30]), (258, 3, [16]), (259, 3, [5]), (262, 3, [1]), (277, 3, [1]),
             (317, 3, [2]), (322, 4, [16]), (323, 4, [16]), (324, 4, [8 + 512 * i for i in range(4)]),
             (325, 4, [512] * 4)]
    plan = image_io._tiff_plan(_ifd_tiff(tiled, body))
    assert plan["tiled"] and plan["code"] == 5 and plan["predictor"] == 2
    assert (plan["across"], plan["ntiles"], plan["tile_w"], plan["tile_h"]) == (2, 4, 16, 16)
    assert plan["bytes"] == 30 * 20 * 2 and int(plan["out_off"][0]) == plan["scratch"] >= plan["bytes"]
    assert list(plan["out_len"]) == [512] * 4 and plan["region"] >= plan["scratch"] + 4 * 512
    strips = [(256, 4, [20]), (257, 4, [30]), (258, 3, [8]), (259, 3, [5]), (262, 3, [1]), (277, 3, [1]),
              (273, 4, [8, 208]), (278, 4, [16]), (279, 4, [200, 100])]
    plan = image_io._tiff_plan(_ifd_tiff(strips, bytes(300)))
    assert not plan["tiled"] and plan["code"] == 5 and list(plan["out_len"]) == [320, 280]
    bad = [e if e[0] != 278 else (278, 4, [0]) for e in strips]
    with pytest.raises(DataError, match="RowsPerStrip"):
        image_io._tiff_plan(_ifd_tiff(bad, bytes(300)))
    huge = [e if e[0] not in (322, 323) else (e[0], 4, [1 << 14]) for e in tiled]
    with pytest.raises(DataError):
        image_io._tiff_plan(_ifd_tiff(huge, body))
    past = [e if e[0] != 279 else (279, 4, [200, 5000]) for e in strips]
    with pytest.raises(DataError, match="past the end"):
        image_io._tiff_plan(_ifd_tiff(past, bytes(300)))
    jpeg = [e if e[0] != 259 else (259, 3, [7]) for e in strips]
    with pytest.raises(image_io._Unsupported):
        image_io._tiff_plan(_ifd_tiff(jpeg, bytes(300)))


def test_damaged_tiff_headers_are_data_errors():
    """Truncated files, directories / tag arrays past the end of the file, empty tag
    arrays and sizes the data cannot fill are DataErrors on the host, before any
    device work (found by tools/fuzz/fuzz_corrupt.py: they used to be struct.error)."""
    img = np.arange(40 * 30, dtype=np.uint16).reshape(40, 30)
    data = image_io._tiff_file(img.tobytes(), np.array([img.nbytes]), 40, 30, 1, 16, 1, 40)
    assert image_io._tiff_plan(data)["bytes"] == img.nbytes
    for cut in (9, len(data) - 5, len(data) - 60):
        with pytest.raises(DataError):
            image_io._plan(data[:cut])
    far = bytearray(data)
    far[4:8] = struct.pack("<I", len(data) + 100)          # directory offset past the end
    with pytest.raises(DataError, match="directory"):
        image_io._plan(bytes(far))
    big = _ifd_tiff([(256, 4, [30]), (257, 4, [1 << 20]), (258, 3, [16]), (259, 3, [8]), (262, 3, [1]),
                     (277, 3, [1]), (273, 4, [8]), (278, 4, [1 << 20]), (279, 4, [100])], bytes(100))
    with pytest.raises(DataError, match="too short"):      # 100 bytes cannot inflate to 60 MB
        image_io._plan(big)
