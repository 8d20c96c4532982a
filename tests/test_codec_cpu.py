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
