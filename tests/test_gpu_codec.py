"""save_image on the device (rendering.py:303-331):
PNG and TIFF written by csrc/codec.cu must decode -- with the reference's own
codec library (cv2 = libpng / libtiff) and with zlib -- to exactly the input
codes, be byte-deterministic, and shrink compressible images (the reference's
test_rendering.py:356-401 cases plus multi-unit / multi-strip sizes)."""

import struct
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
cv2 = pytest.importorskip("cv2")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import image_io  # noqa: E402


def cv2_load(path):
    img = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    assert img is not None, f"cv2 cannot decode {path}"
    if img.ndim == 3:
        img = np.ascontiguousarray(img[:, :, ::-1])  # BGR -> RGB
    return img


def png_chunks(data):
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, out = 8, []
    while pos < len(data):
        (n,) = struct.unpack(">I", data[pos:pos + 4])
        kind, body = data[pos + 4:pos + 8], data[pos + 8:pos + 8 + n]
        (crc,) = struct.unpack(">I", data[pos + 8 + n:pos + 12 + n])
        assert crc == zlib.crc32(kind + body), f"bad CRC in {kind} chunk"
        out.append((kind, body))
        pos += 12 + n
    return out


def smooth(rows, cols, depth, seed=0, channels=1):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:rows, 0:cols]
    top = (1 << depth) - 1
    base = (np.sin(x / 37.0) + np.cos(y / 23.0) + 2) / 4 * top
    imgs = []
    for c in range(channels):
        v = base * (0.6 + 0.2 * c) + rng.normal(0, top * 0.004, size=base.shape)
        imgs.append(np.clip(np.rint(v), 0, top))
    a = np.stack(imgs, -1) if channels == 3 else imgs[0]
    return a.astype(np.uint8 if depth == 8 else np.uint16)


SHAPES = [(1, 1), (20, 30), (7, 33333), (300, 1000), (513, 257)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("depth", [8, 16])
@pytest.mark.parametrize("kind", ["random", "smooth", "zeros"])
def test_png_gray_round_trip(tmp_path, shape, depth, kind):
    rng = np.random.default_rng(6)
    dt = np.uint8 if depth == 8 else np.uint16
    if kind == "random":
        img = rng.integers(0, 2 ** depth, size=shape).astype(dt)
    elif kind == "smooth":
        img = smooth(*shape, depth)
    else:
        img = np.zeros(shape, dtype=dt)
    path = tmp_path / "g.png"
    ut.save_image(img, path)
    data = path.read_bytes()
    chunks = png_chunks(data)
    assert chunks[0][0] == b"IHDR" and chunks[-1][0] == b"IEND"
    raw = zlib.decompress(b"".join(b for k, b in chunks if k == b"IDAT"))
    assert len(raw) == shape[0] * (1 + shape[1] * depth // 8)
    got = cv2_load(path)
    assert got.dtype == dt and np.array_equal(got, img)


@pytest.mark.parametrize("suffix", [".png", ".tif"])
@pytest.mark.parametrize("compression", ["none", "deflate"])
@pytest.mark.parametrize("shape", [(12, 9), (600, 701)])
def test_rgb_round_trip(tmp_path, suffix, compression, shape):
    if suffix == ".png" and compression == "deflate":
        pytest.skip("compression applies to TIFF only")
    rng = np.random.default_rng(7)
    img = rng.integers(0, 256, size=shape + (3,), dtype=np.uint8)
    img[: shape[0] // 2] = smooth(shape[0] // 2, shape[1], 8, channels=3)
    path = tmp_path / f"color{suffix}"
    ut.save_image(img, path, compression=compression)
    assert np.array_equal(cv2_load(path), img)


@pytest.mark.parametrize("shape", [(20, 30), (1, 1), (1000, 300), (97, 6000)])
@pytest.mark.parametrize("depth", [8, 16])
@pytest.mark.parametrize("compression", ["none", "deflate"])
def test_tiff_gray_round_trip(tmp_path, shape, depth, compression):
    rng = np.random.default_rng(8)
    dt = np.uint8 if depth == 8 else np.uint16
    img = smooth(*shape, depth)
    img[::3] = rng.integers(0, 2 ** depth, size=img[::3].shape).astype(dt)
    path = tmp_path / "g.tif"
    ut.save_image(img, path, compression=compression)
    got = cv2_load(path)
    assert got.dtype == dt and np.array_equal(got, img)


def test_device_tensor_input_and_determinism(tmp_path):
    img = smooth(777, 1234, 8)
    t = torch.from_numpy(img).cuda()
    ut.save_image(t, tmp_path / "a.png")
    ut.save_image(img, tmp_path / "b.png")
    assert (tmp_path / "a.png").read_bytes() == (tmp_path / "b.png").read_bytes()
    ut.save_image(t, tmp_path / "a.tif", compression="deflate")
    ut.save_image(img, tmp_path / "b.tif", compression="deflate")
    assert (tmp_path / "a.tif").read_bytes() == (tmp_path / "b.tif").read_bytes()
    assert np.array_equal(cv2_load(tmp_path / "a.tif"), img)


def test_deflate_compresses(tmp_path):
    img = np.zeros((256, 256), dtype=np.uint8)
    ut.save_image(img, tmp_path / "raw.tif", compression="none")
    ut.save_image(img, tmp_path / "packed.tif", compression="deflate")
    assert (tmp_path / "packed.tif").stat().st_size < (tmp_path / "raw.tif").stat().st_size
    big = smooth(2048, 2048, 8)
    png = image_io.encode_png(big)
    assert len(png) < big.nbytes * 0.6


def test_errors(tmp_path):
    with pytest.raises(ut.DataError, match="format"):
        ut.save_image(np.zeros((2, 2), dtype=np.uint8), tmp_path / "x.jpg")
    with pytest.raises(ut.DataError, match="compression"):
        ut.save_image(np.zeros((2, 2), dtype=np.uint8), tmp_path / "x.tif", compression="lzw")
    with pytest.raises(ut.DataError, match="uint8 or uint16"):
        ut.save_image(np.zeros((2, 2), dtype=np.float32), tmp_path / "x.png")
    with pytest.raises(ut.DataError, match="3 channels"):
        ut.save_image(np.zeros((2, 2, 4), dtype=np.uint8), tmp_path / "x.png")
