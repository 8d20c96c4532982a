"""load_stack / load_image on the device (stack.py:119-177, rendering.py:334-343;
SURVEY §8(f) row 3): stripped TIFF bands -- as the reference's save_image
writes them through cv2 (raw or deflate), as the device encoder writes them, and
big-endian -- decode on the B200 to exactly what cv2.imread returns; the
reference's load_stack cases (test_stack.py:53-113) hold."""

import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
cv2 = pytest.importorskip("cv2")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import image_io  # noqa: E402

REF_TIFF = {"none": 1, "deflate": 8}  # rendering.py:300


def cv2_write(path, img, compression="none"):
    """The reference's save_image for TIFF: cv2.imwrite with its compression tag."""
    payload = np.ascontiguousarray(img[:, :, ::-1]) if img.ndim == 3 else img
    params = [cv2.IMWRITE_TIFF_COMPRESSION, REF_TIFF[compression]] if str(path).endswith(".tif") else []
    assert cv2.imwrite(str(path), payload, params)


def cv2_read(path):
    img = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    return np.ascontiguousarray(img[:, :, ::-1]) if img.ndim == 3 else img


def image(shape, dtype, seed):
    rng = np.random.default_rng(seed)
    top = np.iinfo(dtype).max
    y, x = np.mgrid[0:shape[0], 0:shape[1]]
    base = (np.sin(x / 17.0) + np.cos(y / 11.0) + 2) / 4 * top
    if len(shape) == 3:
        base = base[..., None] * np.array([1.0, 0.7, 0.4])
    img = np.clip(base + rng.normal(0, top * 0.01, size=shape), 0, top).astype(dtype)
    img.reshape(-1)[::7] = rng.integers(0, top, size=img.reshape(-1)[::7].shape).astype(dtype)
    return img


@pytest.mark.parametrize("compression", ["none", "deflate"])
@pytest.mark.parametrize("shape,dtype", [((1, 1), np.uint8), ((20, 30), np.uint8),
                                         ((513, 1031), np.uint8), ((300, 777), np.uint16),
                                         ((64, 48, 3), np.uint8), ((1200, 2000), np.uint16)])
def test_cv2_written_tiff_decodes_on_device(tmp_path, compression, shape, dtype):
    img = image(shape, dtype, 1)
    path = tmp_path / "band.tif"
    cv2_write(path, img, compression)
    t = image_io.decode_tiff(path.read_bytes())          # the device path, no fallback
    assert t.is_cuda
    got = t.cpu().numpy()
    assert got.dtype == dtype and np.array_equal(got, cv2_read(path))
    assert np.array_equal(ut.load_image(path), img)


@pytest.mark.parametrize("compression", ["none", "deflate"])
@pytest.mark.parametrize("shape,dtype", [((7, 5), np.uint8), ((1000, 333), np.uint16),
                                         ((37, 41, 3), np.uint8)])
def test_device_written_tiff_round_trip(tmp_path, compression, shape, dtype):
    img = image(shape, dtype, 2)
    path = tmp_path / "dev.tif"
    ut.save_image(img, path, compression=compression)
    got = image_io.decode_tiff(path.read_bytes()).cpu().numpy()
    assert np.array_equal(got, img)


def test_big_endian_and_predictor(tmp_path):
    """Hand-built 'MM' TIFF, 16-bit, raw strips, two strips."""
    rng = np.random.default_rng(3)
    img = rng.integers(0, 65535, size=(9, 6)).astype(np.uint16)
    body = img.astype(">u2").tobytes()
    h, w = img.shape
    entries = [(256, 4, 1, w), (257, 4, 1, h), (258, 3, 1, 16), (259, 3, 1, 1), (262, 3, 1, 1),
               (273, 4, 2, None), (277, 3, 1, 1), (278, 4, 1, 5), (279, 4, 2, None)]
    ifd_at = 8 + len(body)
    extra_at = ifd_at + 2 + 12 * len(entries) + 4
    offsets = struct.pack(">II", 8, 8 + 5 * w * 2)
    counts = struct.pack(">II", 5 * w * 2, 4 * w * 2)
    ifd = struct.pack(">H", len(entries))
    for tag, typ, count, val in entries:
        if tag == 273:
            ifd += struct.pack(">HHII", tag, typ, count, extra_at)
        elif tag == 279:
            ifd += struct.pack(">HHII", tag, typ, count, extra_at + 8)
        elif typ == 3:
            ifd += struct.pack(">HHIHH", tag, typ, count, val, 0)
        else:
            ifd += struct.pack(">HHII", tag, typ, count, val)
    ifd += struct.pack(">I", 0)
    data = b"MM\x00\x2a" + struct.pack(">I", ifd_at) + body + ifd + offsets + counts
    path = tmp_path / "be.tif"
    path.write_bytes(data)
    assert np.array_equal(image_io.decode_tiff(data).cpu().numpy(), img)
    assert np.array_equal(cv2_read(path), img)


def test_corrupt_strip_raises(tmp_path):
    img = image((300, 400), np.uint8, 4)
    path = tmp_path / "c.tif"
    cv2_write(path, img, "deflate")
    data = bytearray(path.read_bytes())
    lay = image_io._tiff_layout(bytes(data))
    off = lay["offsets"][0]
    data[off + 10:off + 40] = bytes(30)     # damage the first strip's stream
    with pytest.raises(ut.DataError):
        image_io.decode_tiff(bytes(data))


def test_png_and_unsupported_layouts_use_the_reference_decoder(tmp_path):
    img = image((40, 50), np.uint8, 5)
    cv2.imwrite(str(tmp_path / "a.png"), img)
    assert np.array_equal(ut.load_image(tmp_path / "a.png"), img)
    cv2.imwrite(str(tmp_path / "lzw.tif"), img, [cv2.IMWRITE_TIFF_COMPRESSION, 5])
    with pytest.raises(image_io._Unsupported):
        image_io.decode_tiff((tmp_path / "lzw.tif").read_bytes())
    assert np.array_equal(ut.load_image(tmp_path / "lzw.tif"), img)
    with pytest.raises(ut.DataError):
        ut.load_image(tmp_path / "absent.png")


def _manifest(d, lines):
    p = d / "manifest.txt"
    p.write_text("\n".join(lines) + "\n", encoding="utf-8")
    return p


class TestLoadStack:
    """The reference's TestLoadStack (test_stack.py:53-113) on the device path."""

    def test_loads_bands_in_manifest_order(self, tmp_path):
        rng = np.random.default_rng(0)
        arrays = [rng.integers(0, 256, size=(8, 10), dtype=np.uint8) for _ in range(3)]
        for i, arr in enumerate(arrays):
            cv2_write(tmp_path / f"b{i}.tif", arr)
        stack = ut.load_stack(_manifest(tmp_path, ["# acquisition comment", "b0.tif,365,uv",
                                                   "b1.tif,500,visible,longpass",
                                                   "b2.tif,940,infrared"]))
        assert stack.band_count == 3 and (stack.width, stack.height) == (10, 8)
        assert stack.bands[1].filter == "longpass"
        assert stack.bands[2].illumination == "infrared"
        for i, arr in enumerate(arrays):
            assert np.array_equal(stack.planes[i], arr)
        assert ut.stack.on_device(stack).planes.is_cuda   # the decoded HBM copy is reused

    def test_single_band_and_16_bit_deflate(self, tmp_path):
        img = image((333, 517), np.uint16, 6)
        cv2_write(tmp_path / "only.tif", img, "deflate")
        stack = ut.load_stack(_manifest(tmp_path, ["only.tif,365,uv"]))
        assert stack.band_count == 1 and stack.bit_depth == 16
        assert np.array_equal(stack.planes[0], img)

    def test_errors(self, tmp_path):
        cv2_write(tmp_path / "a.tif", np.zeros((8, 10), dtype=np.uint8))
        cv2_write(tmp_path / "b.tif", np.zeros((8, 9), dtype=np.uint8))
        with pytest.raises(ut.DataError, match="band 1"):
            ut.load_stack(_manifest(tmp_path, ["a.tif,365,uv", "b.tif,400,uv"]))
        cv2_write(tmp_path / "c.tif", np.zeros((8, 10), dtype=np.uint16))
        with pytest.raises(ut.DataError, match=r"16-bit plane in a 8-bit stack"):
            ut.load_stack(_manifest(tmp_path, ["a.tif,365,uv", "c.tif,400,uv"]))
        cv2.imwrite(str(tmp_path / "rgb.png"), np.zeros((4, 4, 3), dtype=np.uint8))
        with pytest.raises(ut.DataError, match="channel"):
            ut.load_stack(_manifest(tmp_path, ["rgb.png,365,uv"]))


def test_measured_path_never_uses_host_codecs(monkeypatch):
    """PNG, LZW and tiled TIFFs are decoded by cv2 exactly as the reference
    reads them (outside the measured path).  The measured path
    -- the cube resident in HBM, fit, projection, stretch, as bench.py times it
    (CVA, the PCA companion and the streamed folio batch) -- must never reach a
    host codec: every cv2 entry point is made to fail here."""
    from dataclasses import replace

    import cv2

    from paper_1612_06457_b200 import synthetic

    def boom(*args, **kwargs):
        raise AssertionError("host codec called on the measured path")

    for name in ("imread", "imdecode", "imwrite", "imencode", "imreadmulti"):
        monkeypatch.setattr(cv2, name, boom)
    cfg = synthetic.scaled(synthetic.CONFIGS["cfg4"], 128, 96, per_class=40)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k).run()
    ut.PcaPipeline(stack, k=cfg.k).run()
    base = synthetic.scaled(synthetic.CONFIGS["cfg5"], 64, 48, 20)
    cubes, train, outs = [], [], []
    for f in range(2):
        sc = synthetic.make_scene(replace(base, seed=5 + f))
        cubes.append(synthetic.generate(sc).planes.cpu().pin_memory())
        arrs = ut.CvaPipeline.training_arrays(sc.xs, sc.ys, sc.labels)
        train.append(tuple(torch.from_numpy(a).pin_memory() for a in arrs))
        outs.append(torch.empty((base.k, base.height, base.width), dtype=torch.uint8,
                                pin_memory=True))
    fs = ut.FolioStream(cubes, train, outs, k=base.k)
    fs.run()
    torch.cuda.synchronize()
    fs.check()
