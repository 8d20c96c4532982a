"""load_stack / load_image on the device (stack.py:119-177, rendering.py:334-343;
SURVEY §8(f) row 3): TIFF bands -- as the reference's save_image writes them
through cv2 (raw or deflate), as the device encoder writes them, big-endian, LZW
(cv2's default TIFF compression) and tiled -- and PNGs (every scanline filter)
decode on the B200 to exactly what cv2.imread returns; the reference's
load_stack cases (test_stack.py:53-113) hold."""

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


def no_host_codecs(monkeypatch):
    def boom(*args, **kwargs):
        raise AssertionError("host codec called")

    for name in ("imread", "imdecode", "imreadmulti"):
        monkeypatch.setattr(cv2, name, boom)


@pytest.mark.parametrize("shape,dtype", [((1, 1), np.uint8), ((20, 30), np.uint8),
                                         ((513, 1031), np.uint8), ((300, 777), np.uint16),
                                         ((64, 48, 3), np.uint8), ((65, 33, 3), np.uint16),
                                         ((1200, 2000), np.uint16)])
def test_cv2_written_png_decodes_on_device(tmp_path, shape, dtype):
    img = image(shape, dtype, 11)
    path = tmp_path / "a.png"
    cv2_write(path, img)
    want = cv2_read(path)
    assert np.array_equal(want, img)
    t = image_io.decode_png(path.read_bytes())           # the device path, no fallback
    assert t.is_cuda and t.dtype == (torch.uint8 if dtype == np.uint8 else torch.uint16)
    assert np.array_equal(t.cpu().numpy(), want)


def _png_filter_rows(img, kinds):
    """Scanlines of img (H, W[, 3]) filtered with the given per-row filter types
    (PNG specification, section 9), 16-bit samples big endian."""
    h = img.shape[0]
    raw = img.astype(">u2" if img.dtype == np.uint16 else np.uint8).reshape(h, -1).view(np.uint8)
    bpp = raw.shape[1] // img.shape[1]
    out = bytearray()
    prev = np.zeros(raw.shape[1], dtype=np.int32)
    for y in range(h):
        cur = raw[y].astype(np.int32)
        left = np.concatenate([np.zeros(bpp, np.int32), cur[:-bpp]])
        ul = np.concatenate([np.zeros(bpp, np.int32), prev[:-bpp]])
        kind = kinds[y % len(kinds)]
        if kind == 0:
            pred = np.zeros_like(cur)
        elif kind == 1:
            pred = left
        elif kind == 2:
            pred = prev
        elif kind == 3:
            pred = (left + prev) >> 1
        else:
            p = left + prev - ul
            pa, pb, pc = np.abs(p - left), np.abs(p - prev), np.abs(p - ul)
            pred = np.where((pa <= pb) & (pa <= pc), left, np.where(pb <= pc, prev, ul))
        out.append(kind)
        out += ((cur - pred) & 0xFF).astype(np.uint8).tobytes()
        prev = cur
    return bytes(out)


def _png_file(img, kinds, idat_split=1 << 30):
    h, w = img.shape[:2]
    color = 2 if img.ndim == 3 else 0
    depth = 16 if img.dtype == np.uint16 else 8
    chunk = lambda k, d: struct.pack(">I", len(d)) + k + d + struct.pack(">I", zlib.crc32(k + d))  # noqa: E731
    z = zlib.compress(_png_filter_rows(img, kinds), 6)
    idat = b"".join(chunk(b"IDAT", z[i:i + idat_split]) for i in range(0, len(z), idat_split))
    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, color, 0, 0, 0))
            + chunk(b"tEXt", b"Comment\0hand-filtered") + idat + chunk(b"IEND", b""))


@pytest.mark.parametrize("kinds", [[0], [1], [2], [3], [4], [4, 3, 2, 1, 0], [3, 4]])
@pytest.mark.parametrize("shape,dtype", [((70, 45), np.uint8), ((37, 101), np.uint16),
                                         ((40, 67, 3), np.uint8), ((33, 35, 3), np.uint16)])
def test_every_png_filter(tmp_path, kinds, shape, dtype):
    """Hand-filtered PNGs (each scanline filter alone and mixed, rows crossing
    the 32-row wavefront groups, IDAT split over several chunks)."""
    img = image(shape, dtype, 12)
    data = _png_file(img, kinds, idat_split=997)
    got = image_io.decode_png(data).cpu().numpy()
    assert np.array_equal(got, img)
    ref = cv2.imdecode(np.frombuffer(data, np.uint8), cv2.IMREAD_UNCHANGED)
    assert np.array_equal(ref[:, :, ::-1] if ref.ndim == 3 else ref, img)


def test_device_written_png_round_trip(tmp_path):
    for shape, dtype in (((300, 200), np.uint16), ((90, 120, 3), np.uint8)):
        img = image(shape, dtype, 13)
        got = image_io.decode_png(image_io.encode_png(torch.from_numpy(img).cuda()))
        assert np.array_equal(got.cpu().numpy(), img)


def test_corrupt_png_raises():
    img = image((120, 90), np.uint8, 14)
    data = bytearray(_png_file(img, [4]))
    at = data.index(b"IDAT") + 4
    data[at + 20:at + 50] = bytes(30)
    with pytest.raises(ut.DataError, match="CRC"):        # the host's chunk check
        image_io.decode_png(bytes(data))
    (n,) = struct.unpack(">I", data[at - 8:at - 4])        # same damage under a valid CRC:
    data[at + n:at + n + 4] = struct.pack(">I", zlib.crc32(bytes(data[at - 4:at + n])))
    with pytest.raises(ut.DataError, match="undecodable"):  # the device's inflate / Adler-32 check
        image_io.decode_png(bytes(data))
    good = _png_file(img, [0])                     # the same image with a filter byte of 7
    rows = bytearray(_png_filter_rows(img, [0]))
    rows[0] = 7
    chunk = lambda k, d: struct.pack(">I", len(d)) + k + d + struct.pack(">I", zlib.crc32(k + d))  # noqa: E731
    head = good[:good.index(b"IDAT") - 4]
    with pytest.raises(ut.DataError):
        image_io.decode_png(head + chunk(b"IDAT", zlib.compress(bytes(rows))) + chunk(b"IEND", b""))


@pytest.mark.parametrize("shape,dtype", [((1, 1), np.uint8), ((20, 30), np.uint8),
                                         ((513, 1031), np.uint8), ((300, 777), np.uint16),
                                         ((64, 48, 3), np.uint8), ((1200, 2000), np.uint16)])
def test_cv2_written_lzw_tiff_decodes_on_device(tmp_path, shape, dtype):
    """cv2.imwrite's default TIFF compression is LZW (with Predictor 2)."""
    img = image(shape, dtype, 15)
    path = tmp_path / "lzw.tif"
    payload = np.ascontiguousarray(img[:, :, ::-1]) if img.ndim == 3 else img
    assert cv2.imwrite(str(path), payload, [cv2.IMWRITE_TIFF_COMPRESSION, 5])
    assert image_io._tiff_layout(path.read_bytes())["compression"] == 5
    got = image_io.decode_tiff(path.read_bytes())
    assert np.array_equal(got.cpu().numpy(), cv2_read(path))
    assert np.array_equal(got.cpu().numpy(), img)


def test_lzw_flat_image_with_long_strings(tmp_path):
    """Constant and periodic data: long table strings, KwKwK codes, table resets."""
    for k, img in enumerate((np.full((700, 900), 37, np.uint8),
                             np.tile(np.arange(251, dtype=np.uint8), (400, 5)),
                             np.zeros((300, 4000), np.uint16))):
        path = tmp_path / f"flat{k}.tif"
        assert cv2.imwrite(str(path), img, [cv2.IMWRITE_TIFF_COMPRESSION, 5])
        assert np.array_equal(image_io.decode_tiff(path.read_bytes()).cpu().numpy(), img)


def _tiled_tiff(img, tw, th, compression, predictor=1, big_endian=False):
    """A tiled classic TIFF written by hand (raw or zlib tiles, edge tiles padded)."""
    bo = ">" if big_endian else "<"
    h, w = img.shape[:2]
    ch = 3 if img.ndim == 3 else 1
    depth = 16 if img.dtype == np.uint16 else 8
    across, down = -(-w // tw), -(-h // th)
    tiles = []
    for ty in range(down):
        for tx in range(across):
            tile = np.zeros((th, tw) + img.shape[2:], dtype=img.dtype)
            part = img[ty * th:(ty + 1) * th, tx * tw:(tx + 1) * tw]
            tile[:part.shape[0], :part.shape[1]] = part
            if predictor == 2:
                t2 = tile.reshape(th, tw, ch).copy()
                t2[:, 1:] = t2[:, 1:] - t2[:, :-1]
                tile = t2
            raw = tile.astype(tile.dtype.newbyteorder(bo)).tobytes()
            tiles.append(zlib.compress(raw) if compression == 8 else raw)
    body = b"".join(t + b"\0" * (len(t) & 1) for t in tiles)
    offs, at = [], 8
    for t in tiles:
        offs.append(at)
        at += len(t) + (len(t) & 1)
    ifd_at = 8 + len(body)
    entries = [(256, 4, [w]), (257, 4, [h]), (258, 3, [depth] * ch), (259, 3, [compression]),
               (262, 3, [2 if ch == 3 else 1]), (277, 3, [ch]), (284, 3, [1]), (317, 3, [predictor]),
               (322, 4, [tw]), (323, 4, [th]), (324, 4, offs), (325, 4, [len(t) for t in tiles])]
    extra_at = ifd_at + 2 + 12 * len(entries) + 4
    ifd, extra = struct.pack(bo + "H", len(entries)), b""
    for tag, typ, vals in entries:
        raw = struct.pack(bo + ("H" if typ == 3 else "I") * len(vals), *vals)
        if len(raw) <= 4:
            ifd += struct.pack(bo + "HHI", tag, typ, len(vals)) + raw.ljust(4, b"\0")
        else:
            ifd += struct.pack(bo + "HHII", tag, typ, len(vals), extra_at + len(extra))
            extra += raw + b"\0" * (len(raw) & 1)
    ifd += struct.pack(bo + "I", 0)
    return (b"MM\0*" if big_endian else b"II*\0") + struct.pack(bo + "I", ifd_at) + body + ifd + extra


@pytest.mark.parametrize("compression,predictor,big", [(1, 1, False), (8, 1, False), (8, 2, False), (8, 2, True)])
@pytest.mark.parametrize("shape,dtype,tile", [((100, 130), np.uint8, (64, 32)), ((257, 300), np.uint16, (128, 128)),
                                              ((70, 90, 3), np.uint8, (32, 48)), ((16, 16), np.uint16, (16, 16))])
def test_tiled_tiff_decodes_on_device(tmp_path, compression, predictor, big, shape, dtype, tile):
    img = image(shape, dtype, 16)
    data = _tiled_tiff(img, tile[0], tile[1], compression, predictor, big)
    path = tmp_path / "tiled.tif"
    path.write_bytes(data)
    assert np.array_equal(cv2_read(path), img)            # libtiff agrees the file is valid
    got = image_io.decode_tiff(data)
    assert got.is_cuda and np.array_equal(got.cpu().numpy(), img)


def test_files_decode_without_the_host_decoder(tmp_path, monkeypatch):
    """PNG, LZW and tiled TIFF inputs never reach cv2 (the reference's decoder)."""
    img = image((90, 120), np.uint16, 17)
    cv2.imwrite(str(tmp_path / "a.png"), img)
    cv2.imwrite(str(tmp_path / "lzw.tif"), img, [cv2.IMWRITE_TIFF_COMPRESSION, 5])
    (tmp_path / "tiled.tif").write_bytes(_tiled_tiff(img, 64, 64, 8, 2))
    no_host_codecs(monkeypatch)
    for name in ("a.png", "lzw.tif", "tiled.tif"):
        assert np.array_equal(ut.load_image(tmp_path / name), img)
    m = _manifest(tmp_path, ["a.png,365,uv", "lzw.tif,450,vis", "tiled.tif,940,ir"])
    stack = ut.load_stack(m)
    assert stack.planes.shape == (3, 90, 120) and stack.bit_depth == 16
    assert all(np.array_equal(stack.planes[b], img) for b in range(3))


def test_other_layouts_use_the_reference_decoder(tmp_path):
    """Layouts the device decoders do not parse (alpha channels, float samples,
    ...) are read by cv2 exactly as the reference reads them."""
    rgba = np.dstack([image((40, 50, 3), np.uint8, 5), np.full((40, 50), 200, np.uint8)])
    cv2.imwrite(str(tmp_path / "rgba.png"), rgba)
    with pytest.raises(image_io._Unsupported):
        image_io.decode_png((tmp_path / "rgba.png").read_bytes())
    with pytest.raises(ut.DataError, match="expected 3 channels, got 4"):
        ut.load_image(tmp_path / "rgba.png")
    cv2.imwrite(str(tmp_path / "f.tif"), image((40, 50), np.uint8, 6).astype(np.float32))
    with pytest.raises(image_io._Unsupported):
        image_io.decode_tiff((tmp_path / "f.tif").read_bytes())
    with pytest.raises(ut.DataError):
        ut.load_image(tmp_path / "f.tif")
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
    """The measured path -- the cube resident in HBM, fit, projection, stretch, as
    bench.py times it (CVA, the PCA companion and the streamed folio batch) -- must
    never reach a host codec: every cv2 entry point is made to fail here."""
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


def test_decoders_fuzz_vs_cv2():
    """Seeded random images (noise, flat, smooth, periodic rows; gray / RGB, 8 / 16 bit)
    through every container cv2 writes and the device reads; iterations 22, 26 and 44
    of this sequence are streams whose literal runs empty the inflate's bit buffer
    exactly (a refill then holds 32 bits, one short of three 11-bit codes) -- the
    case a first version of the warp decoder got wrong."""
    rng = np.random.default_rng(12345)
    checked = 0
    for it in range(60):
        h, w = int(rng.integers(1, 300)), int(rng.integers(1, 700))
        ch = int(rng.choice([1, 3]))
        dt = rng.choice([np.uint8, np.uint16])
        top = np.iinfo(dt).max
        kind = rng.integers(0, 4)
        shape = (h, w) if ch == 1 else (h, w, 3)
        if kind == 0:
            img = rng.integers(0, top + 1, size=shape).astype(dt)
        elif kind == 1:
            img = np.full(shape, rng.integers(0, top + 1), dtype=dt)
        elif kind == 2:
            y, x = np.mgrid[0:h, 0:w]
            base = (np.sin(x / 9.0) + np.cos(y / 7.0) + 2) / 4 * top
            img = (base if ch == 1 else base[..., None] * np.array([1, .5, .25])).astype(dt)
        else:
            img = np.tile(rng.integers(0, top + 1, size=(1, int(rng.integers(1, 40))) + shape[2:]).astype(dt),
                          (h, w // 1 + 1) + (1,) * (len(shape) - 2))[:, :w]
            img = np.ascontiguousarray(img.reshape(shape))
        payload = np.ascontiguousarray(img[:, :, ::-1]) if ch == 3 else img
        for ext, params in ((".png", []), (".png", [cv2.IMWRITE_PNG_COMPRESSION, int(rng.integers(0, 10))]),
                            (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 5]), (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 8]),
                            (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 1])):
            ok, buf = cv2.imencode(ext, payload, params)
            assert ok
            got = image_io.decode_batch([buf.tobytes()])[0].cpu().numpy()
            assert got.dtype == img.dtype and np.array_equal(got, img), (it, ext, params, shape, kind)
            checked += 1
        t = torch.from_numpy(img).cuda()
        for data in (image_io.encode_png(t), image_io.encode_tiff(t, "deflate")):
            assert np.array_equal(image_io.decode_batch([data])[0].cpu().numpy(), img), (it, shape)
            checked += 1
    assert checked == 60 * 7
