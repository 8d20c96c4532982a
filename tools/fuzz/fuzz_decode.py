"""Random images through every container cv2 / the device encoders write and the device
decoders read, compared with the input (dev tool; python tools/fuzz/fuzz_decode.py [seed]).
A seeded prefix of the same sequence runs in tests/test_gpu_decode.py."""
import sys, zlib
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np, cv2, torch
from paper_1612_06457_b200 import image_io
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 12345)
n_ok = 0
for it in range(400):
    h = int(rng.integers(1, 300)); w = int(rng.integers(1, 700))
    ch = int(rng.choice([1, 3])); dt = rng.choice([np.uint8, np.uint16])
    top = np.iinfo(dt).max
    kind = rng.integers(0, 4)
    shape = (h, w) if ch == 1 else (h, w, 3)
    if kind == 0:
        img = rng.integers(0, top + 1, size=shape).astype(dt)                      # noise
    elif kind == 1:
        img = np.full(shape, rng.integers(0, top + 1), dtype=dt)                  # flat
    elif kind == 2:
        y, x = np.mgrid[0:h, 0:w]
        base = ((np.sin(x / 9.0) + np.cos(y / 7.0) + 2) / 4 * top)
        img = (base if ch == 1 else base[..., None] * np.array([1, .5, .25])).astype(dt)   # smooth
    else:
        img = np.tile(rng.integers(0, top + 1, size=(1, int(rng.integers(1, 40))) + shape[2:]).astype(dt),
                      (h, w // 1 + 1) + (1,) * (len(shape) - 2))[:, :w]          # periodic rows
        img = np.ascontiguousarray(img.reshape(shape))
    payload = np.ascontiguousarray(img[:, :, ::-1]) if ch == 3 else img
    for ext, params in ((".png", []), (".png", [cv2.IMWRITE_PNG_COMPRESSION, int(rng.integers(0, 10))]),
                        (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 5]), (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 8]),
                        (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 1])):
        ok, buf = cv2.imencode(ext, payload, params)
        assert ok
        data = buf.tobytes()
        try:
            got = image_io.decode_batch([data])[0].cpu().numpy()
            assert got.dtype == img.dtype and np.array_equal(got, img)
            n_ok += 1
        except Exception as e:
            print("FAIL", it, ext, params, shape, dt, kind, repr(e)[:120], flush=True)
            open(f"fuzz_fail_{it}{ext}", "wb").write(data)
            np.save(f"fuzz_fail_{it}.npy", img)
# batches of mixed files
datas, imgs = [], []
for it in range(40):
    h = int(rng.integers(1, 200)); w = int(rng.integers(1, 300))
    img = rng.integers(0, 4096, size=(h, w)).astype(np.uint16)
    ext, params = [(".png", []), (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 5]), (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 8])][it % 3]
    datas.append(cv2.imencode(ext, img, params)[1].tobytes()); imgs.append(img)
for got, img in zip(image_io.decode_batch(datas), imgs):
    assert np.array_equal(got.cpu().numpy(), img)
# device-encoded files back through the device decoders
for it in range(60):
    h = int(rng.integers(1, 300)); w = int(rng.integers(1, 500)); ch = int(rng.choice([1, 3]))
    dt = rng.choice([np.uint8, np.uint16])
    shape = (h, w) if ch == 1 else (h, w, 3)
    y, x = np.mgrid[0:h, 0:w]
    base = ((np.sin(x / 9.0) + np.cos(y / 7.0) + 2) / 4 * np.iinfo(dt).max)
    img = (base if ch == 1 else base[..., None] * np.array([1, .5, .25])).astype(dt)
    img = (img + rng.integers(0, 3, size=shape)).astype(dt)
    t = torch.from_numpy(img).cuda()
    for data in (image_io.encode_png(t), image_io.encode_tiff(t, "deflate"), image_io.encode_tiff(t, "none")):
        assert np.array_equal(image_io.decode_batch([data])[0].cpu().numpy(), img), (it, shape, dt)
        n_ok += 1
print("fuzz ok:", n_ok, "single files + 40-file mixed batch")
