"""Corrupted files through the device decoders: random byte flips / truncations of valid
PNG and TIFF files must end in DataError (or in a correct decode when the damage misses the
payload) -- never in a CUDA fault (dev tool; run under `timeout`;
python tools/fuzz/fuzz_corrupt.py [seed])."""
import sys, traceback
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, cv2, torch
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import image_io
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 61)
stats = {"error": 0, "same": 0, "different": 0, "unsupported": 0}
for it in range(400):
    h = int(rng.integers(1, 120)); w = int(rng.integers(1, 200)); ch = int(rng.choice([1, 3]))
    dt = rng.choice([np.uint8, np.uint16]); top = np.iinfo(dt).max
    shape = (h, w) if ch == 1 else (h, w, 3)
    y, x = np.mgrid[0:h, 0:w]
    base = (np.sin(x / 9.0) + np.cos(y / 7.0) + 2) / 4 * top
    img = (base if ch == 1 else base[..., None] * np.array([1, .5, .25]))
    img = np.clip(img + rng.normal(0, top * 0.01, size=shape), 0, top).astype(dt)
    ext, params = [(".png", []), (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 5]), (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 8]),
                   (".tif", [cv2.IMWRITE_TIFF_COMPRESSION, 1])][it % 4]
    data = bytearray(cv2.imencode(ext, np.ascontiguousarray(img[:, :, ::-1]) if ch == 3 else img, params)[1].tobytes())
    mode = it % 3
    if mode == 0:
        for _ in range(int(rng.integers(1, 6))):
            data[int(rng.integers(0, len(data)))] ^= int(rng.integers(1, 256))
    elif mode == 1:
        a = int(rng.integers(0, len(data))); n = int(rng.integers(1, 64))
        data[a:a + n] = bytes(rng.integers(0, 256, size=len(data[a:a + n]), dtype=np.uint8))
    else:
        data = data[: int(rng.integers(8, len(data)))]
    try:
        got = image_io.decode_batch([bytes(data)])[0].cpu().numpy()
        stats["same" if got.shape == img.shape and np.array_equal(got, img) else "different"] += 1
    except ut.DataError:
        stats["error"] += 1
    except image_io._Unsupported:
        stats["unsupported"] += 1
    except Exception as e:   # struct.error etc. from a damaged header: report
        print("UNEXPECTED", it, ext, mode, repr(e)[:160], traceback.format_exc().splitlines()[-3][:140], flush=True)
        stats.setdefault("unexpected", 0); stats["unexpected"] += 1
torch.cuda.synchronize()
print("fuzz corrupt done:", stats)
