"""Hand-built containers through the device decoders: PNGs with random per-row filter
sequences and IDAT splits, tiled TIFFs with random tile sizes / compression / predictor /
byte order, compared with the input and with cv2 (dev tool; python tools/fuzz/fuzz_containers.py [seed])."""
import sys, traceback
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, cv2
from paper_1612_06457_b200 import image_io
from test_gpu_decode import _png_file, _tiled_tiff, image
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 41)
fails = 0
for it in range(250):
    try:
        h = int(rng.integers(1, 200)); w = int(rng.integers(1, 300)); ch = int(rng.choice([1, 3]))
        dt = rng.choice([np.uint8, np.uint16])
        shape = (h, w) if ch == 1 else (h, w, 3)
        img = image(shape, dt, int(rng.integers(0, 1 << 30)))
        kinds = [int(v) for v in rng.integers(0, 5, size=int(rng.integers(1, 12)))]
        data = _png_file(img, kinds, idat_split=int(rng.choice([64, 997, 8192, 1 << 30])))
        got = image_io.decode_png(data).cpu().numpy()
        assert got.dtype == img.dtype and np.array_equal(got, img), ("png", shape, dt, kinds)
        tw, th = 16 * int(rng.integers(1, 9)), 16 * int(rng.integers(1, 9))
        comp, pred = [(1, 1), (8, 1), (8, 2)][int(rng.integers(0, 3))]
        big = bool(rng.integers(0, 2))
        data = _tiled_tiff(img, tw, th, comp, pred, big)
        got = image_io.decode_tiff(data).cpu().numpy()
        assert np.array_equal(got, img), ("tiled", shape, dt, tw, th, comp, pred, big)
        ref = cv2.imdecode(np.frombuffer(data, np.uint8), cv2.IMREAD_UNCHANGED)
        if ref is not None:   # cv2's TIFF reader refuses some valid tile geometries
            ref = ref[:, :, ::-1] if ref.ndim == 3 else ref
            assert np.array_equal(ref, img), ("tiled file invalid for libtiff", shape, tw, th, comp, pred, big)
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:240], traceback.format_exc().splitlines()[-3][:140], flush=True)
print("fuzz containers done, fails:", fails)
