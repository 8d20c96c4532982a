"""Random cubes through K2 (fit_pca_unsupervised on whole images and whole-width regions):
17-32 bands (int8 tensor-core path) and fewer (fp64 tensor-core path), every dtype, value
distributions that stress the fixed-point grid (large offsets, tiny spreads, outliers that
must fall back to fp64, constant bands), against the oracle
(dev tool; python tools/fuzz/fuzz_region.py [seed])."""
import sys, traceback, warnings
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch
import oracle
from golden_util import rel_close
import paper_1612_06457_b200 as ut
warnings.simplefilter("ignore")
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
fails = 0
def tonp(x): return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
for it in range(150):
    try:
        b = int(rng.integers(1, 33)); h = int(rng.integers(4, 400)); w = int(rng.integers(4, 600))
        kind = it % 6
        mix = rng.normal(size=(b, b)) / np.sqrt(b)
        z = np.einsum('ij,jhw->ihw', mix, rng.normal(size=(b, h, w)))
        if kind == 0: x, dt = 0.5 + 0.05 * z, np.float32
        elif kind == 1: x, dt = 1000.0 + 0.001 * z, np.float32                 # big offset, tiny spread
        elif kind == 2:
            x, dt = 0.5 + 0.05 * z, np.float32
            x.reshape(b, -1)[:, rng.integers(0, h * w, size=3)] = 1e6            # outliers -> fp64 fallback
        elif kind == 3: x, dt = np.clip(np.floor(2000 + 300 * z), 0, 4095), np.uint16
        elif kind == 4: x, dt = np.clip(np.floor(128 + 40 * z), 0, 255), np.uint8
        else: x, dt = 0.5 + 0.1 * z, np.float16
        if it % 7 == 0 and b > 1: x[0] = x[0].flat[0]                             # a constant band
        cube = np.ascontiguousarray(x.astype(dt))
        depth = 16 if dt == np.uint16 else 8
        ds = ut.DeviceStack(ut.stack.default_bands(b), torch.from_numpy(cube).cuda(), depth, True)
        y0 = int(rng.integers(0, h - 1)) if it % 2 else 0
        rh = int(rng.integers(2, h - y0 + 1)) if it % 2 else h
        region = (0, y0, w, rh)
        k = min(3, b)
        pm = ut.fit_pca_unsupervised(ds, region=region, k=k)
        rp = oracle.fit_pca_unsupervised(cube, region=region, k=k)
        case = (it, b, h, w, kind, region, np.dtype(dt).name)
        assert rel_close(tonp(pm.mean), rp["mean"], 1e-9), ("mean",) + case
        assert rel_close(tonp(pm.std), rp["std"], 1e-9), ("std",) + case
        le = np.asarray(rp["eigenvalues"])
        assert np.all(np.abs(tonp(pm.eigenvalues) - le) <= 1e-9 * (le.max() + np.abs(le))), ("evals",) + case
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:260], flush=True)
print("fuzz region done, fails:", fails)
