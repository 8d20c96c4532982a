"""Strided views (crops of a larger cube: row stride != width, misaligned starts) through the
CVA path and the PCA fit, against the oracle on the contiguous copy
(dev tool; python tools/fuzz/fuzz_views.py [seed])."""
import sys, traceback
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch
import oracle
from golden_util import plane_close, rel_close
import paper_1612_06457_b200 as ut
from test_gpu_edges import cube_of, pick_points, DTYPES
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 71)
fails = done = 0
def tonp(x): return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
for it in range(120):
    try:
        b = int(rng.integers(1, 33)); classes = int(rng.integers(2, 6))
        H = int(rng.integers(12, 200)); W = int(rng.integers(12, 300))
        dtype = DTYPES[int(rng.integers(0, len(DTYPES)))]
        full, cmap_full = cube_of(rng, b, H, W, dtype, classes=classes)
        y0 = int(rng.integers(0, H - 8)); x0 = int(rng.integers(0, W - 8))
        h = int(rng.integers(8, H - y0 + 1)); w = int(rng.integers(8, W - x0 + 1))
        dev = torch.from_numpy(full).cuda()
        view = dev[:, y0:y0 + h, x0:x0 + w]                      # not contiguous unless w == W
        cube = np.ascontiguousarray(full[:, y0:y0 + h, x0:x0 + w])
        cmap = cmap_full[y0:y0 + h, x0:x0 + w]
        xs, ys, ls = pick_points(rng, cmap, b + 10)
        if len(np.unique(ls)) < 2:
            continue
        k = int(rng.integers(1, min(b, len(np.unique(ls)) - 1) + 1))
        depth = 16 if dtype == np.uint16 else 8
        ds = ut.DeviceStack(ut.stack.default_bands(b), view, depth, True)
        pipe = ut.CvaPipeline(ds, xs, ys, ls, k=k)
        codes = pipe.run().cpu().numpy()
        hst = pipe.check()
        ref = oracle.fit_cva(oracle.assemble(cube, xs, ys), ls, k=k)
        sp = ref["scatter"]
        case = (it, b, (H, W), (y0, x0, h, w), dtype.__name__, k)
        assert np.array_equal(hst["counts"].astype(int), sp["counts"]), ("counts",) + case
        assert rel_close(hst["within"], sp["within"], 1e-9), ("within",) + case
        m = pipe.model()
        want = oracle.project(cube, {"mean": m.mean, "std": None, "coefficients": m.coefficients})
        assert plane_close(tonp(pipe.scores.double()), want) <= 1e-6, ("planes",) + case
        for j in range(k):
            assert np.array_equal(codes[j], oracle.rescale_full(tonp(pipe.scores[j].double()))), ("codes",) + case
        pm = ut.fit_pca_unsupervised(ds, k=min(3, b))
        rp = oracle.fit_pca_unsupervised(cube, k=min(3, b))
        assert rel_close(tonp(pm.mean), rp["mean"], 1e-9), ("pca mean",) + case
        le = np.asarray(rp["eigenvalues"])
        assert np.all(np.abs(tonp(pm.eigenvalues) - le) <= 1e-9 * (le.max() + np.abs(le))), ("pca evals",) + case
        done += 1
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:260], traceback.format_exc().splitlines()[-3][:140], flush=True)
print("fuzz views done:", done, "cases, fails:", fails)
