"""Random shapes / dtypes / class counts / point orders through the CVA path (fit, planes,
codes) and the PCA fit, against the oracle (dev tool; python tools/fuzz/fuzz_path.py [seed] [n]).
A seeded prefix runs in tests/test_gpu_edges.py."""
import sys
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch
import oracle
from golden_util import align_signs, plane_close, rel_close
import paper_1612_06457_b200 as ut
from test_gpu_edges import cube_of, device_stack, pick_points, DTYPES
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 2024)
fails = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 150):
    b = int(rng.integers(1, 33)); classes = int(rng.integers(2, 9))
    h = int(rng.integers(8, 200)); w = int(rng.integers(8, 400))
    dtype = DTYPES[int(rng.integers(0, len(DTYPES)))]
    cube, cmap = cube_of(rng, b, h, w, dtype, classes=classes)
    per = int(rng.integers(max(3, b // classes + 2), 120))
    xs, ys, ls = pick_points(rng, cmap, per)
    if len(np.unique(ls)) < 2:
        continue
    perm = rng.permutation(len(ls)) if it % 2 else np.arange(len(ls))
    xs, ys, ls = xs[perm], ys[perm], ls[perm]
    k = int(rng.integers(1, min(b, len(np.unique(ls)) - 1) + 1))
    try:
        ds = device_stack(cube)
        pipe = ut.CvaPipeline(ds, xs, ys, ls, k=k)
        codes = pipe.run().cpu().numpy()
        hst = pipe.check()
        ref = oracle.fit_cva(oracle.assemble(cube, xs, ys), ls, k=k)
        sp = ref["scatter"]
        assert np.array_equal(hst["counts"].astype(int), sp["counts"]), "counts"
        assert rel_close(hst["within"], sp["within"], 1e-9), "within"
        assert rel_close(hst["between"], sp["between"], 1e-9), "between"
        lam = np.asarray(ref["eigenvalues"]); sig = lam > 1e-6 * lam.max()
        assert np.all(np.abs(hst["evals"][:k][sig] - lam[sig]) <= 1e-9 * np.abs(lam[sig])), "evals"
        # projection of the device model, checked with the oracle projector
        m = pipe.model()
        want = oracle.project(cube, {"mean": m.mean, "std": None, "coefficients": m.coefficients})
        got = pipe.scores.double().cpu().numpy()
        assert plane_close(got, want) <= 1e-6, ("planes", plane_close(got, want))
        for j in range(k):
            assert np.array_equal(codes[j], oracle.rescale_full(pipe.scores[j].double().cpu().numpy())), "codes"
        # PCA on the same cube
        pm = ut.fit_pca_unsupervised(ds, k=min(3, b))
        rp = oracle.fit_pca_unsupervised(cube, k=min(3, b))
        assert rel_close(pm.mean, rp["mean"], 1e-9), "pca mean"
        le = np.asarray(rp["eigenvalues"]); 
        assert np.all(np.abs(np.asarray(pm.eigenvalues) - le) <= 1e-9 * max(le.max(), 1e-300) + 1e-9 * np.abs(le)), "pca evals"
    except Exception as e:
        fails += 1
        print("FAIL", it, dict(b=b, classes=classes, h=h, w=w, dtype=dtype.__name__, per=per, k=k, shuffled=bool(it % 2)), repr(e)[:200], flush=True)
print("fuzz path done, fails:", fails)
