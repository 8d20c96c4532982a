"""Random problems through the eigen-solver, LDA / supervised PCA fits and the device
encoders, against the oracle and cv2 (dev tool; python tools/fuzz/fuzz_solvers.py [seed])."""
import sys, traceback, warnings
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch, cv2
import oracle
from golden_util import align_signs, rel_close
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import image_io
warnings.simplefilter("ignore")
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
fails = 0
for it in range(300):
    try:
        # generalized symmetric eigenproblem
        n = int(rng.integers(1, 33))
        q = rng.normal(size=(n, n + 3)); m = q @ q.T / (n + 3) + 1e-3 * np.eye(n)
        r = int(rng.integers(1, n + 1)); g = rng.normal(size=(n, r)); a = g @ g.T
        sol = ut.solve_gen_eig_sym(a, m)
        ref = oracle.gen_eig_sym(a, m)
        lam = np.asarray(ref[0]); lmax = max(lam.max(), 1e-300)
        got = np.asarray(sol.eigenvalues)
        sig = lam > 1e-6 * lmax
        assert np.all(np.abs(got[sig] - lam[sig]) <= 1e-9 * lam[sig]), ("evals", n, r)
        assert np.all(np.abs(got[~sig] - lam[~sig]) <= 1e-9 * lmax), ("evals0", n, r)
        # well-separated eigenvalues: vectors to 1e-6 after sign alignment
        gaps = np.abs(np.diff(lam[sig])) if sig.sum() > 1 else np.array([1.0])
        if sig.sum() >= 1 and (sig.sum() == 1 or gaps.min() > 1e-3 * lmax):
            v = align_signs(np.asarray(sol.eigenvectors)[:, sig], np.asarray(ref[1])[:, sig])
            assert rel_close(v, np.asarray(ref[1])[:, sig], 1e-6), ("evecs", n, r)
        # LDA (two classes, standardized columns) on a random design matrix
        b = int(rng.integers(2, 33)); c = 2; npts = int(rng.integers(c * (b + 2), 1500))
        labels = rng.integers(0, c, npts); labels[:c] = np.arange(c)
        means = rng.uniform(0.2, 0.8, size=(c, b))
        values = (means[labels] + rng.normal(scale=0.03, size=(npts, b))).T * rng.uniform(0.5, 3.0, size=(b, 1))
        dm = ut.DesignMatrix(np.ascontiguousarray(values), labels.astype(np.intp), tuple())
        k = int(rng.integers(1, min(b, c - 1) + 1))
        mo = ut.fit_lda(dm, k=k)
        ro = oracle.fit_lda(values, labels, k=k)
        le = np.asarray(ro["eigenvalues"])
        assert np.all(np.abs(np.asarray(mo.eigenvalues) - le) <= 1e-9 * le.max()), ("lda evals", b, c, k)
        assert rel_close(mo.mean, ro["mean"], 1e-9) and rel_close(mo.std, ro["std"], 1e-9), ("lda mean/std", b, c)
        # device encoders read back by cv2
        h = int(rng.integers(1, 200)); w = int(rng.integers(1, 300)); ch = int(rng.choice([1, 3]))
        dt = rng.choice([np.uint8, np.uint16]); top = np.iinfo(dt).max
        shape = (h, w) if ch == 1 else (h, w, 3)
        yy, xx = np.mgrid[0:h, 0:w]
        base = (np.sin(xx / 9.0) + np.cos(yy / 7.0) + 2) / 4 * top * rng.uniform(0.1, 1.0)
        img = (base if ch == 1 else base[..., None] * np.array([1, .5, .25]))
        img = np.clip(img + rng.normal(0, top * rng.choice([0, 0.001, 0.05]), size=shape), 0, top).astype(dt)
        t = torch.from_numpy(img).cuda()
        for data in (image_io.encode_png(t), image_io.encode_tiff(t, "deflate"), image_io.encode_tiff(t, "none")):
            back = cv2.imdecode(np.frombuffer(data, np.uint8), cv2.IMREAD_UNCHANGED)
            back = back[:, :, ::-1] if back.ndim == 3 else back
            assert back.dtype == img.dtype and np.array_equal(back, img), ("encode", shape, dt)
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:200], traceback.format_exc().splitlines()[-3][:140], flush=True)
print("fuzz solvers done, fails:", fails)
