"""Random planes / regions / stacks through the stretch modes, sub-region PCA, normalize_stack
and project_stack subsets, against the oracle (dev tool; python tools/fuzz/fuzz_widen.py)."""
import sys, warnings, traceback
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch
import oracle
from golden_util import rel_close, plane_close
import paper_1612_06457_b200 as ut
from test_gpu_edges import cube_of, device_stack, DTYPES
warnings.simplefilter("ignore")
rng = np.random.default_rng(77)
fails = 0
def tonp(x): return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
for it in range(200):
    try:
        # percentile / full stretch on random fp planes (device tensors, fp32 contract)
        h = int(rng.integers(1, 300)); w = int(rng.integers(1, 500))
        kind = it % 4
        if kind == 0: plane = rng.normal(size=(h, w))
        elif kind == 1: plane = rng.integers(-5, 6, size=(h, w)).astype(np.float64)   # many ties
        elif kind == 2: plane = np.full((h, w), 3.25)
        else: plane = rng.standard_cauchy(size=(h, w))
        plane = plane.astype(np.float32).astype(np.float64)
        sp = ut.ScorePlane(plane)
        depth = int(rng.choice([8, 16]))
        got = tonp(ut.rescale_full(sp, depth=depth))
        assert np.array_equal(got, oracle.rescale_full(plane, depth=depth)), "full"
        p = float(rng.choice([0.01, 0.1, 1.0, 5.0]))
        one = bool(rng.integers(0, 2))
        got = tonp(ut.rescale_percentile(sp, p, depth=depth, one_tail=one))
        assert np.array_equal(got, oracle.rescale_percentile(plane, p, depth=depth, one_tail=one)), ("pct", p, one, depth)
        # sub-region PCA
        b = int(rng.integers(1, 33)); hh = int(rng.integers(6, 150)); ww = int(rng.integers(6, 300))
        dtype = DTYPES[int(rng.integers(0, len(DTYPES)))]
        cube, _ = cube_of(rng, b, hh, ww, dtype)
        x0 = int(rng.integers(0, ww - 2)); y0 = int(rng.integers(0, hh - 2))
        rw = int(rng.integers(2, ww - x0 + 1)); rh = int(rng.integers(2, hh - y0 + 1))
        if it % 3 == 0: x0, rw = 0, ww     # whole-width regions take the tensor-core paths
        region = (x0, y0, rw, rh)
        ds = device_stack(cube)
        k = min(3, b)
        pm = ut.fit_pca_unsupervised(ds, region=region, k=k)
        rp = oracle.fit_pca_unsupervised(cube, region=region, k=k)
        assert rel_close(tonp(pm.mean), rp["mean"], 1e-9), ("pca mean", region, b, dtype.__name__)
        assert rel_close(tonp(pm.std), rp["std"], 1e-9), ("pca std", region, b, dtype.__name__)
        le = np.asarray(rp["eigenvalues"])
        assert np.all(np.abs(tonp(pm.eigenvalues) - le) <= 1e-9 * (le.max() + np.abs(le))), ("pca evals", region, b, dtype.__name__)
        # normalize_stack on integer stacks
        if dtype in (np.uint8, np.uint16):
            hs = ut.SpectralStack(ut.stack.default_bands(b), cube, 16 if dtype == np.uint16 else 8, False)
            scope = "per-band" if it % 2 else "global"
            got = ut.normalize_stack(hs, scope)
            want, _ = oracle.normalize_stack(cube, scope)
            assert np.array_equal(tonp(got.planes), want), ("normalize", scope, b, dtype.__name__)
        # project_stack with many components / subsets
        kk = int(rng.integers(1, b + 1))
        coef = rng.normal(size=(b, kk)); mean = rng.uniform(0.2, 0.7, size=b)
        std = rng.uniform(0.5, 2.0, size=b) if it % 2 else None
        model = ut.ProjectionModel("pca_unsupervised" if std is not None else "cva", mean, std, coef, np.ones(kk))
        comps = sorted(set(int(c) for c in rng.integers(0, kk, size=int(rng.integers(1, kk + 1)))))
        planes = ut.project_stack(ds, model, components=comps)
        ref = oracle.project(cube, {"mean": mean, "std": std, "coefficients": coef}, components=comps)
        gotp = np.stack([tonp(pl.values.double()) for pl in planes])
        assert plane_close(gotp, ref) <= 1e-6, ("project", b, kk, comps, dtype.__name__, plane_close(gotp, ref))
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:300], traceback.format_exc().splitlines()[-3][:160], flush=True)
print("fuzz widen done, fails:", fails)
