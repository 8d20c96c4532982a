"""Edge cases of the device path against the oracle: odd / ragged sizes (vector
tails, odd pixel counts that rule out the tensor-core and bulk-copy paths),
strided views, one band, more than 8 components (several projector passes),
many classes (several moment launches, the low-rank solve with C = 20), 16-bit
codes, PCA on sub-regions, every sample dtype with both projector precisions."""

import numpy as np
import pytest

import oracle
from golden_util import align_signs, plane_close, rel_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200.rendering import stretch_planes  # noqa: E402

DTYPES = [np.uint8, np.uint16, np.float16, np.float32, np.float64]


def cube_of(rng, b, h, w, dtype, classes=3):
    means = rng.uniform(0.2, 0.8, size=(classes, b))
    cmap = rng.integers(0, classes, size=(h, w))
    x = means[cmap] + rng.normal(scale=0.03, size=(h, w, b))
    x = np.clip(x, 0, 1).transpose(2, 0, 1)
    if dtype == np.uint8:
        x = np.floor(255 * x + 0.5)
    elif dtype == np.uint16:
        x = np.floor(4095 * x + 0.5)
    return np.ascontiguousarray(x.astype(dtype)), cmap


def device_stack(cube):
    depth = 16 if cube.dtype == np.uint16 else 8
    return ut.DeviceStack(ut.stack.default_bands(cube.shape[0]),
                          torch.from_numpy(cube).cuda(), depth, True)


def pick_points(rng, cmap, per):
    xs, ys, ls = [], [], []
    for c in np.unique(cmap):
        yy, xx = np.nonzero(cmap == c)
        sel = rng.choice(len(yy), size=min(per, len(yy)), replace=False)
        xs += list(xx[sel])
        ys += list(yy[sel])
        ls += [c] * len(sel)
    return np.array(xs), np.array(ys), np.array(ls)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("hw", [(23, 37), (16, 64), (1, 9), (40, 33)])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_projector_sizes_dtypes(dtype, hw, precision):
    rng = np.random.default_rng(hash((str(dtype), hw)) % 2**32)
    h, w = hw
    cube, _ = cube_of(rng, 7, h, w, dtype)
    coef = rng.normal(size=(7, 6))
    mean = cube.reshape(7, -1).astype(np.float64).mean(axis=1)
    model = ut.ProjectionModel("cva", mean, None, coef, np.ones(6))
    planes = ut.project_stack(device_stack(cube), model, precision=precision)
    ref = oracle.project(cube, {"mean": mean, "std": None, "coefficients": coef})
    got = np.stack([p.values.double().cpu().numpy() for p in planes])
    assert plane_close(got, ref) <= (1e-7 if precision == "fp64" else 1e-6)
    for p in planes:
        codes = ut.rescale_full(p).cpu().numpy()
        assert np.array_equal(codes, oracle.rescale_full(p.values.double().cpu().numpy()))


def test_strided_view_and_many_components():
    rng = np.random.default_rng(3)
    cube, _ = cube_of(rng, 12, 40, 50, np.float32)
    view = torch.from_numpy(cube).cuda()[:, 5:31, 7:44]  # row_stride != cols
    ds = ut.DeviceStack(ut.stack.default_bands(12), view, 8, True)
    coef = rng.normal(size=(12, 11))
    mean = rng.uniform(0.3, 0.6, size=12)
    std = rng.uniform(0.5, 2.0, size=12)
    model = ut.ProjectionModel("pca_unsupervised", mean, std, coef, np.ones(11))
    planes = ut.project_stack(ds, model)  # 11 components: two K4 passes
    host = np.ascontiguousarray(cube[:, 5:31, 7:44])
    ref = oracle.project(host, {"mean": mean, "std": std, "coefficients": coef})
    got = np.stack([p.values.double().cpu().numpy() for p in planes])
    assert plane_close(got, ref) <= 1e-7
    sub = ut.project_stack(ds, model, components=[10, 3])
    assert plane_close(np.stack([p.values.double().cpu().numpy() for p in sub]),
                       ref[[10, 3]]) <= 1e-7


def test_single_band():
    rng = np.random.default_rng(4)
    cube, cmap = cube_of(rng, 1, 30, 30, np.float64)
    xs, ys, ls = pick_points(rng, cmap, 20)
    ds = device_stack(cube)
    pipe = ut.CvaPipeline(ds, xs, ys, ls, k=1)
    pipe.run()
    m = pipe.model()
    ref = oracle.fit_cva(oracle.assemble(cube, xs, ys), ls, k=1)
    assert rel_close(m.eigenvalues, ref["eigenvalues"], 1e-9)
    assert rel_close(m.coefficients, ref["coefficients"], 1e-9)
    pm = ut.fit_pca_unsupervised(ds, k=1)
    ref_p = oracle.fit_pca_unsupervised(cube, k=1)
    assert rel_close(pm.eigenvalues, ref_p["eigenvalues"], 1e-9)
    assert rel_close(pm.mean, ref_p["mean"], 1e-12)


def test_many_classes_low_rank_and_moment_launches():
    rng = np.random.default_rng(5)
    cube, cmap = cube_of(rng, 24, 60, 80, np.float32, classes=20)
    xs, ys, ls = pick_points(rng, cmap, 25)
    ds = device_stack(cube)
    for k in (5, 19, 24):  # low-rank path (k <= C-1) and the full path
        pipe = ut.CvaPipeline(ds, xs, ys, ls, k=k)
        pipe.run()
        h = pipe.check()
        ref = oracle.fit_cva(oracle.assemble(cube, xs, ys), ls, k=k)
        sp = ref["scatter"]
        assert np.array_equal(h["counts"].astype(int), sp["counts"])
        assert rel_close(h["within"], sp["within"], 1e-9)
        assert rel_close(h["between"], sp["between"], 1e-9)
        lam = np.asarray(ref["eigenvalues"])
        sig = lam > 1e-6 * lam.max()
        assert np.all(np.abs(h["evals"][:k][sig] - lam[sig]) <= 1e-9 * np.abs(lam[sig]))
        got = align_signs(h["evecs"][:, :k][:, sig], ref["coefficients"][:, sig])
        assert rel_close(got, ref["coefficients"][:, sig], 1e-6)


def test_sixteen_bit_codes_pipeline():
    rng = np.random.default_rng(6)
    cube, cmap = cube_of(rng, 8, 32, 48, np.uint16)
    xs, ys, ls = pick_points(rng, cmap, 30)
    pipe = ut.CvaPipeline(device_stack(cube), xs, ys, ls, k=2, depth=16)
    codes = pipe.run().cpu().numpy()
    assert codes.dtype == np.uint16
    for j in range(2):
        want = oracle.rescale_full(pipe.scores[j].double().cpu().numpy(), depth=16)
        assert np.array_equal(codes[j], want)


def test_pca_subregion_on_device():
    rng = np.random.default_rng(7)
    cube, _ = cube_of(rng, 9, 50, 70, np.float32)
    ds = device_stack(cube)
    for region in [(3, 4, 40, 30), (0, 10, 70, 20), (69, 0, 1, 50)]:
        pm = ut.fit_pca_unsupervised(ds, region=region, k=3)
        ref = oracle.fit_pca_unsupervised(cube, region=region, k=3)
        assert rel_close(pm.mean, ref["mean"], 1e-12)
        assert rel_close(pm.std, ref["std"], 1e-9)
        lam = ref["eigenvalues"]
        assert np.all(np.abs(pm.eigenvalues - lam) <= 1e-9 * np.abs(lam).max())


def test_empty_and_degenerate_inputs():
    rng = np.random.default_rng(8)
    cube, cmap = cube_of(rng, 4, 10, 10, np.float32)
    ds = device_stack(cube)
    with pytest.raises(ut.DataError):
        ut.CvaPipeline(ds, [], [], [], k=1)
    with pytest.raises(ut.DataError):
        ut.CvaPipeline(ds, [1, 2], [1, 2], [0, 0], k=1)  # one class
    with pytest.raises(ut.DataError):
        ut.CvaPipeline(ds, [1, 20], [1, 2], [0, 1], k=1)  # out of bounds
    # constant plane: zeros + warning through the host API
    flat = np.full((2, 6, 6), 7, dtype=np.uint8)
    st = ut.SpectralStack(ut.stack.default_bands(2), flat, 8, True)
    m = ut.ProjectionModel("cva", np.zeros(2), None, np.array([[1.0], [0.0]]), np.ones(1))
    plane = ut.project_stack(st, m)[0]
    with pytest.warns(ut.UndertextWarning):
        out = ut.rescale_full(plane)
    assert not out.any()
    # singular within scatter with ridge 0 -> NumericError (tests/test_cli.py:72-91)
    xs, ys = np.array([0, 1, 2, 3]), np.array([0, 0, 0, 0])
    cube2 = np.zeros((2, 1, 4), np.float64)
    cube2[0, 0] = [1, 1, 5, 5]
    cube2[1, 0] = [2, 2, 7, 7]
    pipe = ut.CvaPipeline(device_stack(cube2), xs, ys, np.array([0, 0, 1, 1]), k=1, ridge=0.0)
    pipe.run()
    with pytest.raises(ut.NumericError):
        pipe.check()


def test_nonfinite_scores_detected():
    cube = np.ones((2, 4, 4), np.float32)
    cube[0, 1, 2] = np.nan
    ds = ut.DeviceStack(ut.stack.default_bands(2), torch.from_numpy(cube).cuda(), 8, True)
    m = ut.ProjectionModel("cva", np.zeros(2), None, np.eye(2), np.ones(2))
    for prec in ("fp64", "fp32"):
        with pytest.raises(ut.DataError, match="NaN"):
            ut.project_stack(ds, m, precision=prec)


def test_folio_stream_matches_independent_pipelines():
    """cfg 5's streaming loop (FolioStream): each folio's codes equal a
    standalone pipeline's on the same cube and training set."""
    from dataclasses import replace

    from paper_1612_06457_b200 import synthetic

    base = synthetic.scaled(synthetic.CONFIGS["cfg5"], 200, 160, 60)
    cubes, train, outs, want = [], [], [], []
    for f in range(3):
        sc = synthetic.make_scene(replace(base, seed=77 + f))
        st = synthetic.generate(sc)
        cubes.append(st.planes.cpu().pin_memory())
        arrs = ut.CvaPipeline.training_arrays(sc.xs, sc.ys, sc.labels)
        train.append(tuple(torch.from_numpy(a).pin_memory() for a in arrs))
        outs.append(torch.empty((base.k, base.height, base.width), dtype=torch.uint8,
                                pin_memory=True))
        ref = ut.CvaPipeline(st, sc.xs, sc.ys, sc.labels, k=base.k)
        want.append(ref.run().cpu().numpy())
    fs = ut.FolioStream(cubes, train, outs, k=base.k)
    for _ in range(2):
        fs.run()
        torch.cuda.synchronize()
        fs.check()
        for o, w in zip(outs, want):
            assert np.array_equal(o.numpy(), w)
    with pytest.raises(ut.DataError):
        fs.pipes[0].load_training(train[0][0][:5], train[0][1][:5], train[0][2])


def _folios(n, nan_folio=None):
    from dataclasses import replace

    from paper_1612_06457_b200 import synthetic

    base = synthetic.scaled(synthetic.CONFIGS["cfg5"], 120, 96, 40)
    cubes, train, outs = [], [], []
    for f in range(n):
        sc = synthetic.make_scene(replace(base, seed=91 + f))
        planes = synthetic.generate(sc).planes.cpu()
        if f == nan_folio:
            planes[0, 7, 9] = float("nan")
        cubes.append(planes.pin_memory())
        arrs = ut.CvaPipeline.training_arrays(sc.xs, sc.ys, sc.labels)
        train.append(tuple(torch.from_numpy(a).pin_memory() for a in arrs))
        outs.append(torch.empty((base.k, base.height, base.width), dtype=torch.uint8,
                                pin_memory=True))
    return base, cubes, train, outs


def test_folio_stream_reports_the_failing_folio():
    """an earlier folio's device error must survive later folios that
    reuse its buffer -- per-folio status slots, reported with the folio index."""
    _, cubes, train, outs = _folios(4, nan_folio=0)
    fs = ut.FolioStream(cubes, train, outs, k=3)
    fs.run()
    torch.cuda.synchronize()
    with pytest.raises(ut.DataError, match=r"folio 0: score plane contains NaN"):
        fs.check()


def test_folio_stream_validates_every_training_set():
    _, cubes, train, outs = _folios(3)
    xy, cls, piv = train[2]
    bad = xy.clone()
    bad[5, 1] = 10_000
    train[2] = (bad, cls, piv)
    with pytest.raises(ut.DataError, match=r"folio 2: .*outside"):
        ut.FolioStream(cubes, train, outs, k=3)


def test_bad_point_reported_in_caller_order():
    """A point swapped in past the stack: K1 flags it; check() names it by its
    coordinates (K1's class-sorted index is not the caller's)."""
    rng = np.random.default_rng(12)
    cube, _ = cube_of(rng, 6, 40, 50, np.float32)
    xs = rng.integers(0, 50, 30)
    ys = rng.integers(0, 40, 30)
    labels = np.arange(30) % 3
    st = ut.DeviceStack(ut.stack.default_bands(6), torch.from_numpy(cube).cuda(), 8, True)
    pipe = ut.CvaPipeline(st, xs, ys, labels, k=2)
    xy, cls, piv = ut.CvaPipeline.training_arrays(xs, ys, labels)
    xy[4] = (51, 3)
    pipe.load_training(torch.from_numpy(xy).cuda(), torch.from_numpy(cls).cuda(),
                       torch.from_numpy(piv).cuda())
    pipe.run()
    with pytest.raises(ut.DataError, match=r"\(51, 3\) outside"):
        pipe.check()


@pytest.mark.parametrize("b,k", [(29, 2), (32, 3), (20, 1), (19, 2)])
def test_wide_fp64_cube_few_components(b, k):
    """fp64 cubes of more than 18 bands with fewer than 4 components: a 512-pixel
    stage of the bulk-copy projector would not fit shared memory three times, so the
    direct-load projector runs (the launch used to fail with an invalid shared-memory
    attribute; found by fuzzing shapes against the oracle)."""
    rng = np.random.default_rng(100 * b + k)
    cube, cmap = cube_of(rng, b, 52, 160, np.float64, classes=4)
    xs, ys, ls = pick_points(rng, cmap, 60)
    pipe = ut.CvaPipeline(device_stack(cube), xs, ys, ls, k=k)
    codes = pipe.run().cpu().numpy()
    pipe.check()
    m = pipe.model()
    want = oracle.project(cube, {"mean": m.mean, "std": None, "coefficients": m.coefficients})
    assert plane_close(pipe.scores.double().cpu().numpy(), want) <= 1e-6
    for j in range(k):
        assert np.array_equal(codes[j], oracle.rescale_full(pipe.scores[j].double().cpu().numpy()))


def test_path_fuzz_vs_oracle():
    """Seeded random shapes / dtypes / class counts / point orders through the whole
    path (fit, planes, codes, PCA) against the oracle."""
    rng = np.random.default_rng(2024)
    done = 0
    for it in range(40):
        b, classes = int(rng.integers(1, 33)), int(rng.integers(2, 9))
        h, w = int(rng.integers(8, 200)), int(rng.integers(8, 400))
        dtype = DTYPES[int(rng.integers(0, len(DTYPES)))]
        cube, cmap = cube_of(rng, b, h, w, dtype, classes=classes)
        per = int(rng.integers(max(3, b // classes + 2), 120))
        xs, ys, ls = pick_points(rng, cmap, per)
        if len(np.unique(ls)) < 2:
            continue
        if it % 2:
            perm = rng.permutation(len(ls))
            xs, ys, ls = xs[perm], ys[perm], ls[perm]
        k = int(rng.integers(1, min(b, len(np.unique(ls)) - 1) + 1))
        ds = device_stack(cube)
        pipe = ut.CvaPipeline(ds, xs, ys, ls, k=k)
        codes = pipe.run().cpu().numpy()
        hst = pipe.check()
        ref = oracle.fit_cva(oracle.assemble(cube, xs, ys), ls, k=k)
        sp = ref["scatter"]
        case = (it, b, classes, h, w, dtype.__name__, k)
        assert np.array_equal(hst["counts"].astype(int), sp["counts"]), case
        assert rel_close(hst["within"], sp["within"], 1e-9), case
        assert rel_close(hst["between"], sp["between"], 1e-9), case
        lam = np.asarray(ref["eigenvalues"])
        sig = lam > 1e-6 * lam.max()
        assert np.all(np.abs(hst["evals"][:k][sig] - lam[sig]) <= 1e-9 * np.abs(lam[sig])), case
        m = pipe.model()
        want = oracle.project(cube, {"mean": m.mean, "std": None, "coefficients": m.coefficients})
        assert plane_close(pipe.scores.double().cpu().numpy(), want) <= 1e-6, case
        for j in range(k):
            assert np.array_equal(codes[j],
                                  oracle.rescale_full(pipe.scores[j].double().cpu().numpy())), case
        pm = ut.fit_pca_unsupervised(ds, k=min(3, b))
        rp = oracle.fit_pca_unsupervised(cube, k=min(3, b))
        assert rel_close(pm.mean, rp["mean"], 1e-9), case
        le = np.asarray(rp["eigenvalues"])
        assert np.all(np.abs(np.asarray(pm.eigenvalues) - le) <= 1e-9 * (le.max() + np.abs(le))), case
        done += 1
    assert done >= 35
