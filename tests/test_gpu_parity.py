"""GPU parity: the B200 path against the golden vectors and the CPU oracle.

Bars (SURVEY.md Appendix A / BASELINE.json north star):
  class ids and counts bit-exact; means and scatter matrices 1e-9 relative
  (per matrix, max|delta| <= 1e-9 max|ref|); significant eigenvalues 1e-9
  relative, the rest |delta| <= 1e-9 lambda_max; kept eigenvectors 1e-6 after
  per-component sign alignment; score planes 1e-6 of the reference plane's
  range; uint8 codes within +-1 (and bit-exact against the oracle's stretch of
  the device's own fp32 planes).
"""

import warnings

import numpy as np
import pytest

import oracle
from golden_util import align_signs, load, plane_close, rel_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402

SCORE_TOL = 1e-6
CUBES = ["cva_f64", "cva_f32", "cva_u16", "cva_f16", "cva_f32_b32", "small_page"]


def host_stack(cube):
    depth = 16 if cube.dtype == np.uint16 else 8
    return ut.SpectralStack(ut.stack.default_bands(cube.shape[0]), cube, depth, normalized=True)


def dm_of(values, labels):
    return ut.DesignMatrix(np.asarray(values, dtype=np.float64),
                           np.asarray(labels, dtype=np.intp), tuple())


def significant(evals):
    """The reference's own threshold (tests/test_acceptance.py:140)."""
    return np.asarray(evals) > 1e-6 * float(np.max(evals))


def eig_close(got, want, tol=1e-9):
    """Significant eigenvalues (> 1e-6 lambda_max) relative; the rest absolute."""
    lam_max = float(np.abs(want).max())
    sig = np.abs(want) > 1e-6 * lam_max
    ok_sig = np.all(np.abs(got[sig] - want[sig]) <= tol * np.abs(want[sig]))
    ok_rest = np.all(np.abs(got[~sig] - want[~sig]) <= tol * lam_max)
    return bool(ok_sig and ok_rest)


def check_codes(got_codes, got_scores, want_codes):
    """+-1 against the reference codes; bit-exact against the oracle's stretch
    of the device's own fp32 planes."""
    got_codes = np.asarray(got_codes)
    assert int(np.abs(got_codes.astype(int) - want_codes.astype(int)).max()) <= 1
    mine = np.stack([oracle.rescale_full(np.asarray(s, dtype=np.float64)) for s in got_scores])
    assert np.array_equal(got_codes, mine)


# ------------------------------------------------------------------ golden

def test_scatter_golden():
    g = load("scatter")
    for i in range(int(g["n"])):
        sp = ut.compute_scatter(dm_of(g[f"{i}_values"], g[f"{i}_labels"]))
        assert np.array_equal(np.array(sp.class_ids), g[f"{i}_ids"])
        assert np.array_equal(sp.counts, g[f"{i}_counts"])
        assert sp.counts.dtype == np.intp
        for got, key in ((sp.within, "within"), (sp.between, "between"),
                         (sp.class_means, "means"), (sp.grand_mean, "grand")):
            assert rel_close(got, g[f"{i}_{key}"], 1e-9), (i, key)
        assert np.array_equal(sp.within, sp.within.T)
        assert np.array_equal(sp.between, sp.between.T)


def test_eigen_golden():
    g = load("eigen")
    for i in range(int(g["n"])):
        sol = ut.solve_gen_eig_sym(g[f"{i}_a"], g[f"{i}_m"], float(g[f"{i}_ridge"]))
        want_l, want_v = g[f"{i}_evals"], g[f"{i}_evecs"]
        assert eig_close(sol.eigenvalues, want_l), i
        v = align_signs(sol.eigenvectors, want_v)
        assert rel_close(v, want_v, 1e-6), i


@pytest.mark.parametrize("name", CUBES)
def test_cube_golden(name):
    g = load(name)
    cube = g["cube"]
    stack = host_stack(cube)
    ts = ut.TrainingSet.from_arrays(g["xs"], g["ys"], g["labels"])
    dm = ut.assemble_matrix(stack, ts)
    assert np.array_equal(dm.values, g["design"])
    k = g["cva_coef"].shape[1]
    model = ut.fit_cva(dm, k=k)
    assert rel_close(model.mean, g["cva_mean"], 1e-9)
    assert eig_close(model.eigenvalues, g["cva_evals"])
    # vectors / planes: significant components only -- null-space CVA
    # directions (lambda ~ 1e-14) are numerically arbitrary (Appendix A)
    sig = significant(g["cva_evals"])
    coef = align_signs(model.coefficients[:, sig], g["cva_coef"][:, sig])
    assert rel_close(coef, g["cva_coef"][:, sig], 1e-6)
    planes = ut.project_stack(stack, model, components=list(np.flatnonzero(sig)))
    signs = np.sign(np.sum(model.coefficients[:, sig] * g["cva_coef"][:, sig], axis=0))
    scores = np.stack([p.values for p in planes]) * signs[:, None, None]
    assert plane_close(scores, g["cva_scores"][sig]) <= SCORE_TOL
    codes = np.stack([ut.rescale_full(p) for p in planes])
    flip = signs < 0
    want = g["cva_codes"][sig].copy()
    want[flip] = 255 - want[flip]  # a flipped plane maps min<->max
    check_codes(codes, [p.values for p in planes], want)
    # PCA (region from the fixture)
    region = tuple(int(v) for v in g["pca_region"]) if "pca_region" in g else None
    pk = g["pca_coef"].shape[1]
    pm = ut.fit_pca_unsupervised(stack, region=region, k=pk)
    assert rel_close(pm.mean, g["pca_mean"], 1e-9)
    assert rel_close(pm.std, g["pca_std"], 1e-9)
    assert eig_close(pm.eigenvalues, g["pca_evals"])
    pc = align_signs(pm.coefficients, g["pca_coef"])
    assert rel_close(pc, g["pca_coef"], 1e-6)
    pplanes = ut.project_stack(stack, pm)
    psigns = np.sign(np.sum(pm.coefficients * g["pca_coef"], axis=0))
    pscores = np.stack([p.values for p in pplanes]) * psigns[:, None, None]
    assert plane_close(pscores, g["pca_scores"]) <= SCORE_TOL


def test_rescale_golden():
    g = load("rescale")
    for key in ("sign", "normal", "ties", "wide"):
        assert np.array_equal(ut.rescale_full(ut.ScorePlane(g[f"{key}_in"])), g[f"{key}_u8"]), key
        out16 = ut.rescale_full(ut.ScorePlane(g[f"{key}_in"]), depth=16)
        assert out16.dtype == np.uint16
        assert np.array_equal(out16, g[f"{key}_u16"]), key
    with pytest.warns(ut.UndertextWarning):
        out = ut.rescale_full(ut.ScorePlane(np.full((4, 4), 3.5)))
    assert not out.any()


# ------------------------------------------------- reference known answers

def test_known_answers():
    # tests/test_projection.py:63-69
    sp = ut.compute_scatter(dm_of([[0.0, 2.0, 10.0, 12.0]], [0, 0, 1, 1]))
    assert sp.within.tolist() == [[4.0]] and sp.between.tolist() == [[100.0]]
    assert sp.grand_mean.tolist() == [6.0] and sp.class_means.tolist() == [[1.0], [11.0]]
    # tests/test_eigen.py:17-35
    sol = ut.solve_gen_eig_sym(np.diag([3.0, 1.0]), np.eye(2), ridge=0.0)
    assert np.allclose(sol.eigenvalues, [3.0, 1.0], atol=1e-14)
    assert np.allclose(sol.eigenvectors, np.eye(2), atol=1e-14)
    sol = ut.solve_gen_eig_sym(np.diag([2.0, 2.0]), np.diag([1.0, 2.0]), ridge=0.0)
    assert np.allclose(sol.eigenvalues, [2.0, 1.0], atol=1e-14)
    assert np.allclose(sol.eigenvectors, [[1.0, 0.0], [0.0, 1 / np.sqrt(2)]], atol=1e-14)
    sol = ut.solve_gen_eig_sym(np.diag([3.0, 1.0]), np.eye(2))
    assert np.allclose(sol.eigenvalues, np.array([3.0, 1.0]) / (1 + 1e-8), rtol=1e-12)
    sol = ut.solve_gen_eig_sym(np.diag([4.0, 1.0]), np.zeros((2, 2)))
    assert np.allclose(sol.eigenvalues, [4e8, 1e8], rtol=1e-10)
    # tests/test_quantize.py:33-48 through the device stretch
    assert ut.linear_to_codes(np.array([-1.0, 0.0, 1.0]), -1.0, 1.0, 8).tolist() == [0, 128, 255]
    assert ut.linear_to_codes(np.array([-5.0, 0.5, 20.0]), 0.0, 1.0, 8).tolist() == [0, 128, 255]
    assert ut.linear_to_codes(np.array([0.0, 1.0]), 0.0, 1.0, 16).tolist() == [0, 65535]
    with pytest.raises(ValueError):
        ut.linear_to_codes(np.array([1.0]), 2.0, 2.0, 8)
    # tests/test_rendering.py:72-86
    assert ut.rescale_full(ut.ScorePlane(np.array([[-1.0, 0.0, 1.0]]))).tolist() == [[0, 128, 255]]
    assert ut.rescale_full(ut.ScorePlane(np.array([[-1.0, 0.0, 1.0]])), 16).tolist() == [[0, 32768, 65535]]


def test_eigen_errors():
    # tests/test_eigen.py:120-135
    with pytest.raises(ut.NumericError, match="condition|definite"):
        ut.solve_gen_eig_sym(np.eye(2), np.diag([2.0, -1.0]))
    a = np.array([[1.0, 2.0], [0.0, 1.0]])
    with pytest.raises(ut.NumericError, match="symmetric"):
        ut.solve_gen_eig_sym(a, np.eye(2))
    with pytest.raises(ut.NumericError, match="symmetric"):
        ut.solve_gen_eig_sym(np.eye(2), a)
    with pytest.raises(ut.NumericError):
        ut.solve_gen_eig_sym(np.eye(3), np.eye(2))


def test_sign_convention_ties():
    # ties break to the lowest index (eigen.py:43-51): A = I, M = I -> columns of I
    sol = ut.solve_gen_eig_sym(np.eye(4), np.eye(4), ridge=0.0)
    for j in range(4):
        col = sol.eigenvectors[:, j]
        lead = int(np.argmax(np.abs(col)))
        assert col[lead] > 0


def test_cva_reference_contracts():
    rng = np.random.default_rng(3)
    # separable clouds (tests/test_projection.py:94-102)
    a = rng.normal(size=(2, 4000))
    b = np.array([[10.0], [0.0]]) + rng.normal(size=(2, 4000))
    model = ut.fit_cva(dm_of(np.concatenate([a, b], axis=1), [0] * 4000 + [1] * 4000))
    v = model.coefficients[:, 0]
    assert abs(v[0]) / np.linalg.norm(v) >= 0.999
    # identical classes -> eigenvalues ~ 0 (tests/test_projection.py:115-120)
    pts = np.array([[0.0, 1.0, 2.0], [5.0, 6.0, 7.0]])
    dm = dm_of(np.concatenate([pts, pts], axis=1), [0, 0, 0, 1, 1, 1])
    m2 = ut.fit_cva(dm)
    assert (np.abs(m2.eigenvalues) <= 1e-10 * np.trace(ut.compute_scatter(dm).within)).all()
    # apply == training_scores bit-exact (tests/test_projection.py:122-127)
    vals = rng.normal(size=(4, 45)) + np.repeat(rng.normal(scale=4, size=(4, 3)), 15, axis=1)
    m3 = ut.fit_cva(dm_of(vals, np.repeat([0, 1, 2], 15)))
    assert np.array_equal(m3.apply(vals.T), m3.training_scores.T)
    with pytest.raises(ut.DataError):
        ut.fit_cva(dm_of(vals, np.repeat([0, 1, 2], 15)), k=5)
    with pytest.raises(ut.DataError):
        ut.compute_scatter(dm_of([[1.0, 2.0]], [0, 0]))


def test_project_known_answers():
    rng = np.random.default_rng(14)
    planes = rng.integers(0, 255, size=(3, 12, 9), dtype=np.uint8)
    model = ut.ProjectionModel("cva", np.zeros(3), None, np.eye(3), np.ones(3))
    out = ut.project_stack(host_stack(planes), model)
    for b in range(3):
        assert np.array_equal(out[b].values, planes[b].astype(np.float64))
    two = np.stack([np.full((4, 4), 9, np.uint8), np.full((4, 4), 3, np.uint8)])
    m = ut.ProjectionModel("cva", np.zeros(2), None, np.array([[1.0], [-1.0]]), np.ones(1))
    assert np.all(ut.project_stack(host_stack(two), m)[0].values == 6.0)
    # errors (tests/test_projection.py:292-307)
    with pytest.raises(ut.DataError, match="bands"):
        ut.project_stack(host_stack(planes), ut.ProjectionModel("cva", np.zeros(4), None,
                                                                np.eye(4), np.ones(4)))
    with pytest.raises(ut.DataError, match="normalized"):
        st = ut.SpectralStack(ut.stack.default_bands(3), planes, 8, normalized=False)
        ut.project_stack(st, ut.ProjectionModel("cva", np.zeros(3), None, np.eye(3), np.ones(3),
                                                provenance={"normalized_input": True}))
    with pytest.raises(ut.DataError):
        ut.project_stack(host_stack(planes), model, components=[3])


def test_pca_region_errors_and_rank_one():
    plane = np.arange(64, dtype=np.uint8).reshape(8, 8)
    pm = ut.fit_pca_unsupervised(host_stack(np.stack([plane, plane, plane])))
    assert pm.eigenvalues[0] == pytest.approx(3.0, rel=1e-8)
    assert np.allclose(pm.eigenvalues[1:], 0.0, atol=1e-9)
    st = host_stack(np.zeros((2, 10, 10), np.uint8) + np.arange(10, dtype=np.uint8))
    with pytest.raises(ut.DataError):
        ut.fit_pca_unsupervised(st, region=(0, 0, 1, 1))
    with pytest.raises(ut.DataError):
        ut.fit_pca_unsupervised(st, region=(5, 5, 8, 8))
    with pytest.raises(ut.DataError):
        ut.fit_pca_unsupervised(st, region=(0, 0, 0, 3))


def test_assemble_errors():
    st = host_stack(np.zeros((2, 5, 5), np.uint8))
    with pytest.raises(ut.DataError, match="outside"):
        ut.assemble_matrix(st, ut.TrainingSet.from_arrays([1, 7], [1, 1], [0, 1]))
    raw = ut.SpectralStack(ut.stack.default_bands(2), np.zeros((2, 5, 5), np.uint8), 8, False)
    with pytest.raises(ut.DataError, match="normalized"):
        ut.assemble_matrix(raw, ut.TrainingSet.from_arrays([1], [1], [0]))


# --------------------------------------------- BASELINE generator configs

def _scaled(name, h, w, per_class=None):
    return synthetic.scaled(synthetic.CONFIGS[name], h, w, per_class)


CVA_CASES = [
    ("cfg1", 512, 512, None),     # full size cfg 1 (the CPU-runnable config)
    ("cfg3", 361, 271, 200),      # cfg 3 generator, u16 12-bit, 23 bands, 4 classes
    ("cfg4", 384, 320, 300),      # cfg 4 generator, f32, 32 bands, 6 classes
    ("cfg5", 256, 192, 150),      # cfg 5 folio generator, f16
]


@pytest.mark.parametrize("name,h,w,per", CVA_CASES)
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_cva_pipeline_vs_oracle(name, h, w, per, precision):
    cfg = _scaled(name, h, w, per)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    cube = stack.planes.cpu().numpy()
    pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k, precision=precision)
    codes = pipe.run().cpu().numpy()
    model = pipe.model()
    ref_model, ref_scores, ref_codes = oracle.cpu_cva_pipeline(
        cube, scene.xs, scene.ys, scene.labels, k=cfg.k, workers=4)
    sp = ref_model["scatter"]
    h_dev = pipe.check()
    assert np.array_equal(h_dev["counts"].astype(np.int64), sp["counts"])
    assert rel_close(h_dev["within"], sp["within"], 1e-9)
    assert rel_close(h_dev["between"], sp["between"], 1e-9)
    assert rel_close(h_dev["class_means"], sp["class_means"], 1e-9)
    assert rel_close(model.mean, ref_model["mean"], 1e-9)
    assert eig_close(model.eigenvalues, ref_model["eigenvalues"])
    coef = align_signs(model.coefficients, ref_model["coefficients"])
    assert rel_close(coef, ref_model["coefficients"], 1e-6)
    signs = np.sign(np.sum(model.coefficients * ref_model["coefficients"], axis=0))
    scores = pipe.scores.double().cpu().numpy() * signs[:, None, None]
    err = plane_close(scores, ref_scores)
    assert err <= SCORE_TOL, f"{precision}: {err:.3e} of range"
    want = ref_codes.copy()
    want[signs < 0] = 255 - want[signs < 0]
    check_codes(codes, pipe.scores.cpu().numpy(), want)


def test_pca_pipeline_vs_oracle_cfg2():
    cfg = _scaled("cfg2", 512, 384)
    stack = synthetic.generate(synthetic.make_scene(cfg))
    cube = stack.planes.cpu().numpy()
    pipe = ut.PcaPipeline(stack, k=cfg.k)
    codes = pipe.run().cpu().numpy()
    pm = pipe.model()
    ref_pm, ref_scores, ref_codes = oracle.cpu_pca_pipeline(cube, k=cfg.k, workers=4)
    assert rel_close(pm.mean, ref_pm["mean"], 1e-9)
    assert rel_close(pm.std, ref_pm["std"], 1e-9)
    assert eig_close(pm.eigenvalues, ref_pm["eigenvalues"])
    assert rel_close(align_signs(pm.coefficients, ref_pm["coefficients"]),
                     ref_pm["coefficients"], 1e-6)
    signs = np.sign(np.sum(pm.coefficients * ref_pm["coefficients"], axis=0))
    scores = pipe.scores.double().cpu().numpy() * signs[:, None, None]
    assert plane_close(scores, ref_scores) <= SCORE_TOL
    want = ref_codes.copy()
    want[signs < 0] = 255 - want[signs < 0]
    check_codes(codes, pipe.scores.cpu().numpy(), want)


def test_pca_b32_vs_oracle():
    cfg = _scaled("cfg4pca", 256, 256)
    stack = synthetic.generate(synthetic.make_scene(cfg))
    cube = stack.planes.cpu().numpy()
    pm = ut.fit_pca_unsupervised(stack, k=5)
    ref = oracle.fit_pca_unsupervised(cube, k=5)
    assert rel_close(pm.mean, ref["mean"], 1e-9)
    assert rel_close(pm.std, ref["std"], 1e-9)
    assert eig_close(pm.eigenvalues, ref["eigenvalues"])


# ------------------------------------------------------- determinism, shards

def test_run_to_run_bit_identical():
    cfg = _scaled("cfg4", 256, 256, 100)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
    a = pipe.run().clone()
    s1 = pipe.scores.clone()
    m1 = pipe.model()
    b = pipe.run()
    assert torch.equal(a, b) and torch.equal(s1, pipe.scores)
    m2 = pipe.model()
    assert np.array_equal(m1.coefficients, m2.coefficients)


def test_sharded_moments_combine_on_device():
    """G row shards' class moments combined by the K3 kernel (groups=G) equal
    the unsharded fit -- the device half of the multi-GPU path, emulated on
    one GPU by computing each shard's moments separately."""
    from paper_1612_06457_b200.projection import CvaDevice, class_index

    cfg = _scaled("cfg4", 320, 256, 200)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    whole = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
    whole.run()
    ref = whole.check()
    ids, cls = class_index(scene.labels)
    for G in (2, 4, 8):
        fit = CvaDevice(cfg.bands, len(ids), stack.planes.device, groups=G)
        mlen = fit.mlen
        for g in range(G):
            r0, r1 = ut.row_bounds(cfg.height, G, g)
            own = ut.route_points(scene.ys, r0, r1 - r0)
            part = CvaDevice(cfg.bands, len(ids), stack.planes.device)
            if len(own):
                vals = torch.from_numpy(oracle.assemble(stack.planes.cpu().numpy(),
                                                        scene.xs[own], scene.ys[own])).cuda()
                part.moments_from(vals, vals.shape[1], torch.from_numpy(cls[own]).cuda(), len(own))
            fit.moments[g * len(ids) * mlen:(g + 1) * len(ids) * mlen] = part.local_moments()
        fit.solve(1e-8)
        h = fit.host()
        assert np.array_equal(h["counts"], ref["counts"])
        assert rel_close(h["within"], ref["within"], 1e-12)
        assert rel_close(h["between"], ref["between"], 1e-12)
        assert eig_close(h["evals"], ref["evals"], 1e-10)


def test_sharded_projection_minmax():
    """Row shards projected separately: MAX-combining their [-min, max]
    records reproduces the whole-image record, and the stretched shards equal
    the whole-image codes."""
    cfg = _scaled("cfg3", 300, 200, 100)
    scene = synthetic.make_scene(cfg)
    whole = synthetic.generate(scene)
    pipe = ut.CvaPipeline(whole, scene.xs, scene.ys, scene.labels, k=3)
    pipe.run()
    from paper_1612_06457_b200.projection import project_device
    from paper_1612_06457_b200.rendering import stretch_planes
    recs, parts = [], []
    for g in range(3):
        r0, r1 = ut.row_bounds(cfg.height, 3, g)
        shard = synthetic.generate(scene, row0=r0, rows=r1 - r0)
        assert torch.equal(shard.planes, whole.planes[:, r0:r1])
        s, mm, _ = project_device(shard, pipe.evecs, pipe.mean, None, range(3))
        recs.append(mm)
        parts.append(s)
    combined = torch.stack(recs).max(dim=0).values
    assert torch.equal(combined, pipe.minmax)
    for g, s in enumerate(parts):
        r0, r1 = ut.row_bounds(cfg.height, 3, g)
        assert torch.equal(s, pipe.scores[:, r0:r1])
        codes = stretch_planes(s, combined)
        assert torch.equal(codes, pipe.codes[:, r0:r1])


def test_device_class_map_matches_host():
    from paper_1612_06457_b200 import _lib
    import ctypes as C
    cfg = _scaled("cfg3", 700, 500, 10)
    scene = synthetic.make_scene(cfg)
    rng = np.random.default_rng(0)
    ys = rng.integers(0, cfg.height, 5000)
    xs = rng.integers(0, cfg.width, 5000)
    xy = torch.from_numpy(np.stack([xs, ys], 1).astype(np.int32)).cuda()
    out = torch.empty(5000, dtype=torch.int32, device="cuda")
    shp = np.ascontiguousarray(scene.shapes)
    _lib.check(_lib.lib().ut_class_of(shp.ctypes.data_as(C.c_void_p), len(shp), xy.data_ptr(),
                                      5000, out.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "class_of")
    assert np.array_equal(out.cpu().numpy(), synthetic.class_map_at(scene.shapes, ys, xs))


# ------------------------------------------------------ full-size properties

def test_cfg3_full_size_properties():
    """cfg 3 at full size (7216 x 5412 x 23 u16): the fused pipeline against
    the oracle on a sample of rows, with the device model; min/max record ==
    true plane extrema; codes == oracle stretch of the device planes."""
    cfg = synthetic.CONFIGS["cfg3"]
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
    codes = pipe.run()
    model = pipe.model()
    # oracle fit from the same training pixels (gathered on the host)
    host_rows = lambda t: np.concatenate(  # noqa: E731  (no uint16 gather on CUDA)
        [t[:, 0:64].cpu().numpy(), t[:, 3000:3064].cpu().numpy(),
         t[:, cfg.height - 64:].cpu().numpy()], axis=1)
    sample = host_rows(stack.planes)
    design = np.stack([stack.planes[:, int(y), int(x)].cpu().numpy()
                       for x, y in zip(scene.xs[:50], scene.ys[:50])], axis=1)
    xy = torch.from_numpy(np.stack([scene.xs[:50], scene.ys[:50]], 1).astype(np.int32)).cuda()
    gathered, bad = ut.annotations.gather(stack, xy, 50)
    assert np.array_equal(design, gathered.cpu().numpy()) and int(bad.item()) == -1
    ref_scores = oracle.project(sample, {"mean": model.mean, "std": None,
                                         "coefficients": model.coefficients})
    dev_scores = host_rows(pipe.scores).astype(np.float64)
    dev_codes = host_rows(codes)
    assert plane_close(dev_scores, ref_scores) <= SCORE_TOL
    for j in range(cfg.k):
        lo = float(pipe.scores[j].min())
        hi = float(pipe.scores[j].max())
        assert -float(pipe.minmax[j]) == lo and float(pipe.minmax[cfg.k + j]) == hi
        want = oracle.linear_to_codes(dev_scores[j], lo, hi)
        assert np.array_equal(dev_codes[j], want)
        assert int(codes[j].min()) == 0 and int(codes[j].max()) == 255


def test_stretch_ties_and_boundaries_bit_exact():
    """K5's fp32 fast path must reproduce the reference fp64 rounding exactly,
    including ties (x.5 -> away from zero) and values next to them."""
    from paper_1612_06457_b200.rendering import stretch_planes

    rng = np.random.default_rng(7)
    ties = np.arange(0.0, 255.0, 0.5, dtype=np.float32)
    near = np.nextafter(ties, np.float32(np.inf)).astype(np.float32)
    below = np.nextafter(ties, np.float32(-np.inf)).astype(np.float32)
    rand = rng.uniform(-3, 300, size=4096).astype(np.float32)
    vals = np.concatenate([ties, near, below, rand, [np.float32(0), np.float32(255)]])
    pad = (-len(vals)) % 16
    vals = np.concatenate([vals, np.full(pad, 17.25, np.float32)])
    for lo, hi in ((0.0, 255.0), (-3.0, 300.0), (1.5, 2.75)):
        plane = np.clip(vals, lo, hi).astype(np.float32)
        lo32, hi32 = float(plane.min()), float(plane.max())
        scores = torch.from_numpy(plane.reshape(1, 1, -1)).cuda()
        mm = torch.tensor([-lo32, hi32], dtype=torch.float32, device="cuda")
        got = stretch_planes(scores, mm).cpu().numpy().reshape(-1)
        want = oracle.linear_to_codes(plane.astype(np.float64), lo32, hi32)
        assert np.array_equal(got, want), (lo, hi)
        got16 = stretch_planes(scores, mm, depth=16).cpu().numpy().reshape(-1)
        want16 = oracle.linear_to_codes(plane.astype(np.float64), lo32, hi32, 16)
        assert np.array_equal(got16, want16), (lo, hi)


@pytest.mark.parametrize("dtype", [np.float32, np.float16, np.uint16, np.uint8, np.float64])
def test_fp64_projector_widening_exact(dtype):
    """The fp64 projector widens samples without F2F/I2F (bit tricks); check it
    against the oracle on awkward values: zeros, negatives, large magnitudes."""
    rng = np.random.default_rng(21)
    shape = (5, 33, 47)
    if dtype in (np.uint16, np.uint8):
        top = 65535 if dtype == np.uint16 else 255
        cube = rng.integers(0, top + 1, size=shape).astype(dtype)
        cube[:, 0, :] = 0
        cube[:, 1, :] = top
    else:
        cube = (rng.normal(size=shape) * 100).astype(dtype)
        cube[:, 0, :5] = 0
        cube[:, 2, :3] = -0.0
        cube[1, 3, :4] = 1e-3
    coef = rng.normal(size=(5, 3))
    mean = rng.normal(size=5)
    model = ut.ProjectionModel("cva", mean, None, coef, np.ones(3))
    depth = 16 if dtype == np.uint16 else 8
    stack = ut.SpectralStack(ut.stack.default_bands(5), cube, depth, normalized=True) \
        if dtype in (np.uint16, np.uint8) else None
    if stack is None:
        ds = ut.DeviceStack(ut.stack.default_bands(5), torch.from_numpy(cube).cuda(), 8, True)
        planes = [p.values.double().cpu().numpy() for p in ut.project_stack(ds, model,
                                                                              precision="fp64")]
    else:
        planes = [p.values for p in ut.project_stack(stack, model, precision="fp64")]
    ref = oracle.project(cube, {"mean": mean, "std": None, "coefficients": coef})
    for got, want in zip(planes, ref):
        rng_ = float(want.max() - want.min())
        assert float(np.abs(got - want).max()) <= 1e-7 * rng_


def test_cuda_graph_replay_matches_eager():
    cfg = _scaled("cfg1", 256, 256, 100)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
    eager = pipe.run().clone()
    scores = pipe.scores.clone()
    pipe.capture()
    pipe.codes.zero_()
    pipe.scores.zero_()
    pipe.replay()
    torch.cuda.synchronize()
    assert torch.equal(pipe.codes, eager) and torch.equal(pipe.scores, scores)
    pca = ut.PcaPipeline(stack, k=2)
    e2 = pca.run().clone()
    pca.capture()
    pca.codes.zero_()
    pca.replay()
    torch.cuda.synchronize()
    assert torch.equal(pca.codes, e2)


def test_device_stack_api_paths():
    cfg = _scaled("cfg4", 96, 80, 40)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    ts = ut.TrainingSet.from_arrays(scene.xs, scene.ys, scene.labels)
    dm = ut.assemble_matrix(stack, ts)          # stays in HBM
    assert dm.on_device
    model = ut.fit_cva(dm, k=cfg.k)
    planes = ut.project_stack(stack, model)     # DeviceScorePlanes
    assert isinstance(planes[0], ut.DeviceScorePlane)
    host = stack.planes.cpu().numpy()
    ref = oracle.project(host, {"mean": model.mean, "std": None,
                                "coefficients": model.coefficients})
    for p, r in zip(planes, ref):
        lo, hi = p.range()
        assert lo == float(p.values.min()) and hi == float(p.values.max())
        codes = ut.rescale_full(p).cpu().numpy()
        assert np.array_equal(codes, oracle.rescale_full(p.values.double().cpu().numpy()))
        assert float(np.abs(p.values.double().cpu().numpy() - r).max()) <= 1e-6 * (r.max() - r.min())
    hm = ut.fit_cva(ut.assemble_matrix(ut.SpectralStack(stack.bands, host, 8, True), ts),
                    k=cfg.k)
    assert np.allclose(hm.coefficients, model.coefficients, atol=1e-12)
    # fit dispatch
    m2 = ut.fit("pca_unsupervised", stack=stack, k=2)
    assert m2.method == "pca_unsupervised" and m2.coefficients.shape == (cfg.bands, 2)
    with pytest.raises(ut.DataError):
        ut.fit("nope", dm=dm)


@pytest.mark.parametrize("k,npix", [(3, 8192 * 2 + 48), (1, 16), (32, 8192 + 4096 + 16), (5, 3 * 8192)])
def test_stretch_ring_multiplane_tails(k, npix):
    """K5's bulk-copy ring over several planes with partial last tiles (32 KB
    tiles of 8192 scores), 8- and 16-bit codes, against the oracle."""
    from paper_1612_06457_b200.rendering import stretch_planes

    rng = np.random.default_rng(k * 1000 + npix % 977)
    planes = rng.normal(0, 3, size=(k, npix)).astype(np.float32)
    planes[0, ::5] = 1.25                                  # repeated values / ties
    lo = planes.min(axis=1).astype(np.float32)
    hi = planes.max(axis=1).astype(np.float32)
    if k > 1:
        planes[1] = 4.0                                    # a constant plane -> zeros
        lo[1] = hi[1] = 4.0
    scores = torch.from_numpy(planes.reshape(k, 1, npix)).cuda()
    mm = torch.from_numpy(np.concatenate([-lo, hi]).astype(np.float32)).cuda()
    for depth in (8, 16):
        got = stretch_planes(scores, mm, depth=depth).cpu().numpy().reshape(k, npix)
        for c in range(k):
            if lo[c] == hi[c]:
                assert not got[c].any()
                continue
            want = oracle.linear_to_codes(planes[c].astype(np.float64), float(lo[c]), float(hi[c]),
                                          depth)
            assert np.array_equal(got[c], want), (c, depth)


@pytest.mark.parametrize("bands,k", [(23, 5), (5, 4), (32, 8), (17, 6)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_dmma_projector_padded_bands(bands, k, dtype):
    """The fp64 tensor-core projector (K >= 4, 4/8-byte samples) with band counts
    that are not multiples of 4: the padded lanes read band 0 and must add
    nothing (zero weights); awkward values (zeros, -0, subnormal, large)."""
    rng = np.random.default_rng(bands * 10 + k)
    cube = (rng.normal(size=(bands, 29, 64)) * 50).astype(dtype)
    cube[:, 0, :7] = 0
    cube[:, 1, :5] = -0.0
    cube[0, 2, :3] = np.finfo(dtype).tiny / 4           # subnormal
    cube[1 % bands, 3, :2] = 1e6
    coef = rng.normal(size=(bands, k))
    mean = rng.normal(size=bands)
    model = ut.ProjectionModel("cva", mean, None, coef, np.ones(k))
    ds = ut.DeviceStack(ut.stack.default_bands(bands), torch.from_numpy(cube).cuda(), 8, True)
    planes = [p.values.double().cpu().numpy() for p in ut.project_stack(ds, model, precision="fp64")]
    ref = oracle.project(cube, {"mean": mean, "std": None, "coefficients": coef})
    for got, want in zip(planes, ref):
        rng_ = float(want.max() - want.min())
        assert float(np.abs(got - want).max()) <= 1e-7 * rng_


@pytest.mark.parametrize("bands", [23, 32])
def test_dmma_projector_nonfinite_band0(bands):
    """A NaN / Inf in band 0 (the band the padded lanes read) is reported."""
    rng = np.random.default_rng(5)
    coef = rng.normal(size=(bands, 5))
    model = ut.ProjectionModel("cva", np.zeros(bands), None, coef, np.ones(5))
    for bad in (np.nan, np.inf):
        cube = rng.normal(size=(bands, 16, 64)).astype(np.float32)
        cube[0, 7, 9] = bad
        ds = ut.DeviceStack(ut.stack.default_bands(bands), torch.from_numpy(cube).cuda(), 8, True)
        with pytest.raises(ut.DataError, match="NaN or Inf"):
            ut.project_stack(ds, model, precision="fp64")


@pytest.mark.parametrize("n", [37887, 37888, 37889, 75776, 75777])
def test_class_moments_partition_boundaries(n):
    """K1 splits n points into one 128-point chunk per CTA up to 296 CTAs and
    two-chunk CTAs above (moments.cu make_layout); both regimes, the exact
    boundary and ragged last ranges match the oracle's two-pass scatter."""
    rng = np.random.default_rng(n)
    b = 32
    values = 0.5 + 0.05 * rng.standard_normal((b, n))
    labels = rng.integers(0, 6, n)
    values[:, labels == 3] += 0.1  # distinct class means
    sp = ut.compute_scatter(dm_of(values, labels))
    want = oracle.scatter(values, labels)
    assert np.array_equal(sp.counts, want["counts"])
    for got, key in ((sp.within, "within"), (sp.between, "between"),
                     (sp.class_means, "class_means"), (sp.grand_mean, "grand_mean")):
        assert rel_close(got, want[key], 1e-9), key


@pytest.mark.parametrize("b,classes,n", [(9, 20, 1000), (32, 17, 4590), (1, 3, 130), (23, 6, 127)])
def test_class_moments_mixed_chunks(b, classes, n):
    """Points in caller order (every 128-point chunk holds several classes: one
    masked tensor-core pass per class present), more than 16 classes (two K1
    launches), band counts off the 8-row groups."""
    rng = np.random.default_rng(1000 * b + classes)
    values = rng.uniform(0.0, 1.0, (b, n)) * rng.uniform(0.5, 2.0, (b, 1))
    labels = rng.integers(0, classes, n)
    labels[:classes] = np.arange(classes)   # every class present
    values += 0.05 * labels[None, :]
    sp = ut.compute_scatter(dm_of(values, labels))
    want = oracle.scatter(values, labels)
    assert np.array_equal(sp.counts, want["counts"])
    for got, key in ((sp.within, "within"), (sp.between, "between"),
                     (sp.class_means, "class_means"), (sp.grand_mean, "grand_mean")):
        assert rel_close(got, want[key], 1e-9), key
