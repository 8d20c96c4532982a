"""The §8(f) rows on the device: normalize_stack (stack.py:180-213) and the
training-range / percentile stretch modes (rendering.py:133-179), against the
golden vectors of the real reference and the oracle: codes bit-exact."""

import math
import warnings

import numpy as np
import pytest

import oracle
from golden_util import load

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402

NORMALIZE_CASES = ["u8", "u16", "u16_span", "f32", "f64_ties", "const"]


def host_stack(planes, depth, normalized=False):
    return ut.SpectralStack(ut.stack.default_bands(planes.shape[0]), planes, depth, normalized)


@pytest.mark.parametrize("key", NORMALIZE_CASES)
@pytest.mark.parametrize("scope", ["per-band", "global"])
def test_normalize_golden(key, scope):
    g = load("normalize")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = ut.normalize_stack(host_stack(g[f"{key}_in"], int(g[f"{key}_depth"])), scope)
    assert out.normalized and out.bit_depth == 8 and out.planes.dtype == np.uint8
    assert np.array_equal(out.planes, g[f"{key}_{scope}"])


def test_normalize_warnings_and_errors():
    planes = np.stack([np.full((4, 5), 7, np.uint8), np.arange(20, dtype=np.uint8).reshape(4, 5)])
    with pytest.warns(ut.UndertextWarning, match="band 0 is constant \\(value 7\\)"):
        out = ut.normalize_stack(host_stack(planes, 8))
    assert out.planes[0].max() == 0 and out.planes[1].max() == 255
    with pytest.raises(ut.DataError, match="already normalized"):
        ut.normalize_stack(host_stack(planes, 8, normalized=True))
    with pytest.raises(ut.DataError, match="scope"):
        ut.normalize_stack(host_stack(planes, 8), scope="per-pixel")


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.float16, np.float32, np.float64])
def test_normalize_device_large_vs_oracle(dtype):
    rng = np.random.default_rng(11)
    shape = (5, 301, 517)                      # odd sizes: the scalar path
    if dtype == np.uint8:
        planes = rng.integers(0, 256, size=shape).astype(dtype)
    elif dtype == np.uint16:
        planes = rng.integers(0, 65536, size=shape).astype(dtype)
    else:
        planes = rng.uniform(0, 250, size=shape).astype(dtype)
    ds = ut.DeviceStack(ut.stack.default_bands(5), torch.from_numpy(planes).cuda(),
                        16 if dtype == np.uint16 else 8, False)
    for scope in ("per-band", "global"):
        got = ut.normalize_stack(ds, scope)
        assert isinstance(got, ut.DeviceStack) and got.normalized
        want, _ = oracle.normalize_stack(planes, scope)
        assert np.array_equal(got.planes.cpu().numpy(), want)


def test_normalize_contiguous_vector_path_and_strided_view():
    rng = np.random.default_rng(12)
    planes = rng.integers(0, 4096, size=(3, 64, 128)).astype(np.uint16)   # 16-aligned
    t = torch.from_numpy(planes).cuda()
    got = ut.normalize_stack(ut.DeviceStack(ut.stack.default_bands(3), t, 16, False))
    assert np.array_equal(got.planes.cpu().numpy(), oracle.normalize_stack(planes)[0])
    view = t[:, 5:50, 3:101]                                              # row_stride != cols
    got = ut.normalize_stack(ut.DeviceStack(ut.stack.default_bands(3), view, 16, False))
    want = oracle.normalize_stack(np.ascontiguousarray(planes[:, 5:50, 3:101]))[0]
    assert np.array_equal(got.planes.cpu().numpy(), want)


def test_normalize_nan_band_gives_zeros():
    planes = np.random.default_rng(13).uniform(0, 1, size=(2, 8, 16)).astype(np.float32)
    planes[1, 3, 3] = np.nan
    ds = ut.DeviceStack(ut.stack.default_bands(2), torch.from_numpy(planes).cuda(), 8, False)
    got = ut.normalize_stack(ds).planes.cpu().numpy()
    assert not got[1].any()
    assert np.array_equal(got[0], oracle.normalize_stack(planes[:1])[0][0])


def _model(scores):
    scores = np.asarray(scores, dtype=np.float64)
    return ut.ProjectionModel("cva", np.zeros(2), None, np.ones((2, scores.shape[0])),
                              np.ones(scores.shape[0]), training_scores=scores)


def test_training_range_golden_and_reference_cases():
    g = load("rescale_modes")
    model = _model(g["training_scores"])
    for k in range(3):
        assert np.array_equal(ut.rescale_training_range(ut.ScorePlane(g["plane"]), model, k),
                              g[f"train_k{k}_u8"])
        assert np.array_equal(ut.rescale_training_range(g["plane"], model, k, depth=16),
                              g[f"train_k{k}_u16"])
    # tests/test_rendering.py:117-141 of the reference
    assert ut.rescale_training_range([[5.0, 12.0, -3.0]], _model([[0.0, 10.0]]), 0).tolist() == \
        [[128, 255, 0]]
    assert ut.rescale_training_range([[10.0]], _model([[0.0, 10.0], [0.0, 20.0]]), 1).tolist() == \
        [[128]]
    with pytest.raises(ut.DataError):
        ut.rescale_training_range([[0.0]], _model([[0.0, 1.0]]), 1)
    with pytest.warns(ut.UndertextWarning):
        out = ut.rescale_training_range([[1.0, 9.0]], _model([[4.0, 4.0]]), 0)
    assert not out.any()
    no_scores = ut.ProjectionModel("pca_unsupervised", np.zeros(2), np.ones(2), np.eye(2),
                                   np.ones(2))
    with pytest.raises(ut.DataError, match="training"):
        ut.rescale_training_range([[0.0]], no_scores, 0)


def test_percentile_golden():
    g = load("rescale_modes")
    plane = ut.ScorePlane(g["plane"])
    for p in (0.01, 0.1, 1.0, 5.0):
        tag = str(p).replace(".", "_")
        assert np.array_equal(ut.rescale_percentile(plane, p), g[f"pct_{tag}"])
        assert np.array_equal(ut.rescale_percentile(plane, p, one_tail=True), g[f"pct_{tag}_one"])
        assert np.array_equal(ut.rescale_percentile(plane, p, depth=16), g[f"pct_{tag}_u16"])
    assert np.array_equal(ut.rescale_percentile(g["lin"], 5.0), g["lin_p5"])


def test_percentile_reference_cases():
    # tests/test_rendering.py:173-198 of the reference
    rng = np.random.default_rng(3)
    plane = ut.ScorePlane(rng.normal(size=(10, 10)))
    assert np.array_equal(ut.rescale_percentile(plane, 0.01), ut.rescale_full(plane))
    values = np.linspace(0.0, 1.0, 100).reshape(10, 10)
    out = ut.rescale_percentile(values, 5.0, one_tail=True)
    assert out[0, 0] == 0 and int((out == 0).sum()) == 1 and int((out == 255).sum()) > 1
    with pytest.raises(ut.DataError):
        ut.rescale_percentile([[0.0, 1.0]], 2.5)
    values = np.full((10, 10), 7.0)
    values[0, 0], values[9, 9] = 0.0, 50.0
    with pytest.warns(ut.UndertextWarning):
        out = ut.rescale_percentile(values, 5.0)
    assert not out.any()


@pytest.mark.parametrize("n", [1, 2, 3, 1000, 65537, 1 << 20])
def test_select_exact_order_statistics_fp32_and_fp64(n):
    rng = np.random.default_rng(n)
    v = rng.normal(size=n) * np.exp(rng.uniform(-5, 5, size=n))
    v[rng.integers(0, n, size=max(1, n // 10))] = v[0]  # duplicates
    if n > 4:
        v[:3] = [-0.0, 0.0, -0.0]
    for dtype in (np.float32, np.float64):
        x = v.astype(dtype)
        srt = np.sort(x.astype(np.float64))
        for p in (0.01, 1.0, 5.0):
            r_lo = max(1, math.ceil(p / 100.0 * n))
            r_hi = max(1, math.ceil((100.0 - p) / 100.0 * n))
            t = torch.from_numpy(x).cuda()
            out = torch.empty(2, dtype=torch.float64, device="cuda")
            from paper_1612_06457_b200 import _lib
            from paper_1612_06457_b200 import device as dev
            import ctypes as C
            L = _lib.lib()
            ws = dev.workspace("plane_select", L.ut_plane_select_ws(), t.device)
            ranks = (C.c_int64 * 2)(r_lo, r_hi)
            dt = _lib.UT_F32 if dtype == np.float32 else _lib.UT_F64
            _lib.check(L.ut_plane_select(t.data_ptr(), dt, n, ranks, out.data_ptr(), ws.data_ptr(),
                                         ws.numel(), dev.stream_handle()), "select")
            lo, hi = out.cpu().numpy()
            assert lo == srt[r_lo - 1] and hi == srt[r_hi - 1], (dtype, p)


def test_percentile_on_device_plane_matches_host_codes():
    """DeviceScorePlane (the pipeline's fp32 planes): same codes as the oracle
    applied to the same fp32 values."""
    from dataclasses import replace
    from paper_1612_06457_b200 import synthetic
    cfg = replace(synthetic.scaled(synthetic.CONFIGS["cfg4"], 300, 257, 60))
    scene = synthetic.make_scene(cfg)
    pipe = ut.CvaPipeline(synthetic.generate(scene), scene.xs, scene.ys, scene.labels, k=cfg.k)
    pipe.run()
    for j in range(cfg.k):
        dp = ut.DeviceScorePlane(pipe.scores, pipe.minmax, j)
        host = pipe.scores[j].double().cpu().numpy()
        for p, one in ((1.0, False), (5.0, True), (0.1, False)):
            got = ut.rescale_percentile(dp, p, one_tail=one).cpu().numpy()
            assert np.array_equal(got, oracle.rescale_percentile(host, p, one_tail=one))
        spec = ut.RenderSpec("percentile", 1.0)
        assert np.array_equal(ut.rescale(dp, spec).cpu().numpy(), oracle.rescale_percentile(host, 1.0))


def _select(x, r_lo, r_hi):
    import ctypes as C
    from paper_1612_06457_b200 import _lib
    from paper_1612_06457_b200 import device as dev
    t = torch.from_numpy(x).cuda()
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    ws = dev.workspace("plane_select", L.ut_plane_select_ws(), t.device)
    ranks = (C.c_int64 * 2)(r_lo, r_hi)
    dt = _lib.UT_F32 if x.dtype == np.float32 else _lib.UT_F64
    _lib.check(L.ut_plane_select(t.data_ptr(), dt, x.size, ranks, out.data_ptr(), ws.data_ptr(),
                                 ws.numel(), dev.stream_handle()), "select")
    return out.cpu().numpy()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_select_sample_blind_spots_fall_back(dtype):
    """A plane whose strided sample sees only one value: the candidate window
    misses the ranks and the full radix select (device-gated) must take over."""
    n = 16384 * 64
    rng = np.random.default_rng(21)
    x = rng.normal(size=n).astype(dtype)
    x[::64] = 0.5                       # exactly the positions the sample reads
    srt = np.sort(x.astype(np.float64))
    for r_lo, r_hi in ((1, n), (n // 100, n - n // 100), (n // 2, n // 2 + 1)):
        lo, hi = _select(x, r_lo, r_hi)
        assert lo == srt[r_lo - 1] and hi == srt[r_hi - 1]


def test_select_heavy_duplicates_and_window_overflow():
    n = 1 << 23
    x = np.zeros(n, np.float32)         # > kCandCap equal keys inside one window
    x[:1000] = np.linspace(-1, 1, 1000, dtype=np.float32)
    srt = np.sort(x.astype(np.float64))
    for r_lo, r_hi in ((1, n), (500, n // 2), (n - 10, 3)):
        lo, hi = _select(x, r_lo, r_hi)
        assert lo == srt[r_lo - 1] and hi == srt[r_hi - 1]
