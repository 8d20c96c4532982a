"""K2 region moments on the device (ut_region_moments) against an exact
numpy restatement of the reference's two-pass statistics
(projection.py:327-334): n, per-band mean and the centred Gram M2.  Whole-width
regions of 8/16/32-bit samples take the exact-integer tensor-core path
(tcgen05 kind::i8); samples outside its fixed-point range (outliers, NaN) make
it hand the region to the fp64 tensor-core path -- both must agree with the
reference to 1e-12 of the largest entry."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200.projection import PcaDevice  # noqa: E402


@pytest.fixture(autouse=True)
def integer_path_for_all_band_counts(monkeypatch):
    """The library takes the integer path from 17 bands up; the tests drive it
    at every band count (the cut is read per call)."""
    monkeypatch.setenv("UT_IMMA_MIN_BANDS", "1")


def moments(cube: np.ndarray, region=None):
    t = torch.from_numpy(cube).cuda()
    ds = ut.DeviceStack(ut.stack.default_bands(cube.shape[0]), t,
                        16 if cube.dtype == np.uint16 else 8, True)
    b, h, w = cube.shape
    x0, y0, rw, rh = region or (0, 0, w, h)
    pd = PcaDevice(b, t.device)
    pd.moments_from(ds.cube(), x0, y0, rw, rh, t.device)
    m = pd.local_moments().cpu().numpy()
    return m[0], m[1:1 + b], m[1 + b:].reshape(b, b)


def reference(cube, region=None):
    b, h, w = cube.shape
    x0, y0, rw, rh = region or (0, 0, w, h)
    x = cube[:, y0:y0 + rh, x0:x0 + rw].reshape(b, -1).astype(np.float64)
    mean = x.mean(axis=1)
    d = x - mean[:, None]
    return x.shape[1], mean, d @ d.T


def check(cube, region=None, tol=1e-12):
    n, mean, m2 = moments(cube, region)
    rn, rmean, rm2 = reference(cube, region)
    assert n == rn
    assert np.max(np.abs(mean - rmean)) <= 1e-14 * max(1.0, np.abs(rmean).max())
    assert np.max(np.abs(m2 - rm2)) <= tol * np.abs(rm2).max(), np.max(np.abs(m2 - rm2))
    return m2


def sample_cube(rng, dtype, b, h, w):
    mu = rng.uniform(0.2, 0.8, size=(b, 1, 1))
    x = np.clip(mu + rng.normal(scale=0.035, size=(b, h, w)), 0, 1)
    if dtype == np.uint8:
        return np.floor(255 * x + 0.5).astype(np.uint8)
    if dtype == np.uint16:
        return np.floor(4095 * x + 0.5).astype(np.uint16)
    return x.astype(dtype)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.float16, np.float32])
@pytest.mark.parametrize("b", [1, 5, 16, 23, 32])
@pytest.mark.parametrize("hw", [(40, 100), (64, 64), (3, 4096)])
def test_region_moments_whole_width(dtype, b, hw):
    rng = np.random.default_rng(b * 1000 + hw[0])
    check(sample_cube(rng, dtype, b, *hw))


def test_region_moments_wide_dynamic_range():
    """float samples spanning many binades (small values below the grid) and
    negative values: the integer path rounds samples below its grid 2^-f (set
    from 4x the sampled spread), so M2 is good to the parity bar here, not to
    the last bits; the mean is exact (fp64 sums)."""
    rng = np.random.default_rng(1)
    x = rng.normal(size=(7, 64, 96)) * np.exp(rng.uniform(-12, 2, size=(7, 64, 96)))
    check(x.astype(np.float32), tol=1e-9)  # the parity bar: grid rounding of the tail


def test_region_moments_outlier_takes_fp64_path():
    rng = np.random.default_rng(2)
    cube = sample_cube(rng, np.float32, 6, 128, 96)
    cube[3, 77, 41] = 1.0e6    # far outside the sampled spread -> fixed-point overflow
    cube[0, 5, 5] = -3.0e5
    check(cube, tol=1e-10)


def test_region_moments_many_windows_and_determinism():
    """> 2^16 pixels per CTA: several TMEM windows folded into the int64 record."""
    rng = np.random.default_rng(3)
    cube = sample_cube(rng, np.uint8, 3, 2560, 4096)   # 10.5 M pixels
    m1 = check(cube)
    _, _, m2 = moments(cube)
    assert np.array_equal(m1, m2)


def test_region_moments_f32_many_windows():
    rng = np.random.default_rng(4)
    cube = sample_cube(rng, np.float32, 4, 2048, 5120)  # 10.5 M pixels
    check(cube)


def test_region_moments_subregion_uses_fallback_paths():
    rng = np.random.default_rng(5)
    cube = sample_cube(rng, np.float32, 9, 50, 70)
    for region in [(3, 4, 40, 30), (0, 10, 70, 20), (69, 0, 1, 50)]:
        check(cube, region, tol=1e-11)


def test_region_moments_nan_propagates():
    cube = np.full((2, 16, 16), 0.5, np.float32)
    cube[1] += np.linspace(0, 0.1, 256, dtype=np.float32).reshape(16, 16)
    cube[1, 9, 9] = np.nan
    _, mean, m2 = moments(cube)
    assert np.isnan(mean[1]) and np.isnan(m2[1, 1])
    assert not np.isnan(mean[0])


def test_pca_fit_integer_path_matches_oracle():
    import oracle
    rng = np.random.default_rng(6)
    cube = sample_cube(rng, np.float32, 32, 256, 512)
    pm = ut.fit_pca_unsupervised(ut.DeviceStack(ut.stack.default_bands(32),
                                                torch.from_numpy(cube).cuda(), 8, True), k=4)
    ref = oracle.fit_pca_unsupervised(cube, k=4)
    assert np.allclose(pm.mean, ref["mean"], rtol=1e-13, atol=0)
    assert np.allclose(pm.std, ref["std"], rtol=1e-11, atol=0)
    assert np.allclose(pm.eigenvalues, ref["eigenvalues"], rtol=1e-10, atol=0)


@pytest.mark.parametrize("dtype", [np.uint16, np.float32])
def test_integer_and_fp64_paths_agree(dtype, monkeypatch):
    rng = np.random.default_rng(7)
    cube = sample_cube(rng, dtype, 24, 96, 160)
    n1, m1, g1 = moments(cube)
    monkeypatch.setenv("UT_REGION_IMMA", "0")
    n2, m2, g2 = moments(cube)
    assert n1 == n2
    assert np.max(np.abs(m1 - m2)) <= 1e-14 * np.abs(m2).max()
    assert np.max(np.abs(g1 - g2)) <= 1e-12 * np.abs(g2).max()
