"""The reference's own hot-path test suite, restated against the drop-in on the GPU.

SURVEY.md §4 item 1 / round-1 VERDICT "missing #2": the reference's tests for
this path -- tests/test_projection.py, test_eigen.py, test_quantize.py,
test_rendering.py::TestFullRange and test_acceptance.py criteria 1-4, 8, 10 --
cannot run on the GPU box (the reference does not travel there), so each case
is restated here: same inputs where they are hand-written, the same property on
freshly seeded data where the reference draws random data, the same tolerance.
Class and test names follow the reference's; each docstring cites the case.
Everything goes through the drop-in's public functions (device kernels behind
the C ABI).
"""

from __future__ import annotations

import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as b  # noqa: E402
from golden_util import load  # noqa: E402


# -- helpers (own code; the reference's oracles.py plays the same role) --------
def dm(values, labels, names=None):
    values = np.asarray(values, dtype=np.float64)
    labels = np.asarray(labels, dtype=np.intp)
    if names is None:
        names = tuple(f"c{i}" for i in range(int(labels.max()) + 1))
    return b.DesignMatrix(values, labels, names)


def labeled(rng, bands, classes, per_class):
    """Gaussian clouds with random class offsets (B x N values, N labels)."""
    centres = rng.normal(scale=3.0, size=(classes, bands))
    values = np.concatenate([centres[c][:, None] + rng.normal(size=(bands, per_class))
                             for c in range(classes)], axis=1)
    labels = np.repeat(np.arange(classes), per_class)
    return values, labels


def sym(rng, n, scale=1.0):
    r = rng.normal(size=(n, n)) * scale
    return (r + r.T) / 2.0


def spd(rng, n, floor=0.5):
    r = rng.normal(size=(n, n))
    return r @ r.T + floor * np.eye(n)


def rayleigh(v, a, m):
    return float(v @ a @ v) / float(v @ m @ v)


def stack_of(planes, normalized=True):
    planes = np.asarray(planes, dtype=np.uint8)
    return b.SpectralStack(b.stack.default_bands(planes.shape[0]), planes, 8, normalized)


def model(coef, mean=None, **kw):
    coef = np.asarray(coef, dtype=np.float64)
    return b.ProjectionModel(method="cva", mean=np.zeros(coef.shape[0]) if mean is None else mean,
                             std=None, coefficients=coef, eigenvalues=np.ones(coef.shape[1]), **kw)


def values_of(plane):
    v = plane.values
    return v.double().cpu().numpy() if torch.is_tensor(v) else np.asarray(v, dtype=np.float64)


@pytest.fixture(scope="module")
def small_stack():
    """The reference's small_page fixture (96 x 96 x 6, normalized; conftest.py:7-15),
    from the golden file generated with the reference."""
    g = load("small_page")
    return b.SpectralStack(b.stack.default_bands(g["cube"].shape[0]), g["cube"], 8, True)


# ---------------------------------------------------- test_projection.py
class TestStandardize:
    def test_hand_example(self):
        """test_projection.py:37-41"""
        out, mean, std = b.standardize(dm([[1.0, 3.0]], [0, 0], ("a",)))
        assert mean.tolist() == [2.0] and std.tolist() == [np.sqrt(2.0)]
        assert np.allclose(np.asarray(out.values), [[-1 / np.sqrt(2), 1 / np.sqrt(2)]])

    def test_constant_row_centred_std_one(self):
        """:43-46"""
        out, _, std = b.standardize(dm([[5.0, 5.0, 5.0]], [0, 0, 0], ("a",)))
        assert np.asarray(out.values).tolist() == [[0.0, 0.0, 0.0]] and std.tolist() == [1.0]

    def test_idempotent_on_standardized_input(self):
        """:48-55"""
        rng = np.random.default_rng(0)
        once, _, _ = b.standardize(dm(rng.normal(size=(3, 40)), [0] * 40, ("a",)))
        twice, mean, std = b.standardize(once)
        assert np.allclose(np.asarray(twice.values), np.asarray(once.values), atol=1e-12)
        assert np.allclose(mean, 0.0, atol=1e-12) and np.allclose(std, 1.0, atol=1e-12)

    def test_needs_two_points(self):
        """:57-59"""
        with pytest.raises(b.DataError):
            b.standardize(dm([[1.0]], [0], ("a",)))


class TestScatter:
    def test_hand_oracle(self):
        """:63-69 -- exact"""
        sp = b.compute_scatter(dm([[0.0, 2.0, 10.0, 12.0]], [0, 0, 1, 1]))
        assert sp.within.tolist() == [[4.0]] and sp.between.tolist() == [[100.0]]
        assert sp.grand_mean.tolist() == [6.0] and sp.class_means.tolist() == [[1.0], [11.0]]

    def test_singleton_classes_zero_within(self):
        """:71-73"""
        assert np.allclose(b.compute_scatter(dm([[1.0, 5.0], [2.0, 3.0]], [0, 1])).within, 0.0)

    def test_identical_means_zero_between(self):
        """:75-78"""
        assert np.allclose(b.compute_scatter(dm([[1.0, 3.0, 1.0, 3.0]], [0, 0, 1, 1])).between, 0.0)

    def test_needs_two_classes(self):
        """:80-82"""
        with pytest.raises(b.DataError):
            b.compute_scatter(dm([[1.0, 2.0]], [0, 0], ("a",)))

    def test_symmetric_and_psd(self):
        """:84-90"""
        v, l = labeled(np.random.default_rng(1), 6, 3, 20)
        sp = b.compute_scatter(dm(v, l))
        assert np.array_equal(sp.within, sp.within.T) and np.array_equal(sp.between, sp.between.T)
        assert np.linalg.eigvalsh(sp.within).min() >= -1e-9


class TestFitCva:
    def test_separable_clouds_recover_axis(self):
        """:94-102"""
        rng = np.random.default_rng(2)
        x = np.concatenate([rng.normal(size=(2, 4000)),
                            np.array([[10.0], [0.0]]) + rng.normal(size=(2, 4000))], axis=1)
        v = b.fit_cva(dm(x, [0] * 4000 + [1] * 4000)).coefficients[:, 0]
        assert abs(v[0]) / np.linalg.norm(v) >= 0.999

    def test_first_direction_beats_random_quotient(self):
        """:104-113"""
        rng = np.random.default_rng(3)
        v, l = labeled(rng, 5, 3, 30)
        sp = b.compute_scatter(dm(v, l))
        top = rayleigh(b.fit_cva(dm(v, l)).coefficients[:, 0], sp.between, sp.within)
        d = rng.normal(size=(10_000, 5))
        q = np.einsum("gi,ij,gj->g", d, sp.between, d) / np.einsum("gi,ij,gj->g", d, sp.within, d)
        assert q.max() <= top * (1 + 1e-9)

    def test_identical_classes_all_eigenvalues_near_zero(self):
        """:115-120"""
        pts = np.array([[0.0, 1.0, 2.0], [5.0, 6.0, 7.0]])
        d = dm(np.concatenate([pts, pts], axis=1), [0, 0, 0, 1, 1, 1])
        scale = np.trace(b.compute_scatter(d).within)
        assert (np.abs(b.fit_cva(d).eigenvalues) <= 1e-10 * scale).all()

    def test_training_scores_consistent_with_apply(self):
        """:122-127 -- bit-exact"""
        v, l = labeled(np.random.default_rng(4), 4, 3, 15)
        m = b.fit_cva(dm(v, l))
        assert np.array_equal(m.apply(v.T), m.training_scores.T)

    def test_k_limits_components(self):
        """:129-136"""
        v, l = labeled(np.random.default_rng(5), 6, 4, 10)
        m = b.fit_cva(dm(v, l), k=2)
        assert m.coefficients.shape == (6, 2) and m.eigenvalues.shape == (2,)
        with pytest.raises(b.DataError):
            b.fit_cva(dm(v, l), k=7)

    def test_eigenvalues_descending(self):
        """:138-142"""
        v, l = labeled(np.random.default_rng(6), 8, 5, 12)
        assert (np.diff(b.fit_cva(dm(v, l)).eigenvalues) <= 1e-12).all()


class TestFitLda:
    def test_requires_exactly_two_classes(self):
        """:146-150"""
        v, l = labeled(np.random.default_rng(7), 3, 3, 10)
        with pytest.raises(b.DataError, match="exactly 2"):
            b.fit_lda(dm(v, l))

    def test_equals_cva_on_standardized_input(self):
        """:152-161 -- bit-exact (the same device kernels on the same matrix)"""
        rng = np.random.default_rng(8)
        for _ in range(10):
            v, l = labeled(rng, 5, 2, 25)
            lda = b.fit_lda(dm(v, l))
            sdm, _, _ = b.standardize(dm(v, l))
            cva = b.fit_cva(sdm)
            assert np.array_equal(lda.coefficients, cva.coefficients)
            assert np.array_equal(lda.eigenvalues, cva.eigenvalues)

    def test_records_standardization(self):
        """:163-168"""
        v, l = labeled(np.random.default_rng(9), 4, 2, 20)
        m = b.fit_lda(dm(v, l))
        assert m.std is not None and np.allclose(m.mean, v.mean(axis=1))

    def test_one_dimensional_input(self):
        """:170-174"""
        m = b.fit_lda(dm([[0.0, 1.0, 10.0, 11.0]], [0, 0, 1, 1]))
        assert m.coefficients.shape == (1, 1) and m.coefficients[0, 0] > 0


class TestFitPca:
    def test_recovers_dominant_direction(self):
        """:178-185"""
        rng = np.random.default_rng(10)
        t = rng.normal(size=400) * 5.0
        pts = np.stack([t, t]) + rng.normal(size=(2, 400)) * 0.1
        v = b.fit_pca(dm(pts, [0] * 400, ("all",))).coefficients[:, 0]
        assert abs(v @ np.array([1.0, 1.0]) / np.sqrt(2.0)) >= 0.999

    def test_orthonormal_basis_and_variance_conservation(self):
        """:187-194"""
        m = b.fit_pca(dm(np.random.default_rng(11).normal(size=(6, 80)), [0] * 80, ("all",)))
        c = m.coefficients
        assert np.allclose(c.T @ c, np.eye(6), atol=1e-10)
        assert np.sum(m.eigenvalues) == pytest.approx(6.0, rel=1e-8)

    def test_matches_correlation_eigensystem(self):
        """:196-202"""
        rng = np.random.default_rng(12)
        v = rng.normal(size=(5, 60)) * rng.uniform(1, 4, size=(5, 1))
        m = b.fit_pca(dm(v, [0] * 60, ("all",)))
        assert np.allclose(m.eigenvalues, np.linalg.eigvalsh(np.corrcoef(v))[::-1], atol=1e-10)

    def test_ignores_labels(self):
        """:204-209"""
        v = np.random.default_rng(13).normal(size=(4, 40))
        m1 = b.fit_pca(dm(v, [0] * 40, ("a",)))
        m2 = b.fit_pca(dm(v, [0] * 20 + [1] * 20, ("a", "b")))
        assert np.array_equal(m1.coefficients, m2.coefficients)


class TestFitPcaUnsupervised:
    def test_component_count(self, small_stack):
        """:213-217"""
        m = b.fit_pca_unsupervised(small_stack, k=5)
        assert m.coefficients.shape == (6, 5) and m.training_scores is None
        assert m.method == "pca_unsupervised"

    def test_matches_supervised_pca_on_same_pixels(self, small_stack):
        """:219-227"""
        x0, y0, w, h = region = (8, 8, 16, 16)
        m = b.fit_pca_unsupervised(small_stack, region=region)
        px = small_stack.planes[:, y0:y0 + h, x0:x0 + w].reshape(6, -1).astype(np.float64)
        ref = b.fit_pca(dm(px, [0] * (w * h), ("all",)))
        assert np.allclose(m.eigenvalues, ref.eigenvalues, atol=1e-9)
        assert np.allclose(m.coefficients, ref.coefficients, atol=1e-8)

    def test_single_pixel_region_rejected(self, small_stack):
        """:229-231"""
        with pytest.raises(b.DataError):
            b.fit_pca_unsupervised(small_stack, region=(0, 0, 1, 1))

    def test_region_bounds_checked(self, small_stack):
        """:233-235"""
        with pytest.raises(b.DataError):
            b.fit_pca_unsupervised(small_stack, region=(90, 90, 16, 16))

    def test_equal_bands_rank_one(self):
        """:237-242"""
        plane = np.arange(64, dtype=np.uint8).reshape(8, 8)
        m = b.fit_pca_unsupervised(stack_of(np.stack([plane, plane, plane])))
        assert m.eigenvalues[0] == pytest.approx(3.0, rel=1e-8)
        assert np.allclose(m.eigenvalues[1:], 0.0, atol=1e-9)


class TestProjectStack:
    def test_identity_model_returns_bands(self):
        """:246-256 -- exact"""
        planes = np.random.default_rng(14).integers(0, 255, size=(3, 12, 9), dtype=np.uint8)
        out = b.project_stack(stack_of(planes), model(np.eye(3)))
        for k in range(3):
            assert np.array_equal(values_of(out[k]), planes[k].astype(np.float64))

    def test_difference_column(self):
        """:258-268 -- exact"""
        planes = np.stack([np.full((4, 4), 9, np.uint8), np.full((4, 4), 3, np.uint8)])
        out = b.project_stack(stack_of(planes), model([[1.0], [-1.0]]))
        assert np.all(values_of(out[0]) == 6.0)

    def test_linearity_under_doubling(self):
        """:270-281"""
        planes = np.random.default_rng(15).integers(0, 127, size=(2, 6, 6), dtype=np.uint8)
        m = model([[0.5, 1.0], [2.0, -1.0]])
        one = b.project_stack(stack_of(planes), m)
        two = b.project_stack(stack_of(planes * 2), m)
        for k in range(2):
            assert np.allclose(values_of(two[k]), 2.0 * values_of(one[k]), atol=0)

    def test_workers_bit_identical(self, small_stack):
        """:283-290 -- the device ignores `workers`; results bit-identical"""
        g = load("small_page")
        d = dm(small_stack.planes[:, g["ys"], g["xs"]].astype(np.float64), g["labels"])
        m = b.fit_cva(d)
        seq = b.project_stack(small_stack, m, workers=1)
        par = b.project_stack(small_stack, m, workers=4)
        for s, p in zip(seq, par):
            assert np.array_equal(values_of(s), values_of(p))

    def test_band_count_mismatch(self, small_stack):
        """:292-298"""
        with pytest.raises(b.DataError, match="bands"):
            b.project_stack(small_stack, model(np.eye(4)))

    def test_normalization_flag_mismatch(self, small_stack):
        """:300-307"""
        raw = b.SpectralStack(small_stack.bands, small_stack.planes, 8, normalized=False)
        with pytest.raises(b.DataError, match="normalized"):
            b.project_stack(raw, model(np.eye(6), provenance={"normalized_input": True}))

    def test_plane_variance_follows_eigenvalue_order(self):
        """:309-321 -- the training multiset laid out as an image: a plane's
        variance is (1 + lambda) / N.  The 3 = C - 1 significant components must
        come in order; the two null-space components (lambda ~ 1e-14, vectors
        numerically arbitrary -- SURVEY Appendix A) have equal variance up to
        the fp32 storage of the planes (1e-6 here, not the reference's fp64 1e-9)."""
        rng = np.random.default_rng(16)
        v = rng.integers(0, 255, size=(5, 64)).astype(np.float64)
        labels = np.repeat(np.arange(4), 16)
        m = b.fit_cva(dm(v, labels))
        planes = b.project_stack(stack_of(v.reshape(5, 8, 8)), m)
        var = np.array([values_of(p).var() for p in planes])
        assert (np.diff(var[:3]) <= 1e-9 * var.max()).all()
        assert (np.diff(var) <= 1e-6 * var.max()).all()


class TestModelSerialization:
    def test_round_trip_exact_and_deterministic(self, tmp_path):
        """:330-347"""
        v, l = labeled(np.random.default_rng(17), 4, 3, 12)
        m = b.fit_cva(dm(v, l), provenance={"manifest_sha256": "ab"})
        m.save(tmp_path / "a.json")
        m.save(tmp_path / "b.json")
        assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
        again = b.ProjectionModel.load(tmp_path / "a.json")
        for f in ("mean", "coefficients", "eigenvalues", "training_scores"):
            assert np.array_equal(getattr(again, f), getattr(m, f)), f
        assert again.std is None and again.provenance == m.provenance

    def test_lda_round_trip_keeps_std(self, tmp_path):
        """:360-367"""
        v, l = labeled(np.random.default_rng(18), 3, 2, 10)
        m = b.fit_lda(dm(v, l))
        m.save(tmp_path / "lda.json")
        assert np.array_equal(b.ProjectionModel.load(tmp_path / "lda.json").std, m.std)


# -------------------------------------------------------- test_eigen.py
class TestEigenHandCases:
    def test_identity_m_reduces_to_plain_eig(self):
        """test_eigen.py:17-20"""
        s = b.solve_gen_eig_sym(np.diag([3.0, 1.0]), np.eye(2), ridge=0.0)
        assert np.allclose(s.eigenvalues, [3.0, 1.0], atol=1e-14)
        assert np.allclose(s.eigenvectors, np.eye(2), atol=1e-14)

    def test_two_by_two_generalized(self):
        """:22-29"""
        s = b.solve_gen_eig_sym(np.diag([2.0, 2.0]), np.diag([1.0, 2.0]), ridge=0.0)
        assert np.allclose(s.eigenvalues, [2.0, 1.0], atol=1e-14)
        assert np.allclose(s.eigenvectors, [[1.0, 0.0], [0.0, 1 / np.sqrt(2.0)]], atol=1e-14)

    def test_default_ridge_shifts_by_relative_epsilon(self):
        """:31-35"""
        s = b.solve_gen_eig_sym(np.diag([3.0, 1.0]), np.eye(2))
        assert np.allclose(s.eigenvalues, np.array([3.0, 1.0]) / (1 + 1e-8), rtol=1e-12)


class TestEigenContracts:
    def test_descending_order_and_m_orthonormal_columns(self):
        """:39-49"""
        rng = np.random.default_rng(7)
        for _ in range(20):
            n = int(rng.integers(2, 9))
            a, m = sym(rng, n), spd(rng, n)
            s = b.solve_gen_eig_sym(a, m)
            assert (np.diff(s.eigenvalues) <= 1e-12).all()
            mp = b.regularize(m, b.DEFAULT_RIDGE)
            assert np.allclose(s.eigenvectors.T @ mp @ s.eigenvectors, np.eye(n), atol=1e-8)

    def test_residual_bound_without_ridge(self):
        """:51-62"""
        rng = np.random.default_rng(8)
        for _ in range(50):
            n = int(rng.integers(2, 9))
            a, m = sym(rng, n), spd(rng, n)
            s = b.solve_gen_eig_sym(a, m, ridge=0.0)
            r = np.linalg.norm(a @ s.eigenvectors - m @ s.eigenvectors * s.eigenvalues, axis=0)
            assert r.max() <= 1e-8 * np.linalg.norm(a, 2)

    def test_first_eigenvector_maximizes_rayleigh(self):
        """:74-82"""
        rng = np.random.default_rng(10)
        a, m = sym(rng, 6), spd(rng, 6)
        s = b.solve_gen_eig_sym(a, m, ridge=0.0)
        top = rayleigh(s.eigenvectors[:, 0], a, m)
        for _ in range(500):
            assert rayleigh(rng.normal(size=6), a, m) <= top + 1e-9 * abs(top)


class TestEigenSignAndDegenerate:
    def test_sign_convention(self):
        """:86-96"""
        out = b.sign_normalize(np.array([[0.3, -0.8], [-0.6, 0.1]]))
        assert np.allclose(out, [[-0.3, 0.8], [0.6, -0.1]])
        out = b.sign_normalize(np.array([[-0.5, 0.5], [0.5, -0.5]]))
        assert out[0, 0] > 0 and out[0, 1] > 0

    def test_solver_output_deterministic(self):
        """:98-105"""
        rng = np.random.default_rng(11)
        a, m = sym(rng, 5), spd(rng, 5)
        s1, s2 = b.solve_gen_eig_sym(a, m), b.solve_gen_eig_sym(a.copy(), m.copy())
        assert np.array_equal(s1.eigenvalues, s2.eigenvalues)
        assert np.array_equal(s1.eigenvectors, s2.eigenvectors)

    def test_zero_m_uses_scaled_identity(self):
        """:109-113"""
        s = b.solve_gen_eig_sym(np.diag([4.0, 1.0]), np.zeros((2, 2)))
        assert np.allclose(s.eigenvalues, [4e8, 1e8], rtol=1e-10)

    def test_errors(self):
        """:120-135"""
        with pytest.raises(b.NumericError, match="condition|definite"):
            b.solve_gen_eig_sym(np.eye(2), np.diag([2.0, -1.0]))
        asym = np.array([[1.0, 2.0], [0.0, 1.0]])
        with pytest.raises(b.NumericError, match="symmetric"):
            b.solve_gen_eig_sym(asym, np.eye(2))
        with pytest.raises(b.NumericError, match="symmetric"):
            b.solve_gen_eig_sym(np.eye(2), asym)
        with pytest.raises(b.NumericError):
            b.solve_gen_eig_sym(np.eye(3), np.eye(2))


# ---------------------------------- test_quantize.py / TestFullRange (device codes)
class TestQuantizeOnDevice:
    def test_ties_and_endpoints(self):
        """test_quantize.py:11-49 through the device stretch (ut_linear_to_codes)"""
        codes = b.linear_to_codes(np.array([-1.0, 0.0, 1.0]), -1.0, 1.0, 8)
        assert np.asarray(codes).tolist() == [0, 128, 255]
        codes = b.linear_to_codes(np.array([-5.0, 0.5, 20.0]), 0.0, 1.0, 8)
        assert np.asarray(codes).tolist() == [0, 128, 255]
        codes = b.linear_to_codes(np.array([0.0, 1.0]), 0.0, 1.0, 16)
        assert np.asarray(codes).tolist() == [0, 65535]
        assert np.asarray(b.round_half_away(np.array([0.5, 1.5, 2.5, -0.5, -1.5, -2.5]))).tolist() \
            == [1, 2, 3, -1, -2, -3]

    def test_linear_map_is_monotone(self):
        """test_quantize.py:59-66 on 20,000 random values"""
        v = np.random.default_rng(30).uniform(-100, 100, 20_000)
        out = np.asarray(b.linear_to_codes(v, -100.0, 100.0, 8)).astype(int)
        assert (np.diff(out[np.argsort(v, kind="stable")]) >= 0).all()


class TestFullRange:
    def test_sign_triple(self):
        """test_rendering.py:72-75"""
        out = np.asarray(b.rescale_full(b.ScorePlane(np.array([[-1.0, 0.0, 1.0]]))))
        assert out.tolist() == [[0, 128, 255]] and out.dtype == np.uint8

    def test_spans_entire_code_range(self):
        """:77-81"""
        out = np.asarray(b.rescale_full(b.ScorePlane(np.random.default_rng(0).normal(size=(40, 40)))))
        assert out.min() == 0 and out.max() == 255

    def test_sixteen_bit(self):
        """:83-86"""
        out = np.asarray(b.rescale_full(b.ScorePlane(np.array([[-1.0, 0.0, 1.0]])), depth=16))
        assert out.tolist() == [[0, 32768, 65535]] and out.dtype == np.uint16

    def test_constant_plane_warns_and_zeroes(self):
        """:88-91"""
        with pytest.warns(b.UndertextWarning):
            out = np.asarray(b.rescale_full(b.ScorePlane(np.full((4, 4), 3.5))))
        assert not out.any()

    def test_monotone(self):
        """:93-101 on 200 random rows"""
        rng = np.random.default_rng(31)
        for _ in range(200):
            row = rng.uniform(-1e6, 1e6, size=int(rng.integers(2, 61)))
            out = np.asarray(b.rescale_full(b.ScorePlane(row[None, :])))[0].astype(int)
            assert (np.diff(out[np.argsort(row, kind="stable")]) >= 0).all()


# ------------------------------------------------------- test_acceptance.py
def test_criterion_01_eigensolver_residuals():
    """test_acceptance.py:50-89: residual <= 1e-8 |A| over many random pencils
    (the top-eigenvalue oracle is the host reference's LAPACK, within 1e-6)."""
    rng = np.random.default_rng(101)
    for n in rng.integers(2, 9, size=200):
        n = int(n)
        a, m = sym(rng, n, scale=2.0), spd(rng, n)
        s = b.solve_gen_eig_sym(a, m, ridge=0.0)
        r = np.linalg.norm(a @ s.eigenvectors - m @ s.eigenvectors * s.eigenvalues, axis=0)
        assert r.max() <= 1e-8 * np.linalg.norm(a, 2)
        top = float(np.max(np.linalg.eigvals(np.linalg.solve(m, a)).real))
        assert abs(s.eigenvalues[0] - top) <= 1e-6 * abs(top)


def test_criterion_02_cva_optimality():
    """:92-113: the first canonical direction is never beaten by 1000 random ones"""
    rng = np.random.default_rng(102)
    for _ in range(100):
        bands, classes = int(rng.integers(2, 11)), int(rng.integers(3, 6))
        v, l = labeled(rng, bands, classes, int(rng.integers(8, 25)))
        sp = b.compute_scatter(dm(v, l))
        top = rayleigh(b.fit_cva(dm(v, l)).coefficients[:, 0], sp.between, sp.within)
        d = rng.normal(size=(1000, bands))
        q = np.einsum("gi,ij,gj->g", d, sp.between, d) / np.einsum("gi,ij,gj->g", d, sp.within, d)
        assert top >= q.max()


def test_criterion_03_lda_cva_agreement():
    """:116-132: LDA's first direction == CVA's on standardized input, 1e-10"""
    rng = np.random.default_rng(103)
    for _ in range(50):
        bands = int(rng.integers(2, 9))
        v, l = labeled(rng, bands, 2, int(rng.integers(8, 30)))
        lda = b.fit_lda(dm(v, l, ("a", "b")))
        sdm, _, _ = b.standardize(dm(v, l, ("a", "b")))
        cva = b.fit_cva(sdm)
        va = b.sign_normalize(lda.coefficients[:, :1])[:, 0]
        vb = b.sign_normalize(cva.coefficients[:, :1])[:, 0]
        assert np.abs(va - vb).max() <= 1e-10


def test_criterion_04_rank_structure():
    """:135-146: a 4-class 23-band page has exactly 3 eigenvalues > 1e-6 lambda_max
    (the BASELINE cfg 3 generator: 4 classes, 23 bands, 12-bit samples)."""
    from paper_1612_06457_b200 import synthetic

    cfg = synthetic.scaled(synthetic.CONFIGS["cfg3"], 256, 256, per_class=50)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    xy = torch.from_numpy(np.stack([scene.xs, scene.ys], 1).astype(np.int32)).cuda()
    values, _ = b.annotations.gather(stack, xy, len(scene.xs))
    ev = b.fit_cva(dm(values.cpu().numpy(), scene.labels)).eigenvalues
    assert int((ev > 1e-6 * ev[0]).sum()) == 3, ev[:6]


def test_criterion_08_cva_separates_better_than_any_band():
    """:236-258 restated without the DB metric (out of scope): on the BASELINE
    cfg 3 generator, the first CVA plane's Fisher ratio between the undertext-
    like class and the background beats every raw band's."""
    from paper_1612_06457_b200 import synthetic

    cfg = synthetic.scaled(synthetic.CONFIGS["cfg3"], 256, 256, per_class=50)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    pipe = b.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=1)
    pipe.run()
    score = pipe.scores[0].double().cpu().numpy()
    cube = stack.planes.cpu().numpy().astype(np.float64)
    ys, xs = np.mgrid[0:cfg.height, 0:cfg.width]
    cmap = synthetic.class_map_at(scene.shapes, ys, xs)
    a, c = cmap == 0, cmap == 2

    def fisher(x):
        return (x[a].mean() - x[c].mean()) ** 2 / (x[a].var() + x[c].var())

    assert fisher(score) > max(fisher(cube[i]) for i in range(cube.shape[0]))


def test_criterion_10_determinism(tmp_path):
    """:277-309: fit + render twice -> byte-identical model JSON and images"""
    from paper_1612_06457_b200 import pipeline as bp

    g = load("small_page")
    stack = b.SpectralStack(b.stack.default_bands(g["cube"].shape[0]), g["cube"], 8, True)
    blobs = []
    for run in ("one", "two"):
        d = dm(g["cube"][:, g["ys"], g["xs"]].astype(np.float64), g["labels"])
        m = b.fit_cva(d)
        out = tmp_path / run
        out.mkdir()
        m.save(out / "model.json")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            bp.render_planes(stack, m, [b.RenderSpec(), b.RenderSpec("percentile", 1.0)], out,
                             recipe=b.CompositeRecipe(1, 0, 2))
        blobs.append({p.name: p.read_bytes() for p in sorted(out.iterdir())})
    assert blobs[0].keys() == blobs[1].keys() and len(blobs[0]) >= 4
    for name, blob in blobs[0].items():
        assert blob == blobs[1][name], name
