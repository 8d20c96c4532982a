"""Pin the CPU oracle against golden vectors produced by the real reference.

The oracle restates the reference operation for operation, so on the machine
that generated the fixtures the results are bit-identical; across machines a
BLAS reduction order may differ in the last ulp, hence the 1e-12 relative
allowance on matrix products (uint8 codes, labels and counts stay exact).
Also re-states the reference's own known-answer tests.
"""

import numpy as np
import pytest

import oracle
from golden_util import load, rel_close

CUBES = ["cva_f64", "cva_f32", "cva_u16", "cva_f16", "cva_f32_b32", "small_page"]


def test_scatter_golden():
    g = load("scatter")
    for i in range(int(g["n"])):
        sp = oracle.scatter(g[f"{i}_values"], g[f"{i}_labels"])
        assert np.array_equal(np.array(sp["class_ids"]), g[f"{i}_ids"])
        assert np.array_equal(sp["counts"], g[f"{i}_counts"])
        for key, gk in (("within", "within"), ("between", "between"),
                        ("class_means", "means"), ("grand_mean", "grand")):
            assert rel_close(sp[key], g[f"{i}_{gk}"], 1e-12), (i, key)


def test_eigen_golden():
    g = load("eigen")
    for i in range(int(g["n"])):
        lam, vec = oracle.gen_eig_sym(g[f"{i}_a"], g[f"{i}_m"], float(g[f"{i}_ridge"]))
        assert rel_close(lam, g[f"{i}_evals"], 1e-10), i
        assert rel_close(vec, g[f"{i}_evecs"], 1e-8), i


@pytest.mark.parametrize("name", CUBES)
def test_cube_golden(name):
    g = load(name)
    cube = g["cube"]
    design = oracle.assemble(cube, g["xs"], g["ys"])
    assert np.array_equal(design, g["design"])
    k = int(g["k"]) if "k" in g else None
    model = oracle.fit_cva(design, g["labels"], k=k)
    assert rel_close(model["mean"], g["cva_mean"], 1e-12)
    assert rel_close(model["eigenvalues"], g["cva_evals"], 1e-10)
    assert rel_close(model["coefficients"], g["cva_coef"], 1e-8)
    scores = oracle.project(cube, model)
    assert rel_close(scores, g["cva_scores"], 1e-8)
    codes = np.stack([oracle.rescale_full(s) for s in g["cva_scores"]])
    assert np.array_equal(codes, g["cva_codes"])
    region = tuple(int(v) for v in g["pca_region"]) if "pca_region" in g else None
    pm = oracle.fit_pca_unsupervised(cube, region=region, k=g["pca_coef"].shape[1])
    assert rel_close(pm["mean"], g["pca_mean"], 1e-12)
    assert rel_close(pm["std"], g["pca_std"], 1e-12)
    assert rel_close(pm["eigenvalues"], g["pca_evals"], 1e-10)
    assert rel_close(pm["coefficients"], g["pca_coef"], 1e-8)
    pcodes = np.stack([oracle.rescale_full(s) for s in g["pca_scores"]])
    assert np.array_equal(pcodes, g["pca_codes"])
    pscores = oracle.project(cube, pm)
    assert rel_close(pscores, g["pca_scores"], 1e-8)


def test_rescale_golden():
    g = load("rescale")
    for key in ("sign", "normal", "ties", "wide"):
        assert np.array_equal(oracle.rescale_full(g[f"{key}_in"]), g[f"{key}_u8"])
        assert np.array_equal(oracle.rescale_full(g[f"{key}_in"], 16), g[f"{key}_u16"])
    assert not oracle.rescale_full(np.full((4, 4), 3.5)).any()


def test_workers_bit_identical():
    g = load("cva_f32")
    model = oracle.fit_cva(g["design"], g["labels"], k=3)
    a = oracle.project(g["cube"], model, workers=1)
    b = oracle.project(g["cube"], model, workers=4)
    assert np.array_equal(a, b)


# ---- the reference's own known-answer tests, restated ----

def test_scatter_hand_oracle():
    # tests/test_projection.py:63-69
    sp = oracle.scatter(np.array([[0.0, 2.0, 10.0, 12.0]]), np.array([0, 0, 1, 1]))
    assert sp["within"].tolist() == [[4.0]]
    assert sp["between"].tolist() == [[100.0]]
    assert sp["grand_mean"].tolist() == [6.0]
    assert sp["class_means"].tolist() == [[1.0], [11.0]]


def test_eigen_hand_cases():
    # tests/test_eigen.py:17-35, :109-118
    lam, vec = oracle.gen_eig_sym(np.diag([3.0, 1.0]), np.eye(2), 0.0)
    assert np.allclose(lam, [3.0, 1.0], atol=1e-14) and np.allclose(vec, np.eye(2), atol=1e-14)
    lam, vec = oracle.gen_eig_sym(np.diag([2.0, 2.0]), np.diag([1.0, 2.0]), 0.0)
    assert np.allclose(lam, [2.0, 1.0], atol=1e-14)
    assert np.allclose(vec, [[1.0, 0.0], [0.0, 1.0 / np.sqrt(2.0)]], atol=1e-14)
    lam, _ = oracle.gen_eig_sym(np.diag([3.0, 1.0]), np.eye(2))
    assert np.allclose(lam, np.array([3.0, 1.0]) / (1 + 1e-8), rtol=1e-12)
    lam, _ = oracle.gen_eig_sym(np.diag([4.0, 1.0]), np.zeros((2, 2)))
    assert np.allclose(lam, [4e8, 1e8], rtol=1e-10)
    assert np.allclose(np.diag(oracle.regularize(np.diag([2.0, 4.0]), 1e-8)),
                       [2.0 + 3e-8, 4.0 + 3e-8])
    with pytest.raises(oracle.OracleNumericError):
        oracle.gen_eig_sym(np.eye(2), np.diag([2.0, -1.0]))
    with pytest.raises(oracle.OracleNumericError):
        oracle.gen_eig_sym(np.array([[1.0, 2.0], [0.0, 1.0]]), np.eye(2))


def test_sign_convention():
    # tests/test_eigen.py:86-96
    out = oracle.sign_normalize(np.array([[0.3, -0.8], [-0.6, 0.1]]))
    assert np.allclose(out, [[-0.3, 0.8], [0.6, -0.1]])
    out = oracle.sign_normalize(np.array([[-0.5, 0.5], [0.5, -0.5]]))
    assert out[0, 0] > 0 and out[0, 1] > 0


def test_quantize_known_answers():
    # tests/test_quantize.py:11-48
    assert oracle.round_half_away(np.array([0.5, 1.5, 2.5, -0.5, -1.5, -2.5])).tolist() == [1, 2, 3, -1, -2, -3]
    assert oracle.linear_to_codes(np.array([-1.0, 0.0, 1.0]), -1.0, 1.0).tolist() == [0, 128, 255]
    assert oracle.linear_to_codes(np.array([-5.0, 0.5, 20.0]), 0.0, 1.0).tolist() == [0, 128, 255]
    assert oracle.linear_to_codes(np.array([0.0, 1.0]), 0.0, 1.0, 16).tolist() == [0, 65535]


def test_pca_equal_bands_rank_one():
    # tests/test_projection.py:237-242
    plane = np.arange(64, dtype=np.uint8).reshape(8, 8)
    pm = oracle.fit_pca_unsupervised(np.stack([plane, plane, plane]))
    assert pm["eigenvalues"][0] == pytest.approx(3.0, rel=1e-8)
    assert np.allclose(pm["eigenvalues"][1:], 0.0, atol=1e-9)


NORMALIZE_CASES = ["u8", "u16", "u16_span", "f32", "f64_ties", "const"]


@pytest.mark.parametrize("key", NORMALIZE_CASES)
@pytest.mark.parametrize("scope", ["per-band", "global"])
def test_normalize_golden(key, scope):
    """stack.py:180-213 restated: bit-identical codes on every sample type."""
    g = load("normalize")
    codes, _ = oracle.normalize_stack(g[f"{key}_in"], scope)
    assert np.array_equal(codes, g[f"{key}_{scope}"])


def test_normalize_known_answers():
    # tests/test_stack.py:113-154 of the reference, restated
    codes, _ = oracle.normalize_stack(np.array([[[0, 32768, 65535]]], dtype=np.uint16))
    assert codes[0].tolist() == [[0, 128, 255]]
    ident = np.arange(256, dtype=np.uint8).reshape(1, 16, 16)
    assert np.array_equal(oracle.normalize_stack(ident)[0], ident)
    two = np.stack([np.array([[0, 50]], np.uint8), np.array([[50, 100]], np.uint8)])
    g, _ = oracle.normalize_stack(two, "global")
    assert g[0].tolist() == [[0, 128]] and g[1].tolist() == [[128, 255]]
    c, flags = oracle.normalize_stack(np.full((1, 2, 2), 7, np.uint8))
    assert c.max() == 0 and flags.tolist() == [True]


def test_rescale_modes_golden():
    """rendering.py:133-179 restated: training-range and percentile windows."""
    g = load("rescale_modes")
    plane, scores = g["plane"], g["training_scores"]
    for k in range(3):
        assert np.array_equal(oracle.rescale_training_range(plane, scores, k), g[f"train_k{k}_u8"])
        assert np.array_equal(oracle.rescale_training_range(plane, scores, k, 16),
                              g[f"train_k{k}_u16"])
    for p in (0.01, 0.1, 1.0, 5.0):
        tag = str(p).replace(".", "_")
        assert np.array_equal(oracle.rescale_percentile(plane, p), g[f"pct_{tag}"])
        assert np.array_equal(oracle.rescale_percentile(plane, p, one_tail=True), g[f"pct_{tag}_one"])
        assert np.array_equal(oracle.rescale_percentile(plane, p, 16), g[f"pct_{tag}_u16"])
    assert np.array_equal(oracle.rescale_percentile(g["lin"], 5.0), g["lin_p5"])
    flat = np.sort(np.random.default_rng(1).normal(size=1000))
    assert oracle.nearest_rank(flat, 1.0) == flat[9] and oracle.nearest_rank(flat, 99.0) == flat[989]


def test_lda_golden():
    """standardize + fit_lda (projection.py:152-169, :240-260) vs the reference,
    incl. a constant band (std 1) and non-contiguous label ids."""
    g = load("lda")
    for i in range(int(g["n"])):
        sv, mean, std = oracle.standardize(g[f"{i}_values"])
        assert rel_close(sv, g[f"{i}_std_values"], 1e-12), i
        assert rel_close(mean, g[f"{i}_mean"], 1e-12), i
        assert rel_close(std, g[f"{i}_std"], 1e-12), i
        m = oracle.fit_lda(g[f"{i}_values"], g[f"{i}_labels"], k=1)
        assert rel_close(m["eigenvalues"], g[f"{i}_evals"], 1e-10), i
        assert rel_close(m["coefficients"], g[f"{i}_coef"], 1e-8), i
        assert rel_close(m["training_scores"], g[f"{i}_scores"], 1e-8), i
