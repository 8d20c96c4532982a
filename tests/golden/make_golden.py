"""Generate the golden vectors that pin the oracle (and the CUDA path).

Run ONLY in the build container, where the read-only reference is mounted:

    python tests/golden/make_golden.py

It imports the real reference package from /root/reference/pkg/src (plus its
test helpers in /root/reference/pkg/tests/oracles.py), runs the hot-path
functions on seeded inputs and writes small .npz fixtures next to this file.
The GPU box never runs this script; tests only read the committed .npz files.
"""

from __future__ import annotations

import sys
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))
sys.path.insert(0, str(HERE.parent))

from cubes import make_cube  # noqa: E402
from oracles import random_labeled, random_spd, random_sym  # noqa: E402
from undertext.annotations import (  # noqa: E402
    AnnotatedPoint, ClassLabel, DesignMatrix, TrainingSet, assemble_matrix,
)
from undertext.eigen import solve_gen_eig_sym  # noqa: E402
from undertext.projection import (  # noqa: E402
    compute_scatter, fit_cva, fit_lda, fit_pca_unsupervised, project_stack, standardize,
)
from undertext.projection import ProjectionModel  # noqa: E402
from undertext.rendering import (ScorePlane, rescale_full, rescale_percentile,  # noqa: E402
                                 rescale_training_range)
from undertext.stack import BandMeta, SpectralStack, normalize_stack  # noqa: E402
from undertext.synthetic import make_palimpsest  # noqa: E402


def _stack(planes, depth):
    metas = tuple(BandMeta(i, 400.0 + i, "x") for i in range(planes.shape[0]))
    return SpectralStack(metas, planes, depth, normalized=True)


def _training(xs, ys, labels):
    names = sorted(set(int(v) for v in labels))
    cls = {c: ClassLabel(f"c{c}", c) for c in names}
    pts = tuple(AnnotatedPoint(int(x), int(y), cls[int(l)]) for x, y, l in zip(xs, ys, labels))
    return TrainingSet(tuple(cls[c] for c in names), pts)


def scatter_cases():
    out = {}
    cases = [(np.array([[0.0, 2.0, 10.0, 12.0]]), np.array([0, 0, 1, 1]))]
    rng = np.random.default_rng(2024)
    for b, c, n in [(6, 3, 20), (16, 3, 40), (23, 4, 25), (32, 6, 30), (5, 2, 7)]:
        v, l = random_labeled(rng, b, c, n)
        cases.append((v, l))
    # non-contiguous, unsorted label ids
    v, l = random_labeled(rng, 4, 3, 10)
    cases.append((v, np.array([7, 2, 9])[l]))
    for i, (v, l) in enumerate(cases):
        sp = compute_scatter(DesignMatrix(np.asarray(v, dtype=np.float64), np.asarray(l, dtype=np.intp), tuple()))
        out.update({f"{i}_values": v, f"{i}_labels": l, f"{i}_within": sp.within,
                    f"{i}_between": sp.between, f"{i}_means": sp.class_means,
                    f"{i}_ids": np.array(sp.class_ids), f"{i}_counts": sp.counts,
                    f"{i}_grand": sp.grand_mean})
    out["n"] = np.array(len(cases))
    np.savez_compressed(HERE / "scatter.npz", **out)


def eigen_cases():
    out = {}
    rng = np.random.default_rng(77)
    i = 0
    for b in [2, 3, 5, 8, 16, 23, 32]:
        for ridge in (1e-8, 0.0):
            a = random_sym(rng, b)
            m = random_spd(rng, b)
            sol = solve_gen_eig_sym(a, m, ridge)
            out.update({f"{i}_a": a, f"{i}_m": m, f"{i}_ridge": np.array(ridge),
                        f"{i}_evals": sol.eigenvalues, f"{i}_evecs": sol.eigenvectors})
            i += 1
    out["n"] = np.array(i)
    np.savez_compressed(HERE / "eigen.npz", **out)


def cube_case(name, h, w, b, c, dtype, seed, per_class, k, depth, per_class_cov=False,
              blobs=False, pca_region=None):
    cube, xs, ys, labels = make_cube(h, w, b, c, dtype, seed, per_class,
                                     per_class_cov=per_class_cov, blobs=blobs)
    stack = _stack(cube, depth)
    dm = assemble_matrix(stack, _training(xs, ys, labels))
    model = fit_cva(dm, k=k)
    planes = project_stack(stack, model)
    codes = np.stack([rescale_full(p) for p in planes])
    sp = compute_scatter(dm)
    pmodel = fit_pca_unsupervised(stack, region=pca_region, k=k)
    pplanes = project_stack(stack, pmodel)
    pcodes = np.stack([rescale_full(p) for p in pplanes])
    np.savez_compressed(
        HERE / f"{name}.npz",
        cube=cube, xs=xs, ys=ys, labels=labels, k=np.array(k),
        design=dm.values,
        within=sp.within, between=sp.between, class_means=sp.class_means,
        counts=sp.counts, grand_mean=sp.grand_mean,
        cva_mean=model.mean, cva_coef=model.coefficients, cva_evals=model.eigenvalues,
        cva_train_scores=model.training_scores,
        cva_scores=np.stack([p.values for p in planes]), cva_codes=codes,
        pca_region=np.array(pca_region if pca_region else (0, 0, w, h)),
        pca_mean=pmodel.mean, pca_std=pmodel.std, pca_coef=pmodel.coefficients,
        pca_evals=pmodel.eigenvalues,
        pca_scores=np.stack([p.values for p in pplanes]), pca_codes=pcodes,
    )


def small_page_case():
    """The reference's own session fixture (tests/conftest.py:7-15)."""
    page = make_palimpsest(96, 96, bands=6, seed=1, eval_per_class=40)
    stack = normalize_stack(page.stack)
    pts = page.training.points
    xs = np.array([p.x for p in pts], dtype=np.int32)
    ys = np.array([p.y for p in pts], dtype=np.int32)
    labels = np.array([p.label.id for p in pts], dtype=np.int32)
    dm = assemble_matrix(stack, page.training)
    model = fit_cva(dm)
    planes = project_stack(stack, model)
    codes = np.stack([rescale_full(p) for p in planes])
    pmodel = fit_pca_unsupervised(stack, k=5)
    pplanes = project_stack(stack, pmodel)
    pcodes = np.stack([rescale_full(p) for p in pplanes])
    np.savez_compressed(
        HERE / "small_page.npz",
        cube=stack.planes, xs=xs, ys=ys, labels=labels, design=dm.values,
        cva_mean=model.mean, cva_coef=model.coefficients, cva_evals=model.eigenvalues,
        cva_scores=np.stack([p.values for p in planes]), cva_codes=codes,
        pca_mean=pmodel.mean, pca_std=pmodel.std, pca_coef=pmodel.coefficients,
        pca_evals=pmodel.eigenvalues,
        pca_scores=np.stack([p.values for p in pplanes]), pca_codes=pcodes,
    )


def rescale_cases():
    rng = np.random.default_rng(5)
    planes = {
        "sign": np.array([[-1.0, 0.0, 1.0]]),
        "normal": rng.normal(size=(40, 40)),
        "ties": np.array([[0.0, 0.5 / 255.0, 1.5 / 255.0, 2.5 / 255.0, 1.0]]),
        "wide": rng.uniform(-1e6, 1e6, size=(7, 9)),
    }
    out = {}
    for key, p in planes.items():
        out[f"{key}_in"] = p
        out[f"{key}_u8"] = rescale_full(ScorePlane(p))
        out[f"{key}_u16"] = rescale_full(ScorePlane(p), depth=16)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out["const_u8"] = rescale_full(ScorePlane(np.full((4, 4), 3.5)))
    np.savez_compressed(HERE / "rescale.npz", **out)


def normalize_cases():
    """stack.py:180-213 on raw (not normalized) stacks of every sample type."""
    rng = np.random.default_rng(9)
    cases = {
        "u8": (rng.integers(3, 220, size=(3, 17, 23)).astype(np.uint8), 8),
        "u16": (rng.integers(100, 4000, size=(4, 16, 20)).astype(np.uint16), 16),
        "u16_span": (np.array([[[0, 32768, 65535]]], dtype=np.uint16), 16),
        "f32": (rng.uniform(0, 200, size=(2, 12, 15)).astype(np.float32), 8),
        "f64_ties": (np.array([[[0.0, 0.5, 1.0, 127.0, 255.0, 2.0, 254.0]]]), 8),
        "const": (np.stack([np.full((4, 5), 7, np.uint8),
                            rng.integers(0, 9, size=(4, 5)).astype(np.uint8)]), 8),
    }
    out = {}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for key, (planes, depth) in cases.items():
            metas = tuple(BandMeta(i, 400.0 + i, "x") for i in range(planes.shape[0]))
            st = SpectralStack(metas, planes, depth)
            out[f"{key}_in"] = planes
            out[f"{key}_depth"] = np.array(depth)
            for scope in ("per-band", "global"):
                out[f"{key}_{scope}"] = normalize_stack(st, scope=scope).planes
    np.savez_compressed(HERE / "normalize.npz", **out)


def rescale_mode_cases():
    """rendering.py:133-179: training-range and percentile windows."""
    rng = np.random.default_rng(10)
    out = {}
    plane = rng.normal(size=(37, 41))
    out["plane"] = plane
    scores = rng.normal(scale=0.8, size=(3, 50))
    model = ProjectionModel(method="cva", mean=np.zeros(2), std=None,
                            coefficients=np.ones((2, 3)), eigenvalues=np.ones(3),
                            training_scores=scores)
    out["training_scores"] = scores
    for k in range(3):
        out[f"train_k{k}_u8"] = rescale_training_range(ScorePlane(plane), model, k)
        out[f"train_k{k}_u16"] = rescale_training_range(ScorePlane(plane), model, k, depth=16)
    for p in (0.01, 0.1, 1.0, 5.0):
        tag = str(p).replace(".", "_")
        out[f"pct_{tag}"] = rescale_percentile(ScorePlane(plane), p)
        out[f"pct_{tag}_one"] = rescale_percentile(ScorePlane(plane), p, one_tail=True)
        out[f"pct_{tag}_u16"] = rescale_percentile(ScorePlane(plane), p, depth=16)
    lin = rng.permutation(np.linspace(0.0, 1.0, 1000)).reshape(25, 40)
    out["lin"] = lin
    out["lin_p5"] = rescale_percentile(ScorePlane(lin), 5.0)
    np.savez_compressed(HERE / "rescale_modes.npz", **out)


def lda_cases():
    """fit_lda / standardize (projection.py:152-169, :240-260) on two-class sets,
    incl. a constant band (std recorded as 1)."""
    out = {}
    rng = np.random.default_rng(4242)
    cases = []
    for b, n in [(6, 30), (16, 50), (32, 80)]:
        v, l = random_labeled(rng, b, 2, n)
        cases.append((np.asarray(v, dtype=np.float64), np.asarray(l)))
    v, l = random_labeled(rng, 5, 2, 12)
    v = np.asarray(v, dtype=np.float64).copy()
    v[2] = 0.375
    cases.append((v, np.array([3, 8])[np.asarray(l)]))
    for i, (v, l) in enumerate(cases):
        dm = DesignMatrix(v, np.asarray(l, dtype=np.intp), tuple())
        sdm, mean, std = standardize(dm)
        m = fit_lda(dm, k=1)
        out.update({f"{i}_values": v, f"{i}_labels": l, f"{i}_std_values": sdm.values,
                    f"{i}_mean": mean, f"{i}_std": std, f"{i}_coef": m.coefficients,
                    f"{i}_evals": m.eigenvalues, f"{i}_scores": m.training_scores})
    out["n"] = np.array(len(cases))
    np.savez_compressed(HERE / "lda.npz", **out)


if __name__ == "__main__":
    lda_cases()
    scatter_cases()
    eigen_cases()
    cube_case("cva_f64", 48, 64, 16, 3, np.float64, 11, 60, 2, 8)
    cube_case("cva_f32", 40, 56, 16, 3, np.float32, 12, 60, 3, 8, pca_region=(5, 3, 40, 30))
    cube_case("cva_u16", 40, 48, 23, 4, np.uint16, 13, 50, 3, 16, blobs=True)
    cube_case("cva_f16", 32, 40, 23, 4, np.float16, 14, 40, 3, 8, blobs=True)
    cube_case("cva_f32_b32", 40, 40, 32, 6, np.float32, 15, 40, 5, 8, per_class_cov=True)
    small_page_case()
    rescale_cases()
    normalize_cases()
    rescale_mode_cases()
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)
