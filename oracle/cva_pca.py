"""numpy restatement of the reference CVA / PCA hot path (test oracle only).

Each function names the reference lines it restates (paths relative to
``/root/reference/pkg/src/undertext``).  The arithmetic is kept operation for
operation -- same numpy reductions, same chunking, same summation order -- so
that on one machine the outputs are bit-identical to the reference's; the
pinning tests in ``tests/test_oracle_golden.py`` check exactly that against
``tests/golden/*.npz``.

Inputs are plain arrays, not the reference's dataclasses:

* ``planes``  -- (B, H, W) band-sequential cube, any real dtype;
* ``values``  -- (B, N) design matrix (float64), ``labels`` -- (N,) ints;
* a *model* is a dict with ``mean``, ``std`` (or None), ``coefficients`` (B, K)
  and ``eigenvalues`` (K,).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

RIDGE_DEFAULT = 1e-8          # eigen.py:23
SYMMETRY_RTOL = 1e-10         # eigen.py:25
ROW_CHUNK = 64                # projection.py:36


class OracleError(Exception):
    """Bad input (the reference raises DataError, errors.py:12)."""


class OracleNumericError(Exception):
    """Numeric failure (the reference raises NumericError, errors.py:17)."""


# --------------------------------------------------------------------------
# quantize.py / rendering.py
# --------------------------------------------------------------------------

def round_half_away(x):
    """quantize.py:13-21 -- nearest integer, ties away from zero."""
    a = np.asarray(x, dtype=np.float64)
    return np.sign(a) * np.floor(np.abs(a) + 0.5)


def linear_to_codes(v, lo: float, hi: float, depth: int = 8) -> np.ndarray:
    """quantize.py:36-46 -- [lo, hi] -> [0, 2^depth - 1], clip, round."""
    if depth not in (8, 16):
        raise ValueError(f"unsupported depth {depth}")
    if not (np.isfinite(lo) and np.isfinite(hi)) or lo >= hi:
        raise ValueError(f"invalid rescale range [{lo}, {hi}]")
    top = (1 << depth) - 1
    scaled = (np.asarray(v, dtype=np.float64) - lo) * (top / (hi - lo))
    codes = round_half_away(np.clip(scaled, 0.0, top))
    return codes.astype(np.uint8 if depth == 8 else np.uint16)


def rescale_full(plane, depth: int = 8) -> np.ndarray:
    """rendering.py:124-130 (+ ScorePlane finite check :49-50).

    A constant plane renders as zeros (the reference also warns, :119-121).
    """
    p = np.asarray(plane, dtype=np.float64)
    if not np.isfinite(p).all():
        raise OracleError("score plane contains NaN or Inf")
    lo, hi = float(p.min()), float(p.max())
    if lo == hi:
        return np.zeros(p.shape, dtype=np.uint8 if depth == 8 else np.uint16)
    return linear_to_codes(p, lo, hi, depth)


def rescale_training_range(plane, training_scores, k: int, depth: int = 8) -> np.ndarray:
    """rendering.py:133-152 -- window = span of component k's training scores."""
    row = np.asarray(training_scores)[k]
    lo, hi = float(row.min()), float(row.max())
    p = np.asarray(plane, dtype=np.float64)
    if lo == hi:
        return np.zeros(p.shape, dtype=np.uint8 if depth == 8 else np.uint16)
    return linear_to_codes(p, lo, hi, depth)


def nearest_rank(sorted_values, p: float) -> float:
    """rendering.py:146-152 -- element ceil(p/100 n) of the ascending sample."""
    n = len(sorted_values)
    rank = max(1, math.ceil(p / 100.0 * n))
    return float(sorted_values[rank - 1])


def rescale_percentile(plane, p: float, depth: int = 8, one_tail: bool = False) -> np.ndarray:
    """rendering.py:155-179 -- nearest-rank window [p, 100-p] (or [min, 100-p])."""
    v = np.asarray(plane, dtype=np.float64)
    flat = np.sort(v, axis=None)
    lo = float(flat[0]) if one_tail else nearest_rank(flat, p)
    hi = nearest_rank(flat, 100.0 - p)
    if lo == hi:
        return np.zeros(v.shape, dtype=np.uint8 if depth == 8 else np.uint16)
    return linear_to_codes(v, lo, hi, depth)


# --------------------------------------------------------------------------
# stack.py
# --------------------------------------------------------------------------

def normalize_stack(planes, scope: str = "per-band"):
    """stack.py:180-213 -- (codes uint8, constant-band flags).

    lo/hi per band (or over the cube); 255 * (v - lo) / (hi - lo) in float64,
    rounded half away; a constant band maps to zeros (the reference warns).
    """
    planes = np.asarray(planes)
    out = np.empty(planes.shape, dtype=np.uint8)
    flags = np.zeros(planes.shape[0], dtype=bool)
    if scope == "global":
        lo, hi = float(planes.min()), float(planes.max())
    for i in range(planes.shape[0]):
        plane = planes[i]
        if scope == "per-band":
            lo, hi = float(plane.min()), float(plane.max())
        if lo == hi:
            flags[i] = True
            out[i] = 0
            continue
        scaled = 255.0 * (plane.astype(np.float64) - lo) / (hi - lo)
        with np.errstate(invalid="ignore"):
            out[i] = round_half_away(scaled).astype(np.uint8)
    return out, flags


# --------------------------------------------------------------------------
# annotations.py
# --------------------------------------------------------------------------

def assemble(planes, xs, ys) -> np.ndarray:
    """annotations.py:195-215 -- B x N float64 gather, in point order."""
    b, h, w = planes.shape
    xs = np.asarray(xs)
    ys = np.asarray(ys)
    out = np.empty((b, len(xs)), dtype=np.float64)
    for j in range(len(xs)):
        x, y = int(xs[j]), int(ys[j])
        if not (0 <= x < w and 0 <= y < h):
            raise OracleError(f"point ({x}, {y}) outside {w}x{h} stack")
        out[:, j] = planes[:, y, x]
    return out


# --------------------------------------------------------------------------
# eigen.py
# --------------------------------------------------------------------------

def sign_normalize(vecs: np.ndarray) -> np.ndarray:
    """eigen.py:40-52 -- largest-|entry| positive, first maximizer wins."""
    out = np.array(vecs, dtype=np.float64, copy=True)
    for j in range(out.shape[1]):
        lead = int(np.argmax(np.abs(out[:, j])))
        if out[lead, j] < 0:
            out[:, j] = -out[:, j]
    return out


def regularize(m: np.ndarray, ridge: float = RIDGE_DEFAULT) -> np.ndarray:
    """eigen.py:63-72 -- M + ridge*(tr M / B)*I, or ridge*I if tr M <= 0."""
    n = m.shape[0]
    tr = float(np.trace(m))
    return m + (ridge * (tr / n if tr > 0.0 else 1.0)) * np.eye(n)


def _asym(mat: np.ndarray) -> bool:
    """eigen.py:55-60."""
    top = float(np.abs(mat).max())
    return top != 0.0 and float(np.abs(mat - mat.T).max()) > SYMMETRY_RTOL * top


def gen_eig_sym(a, m, ridge: float = RIDGE_DEFAULT):
    """eigen.py:75-113 -- A v = lambda M' v; returns (evals desc, evecs)."""
    a = np.asarray(a, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    if a.ndim != 2 or a.shape != m.shape or a.shape[0] != a.shape[1]:
        raise OracleNumericError(f"shape mismatch {a.shape} vs {m.shape}")
    if _asym(a) or _asym(m):
        raise OracleNumericError("matrix is not symmetric")
    mr = regularize(m, ridge)
    try:
        chol = np.linalg.cholesky(mr)
    except np.linalg.LinAlgError:
        raise OracleNumericError("regularized M is not positive definite") from None
    # C = L^-1 A L^-T via two general solves, then symmetrized (eigen.py:107-109)
    c = np.linalg.solve(chol, np.linalg.solve(chol, a).T)
    c = (c + c.T) / 2.0
    lam, u = np.linalg.eigh(c)
    lam = np.ascontiguousarray(lam[::-1])
    v = np.linalg.solve(chol.T, u[:, ::-1])
    return lam, sign_normalize(v)


# --------------------------------------------------------------------------
# projection.py -- scatter and fits
# --------------------------------------------------------------------------

def _top_k(k, b):
    """projection.py:204-208."""
    k = b if k is None else int(k)
    if not 1 <= k <= b:
        raise OracleError(f"requested {k} components from {b} bands")
    return k


def scatter(values, labels) -> dict:
    """projection.py:172-201 -- two-pass per-class scatter, symmetrized."""
    values = np.asarray(values, dtype=np.float64)
    labels = np.asarray(labels)
    ids = [int(c) for c in np.unique(labels)]
    if len(ids) < 2:
        raise OracleError(f"scatter needs at least 2 classes, got {len(ids)}")
    b = values.shape[0]
    grand = values.mean(axis=1)
    sw = np.zeros((b, b))
    sb = np.zeros((b, b))
    means = np.empty((len(ids), b))
    counts = np.empty(len(ids), dtype=np.intp)
    for i, cid in enumerate(ids):
        members = values[:, labels == cid]
        mc = members.mean(axis=1)
        means[i] = mc
        counts[i] = members.shape[1]
        dev = members - mc[:, None]
        sw += dev @ dev.T
        gap = mc - grand
        sb += counts[i] * np.outer(gap, gap)
    return {
        "within": (sw + sw.T) / 2.0,
        "between": (sb + sb.T) / 2.0,
        "class_means": means,
        "class_ids": tuple(ids),
        "counts": counts,
        "grand_mean": grand,
    }


def fit_cva(values, labels, k=None, ridge: float = RIDGE_DEFAULT) -> dict:
    """projection.py:211-237 -- CVA on raw values; training scores included."""
    values = np.asarray(values, dtype=np.float64)
    sp = scatter(values, labels)
    lam, vecs = gen_eig_sym(sp["between"], sp["within"], ridge)
    k = _top_k(k, values.shape[0])
    coef = np.ascontiguousarray(vecs[:, :k])
    return {
        "method": "cva",
        "mean": sp["grand_mean"],
        "std": None,
        "coefficients": coef,
        "eigenvalues": np.ascontiguousarray(lam[:k]),
        "training_scores": coef.T @ (values - sp["grand_mean"][:, None]),
        "scatter": sp,
    }


def standardize(values):
    """projection.py:152-169 -- rows to mean 0 and sample std 1 (divisor N-1);
    constant rows are centred only, their std recorded as 1."""
    values = np.asarray(values, dtype=np.float64)
    if values.shape[1] < 2:
        raise OracleError("standardization needs at least 2 points")
    mean = values.mean(axis=1)
    centered = values - mean[:, None]
    var = (centered * centered).sum(axis=1) / (values.shape[1] - 1)
    std = np.sqrt(var)
    std[std == 0.0] = 1.0
    return centered / std[:, None], mean, std


def fit_lda(values, labels, k=None, ridge: float = RIDGE_DEFAULT) -> dict:
    """projection.py:240-260 -- two-class discriminant: CVA on standardized rows."""
    if len(np.unique(np.asarray(labels))) != 2:
        raise OracleError("LDA requires exactly 2 classes")
    sv, mean, std = standardize(values)
    core = fit_cva(sv, labels, k=k, ridge=ridge)
    core.update(method="lda", mean=mean, std=std)
    return core


def _pca_eig(cov, k):
    """projection.py:263-270."""
    cov = (cov + cov.T) / 2.0
    lam, vecs = np.linalg.eigh(cov)
    lam = np.ascontiguousarray(lam[::-1][:k])
    return lam, sign_normalize(np.ascontiguousarray(vecs[:, ::-1][:, :k]))


def fit_pca_unsupervised(planes, region=None, k=None) -> dict:
    """projection.py:298-347 -- mean pass, 64-row centred Gram pass, correlation."""
    b, height, width = planes.shape
    if region is None:
        x0, y0, w, h = 0, 0, width, height
    else:
        x0, y0, w, h = region
        if w <= 0 or h <= 0:
            raise OracleError(f"empty region {region}")
        if x0 < 0 or y0 < 0 or x0 + w > width or y0 + h > height:
            raise OracleError(f"region {region} outside {width}x{height} stack")
    n = w * h
    if n < 2:
        raise OracleError("unsupervised PCA needs at least 2 pixels")
    k = _top_k(k, b)
    sub = planes[:, y0:y0 + h, x0:x0 + w]
    mean = np.array([sub[i].astype(np.float64).mean() for i in range(b)])
    gram = np.zeros((b, b))
    for r0 in range(0, h, ROW_CHUNK):
        block = sub[:, r0:r0 + ROW_CHUNK, :].reshape(b, -1).astype(np.float64)
        block -= mean[:, None]
        gram += block @ block.T
    std = np.sqrt(np.diag(gram) / (n - 1))
    std[std == 0.0] = 1.0
    lam, coef = _pca_eig(gram / (n - 1) / np.outer(std, std), k)
    return {
        "method": "pca_unsupervised",
        "mean": mean,
        "std": std,
        "coefficients": coef,
        "eigenvalues": lam,
        "training_scores": None,
        "gram": gram,
    }


# --------------------------------------------------------------------------
# projection.py -- projector
# --------------------------------------------------------------------------

def _project_block(planes, model, comps, out, r0, r1):
    """projection.py:371-388 -- per-chunk band-ordered multiply-then-add."""
    block = planes[:, r0:r1, :].astype(np.float64)
    block -= model["mean"][:, None, None]
    if model.get("std") is not None:
        block /= model["std"][:, None, None]
    coef = model["coefficients"]
    for slot, kk in enumerate(comps):
        acc = np.zeros_like(block[0])
        for i in range(block.shape[0]):
            acc += coef[i, kk] * block[i]
        out[slot, r0:r1, :] = acc


def project(planes, model, components=None, workers: int = 1) -> np.ndarray:
    """projection.py:391-439 -> (len(components), H, W) float64 score planes."""
    b, h, w = planes.shape
    coef = model["coefficients"]
    if coef.shape[0] != b:
        raise OracleError(f"stack has {b} bands but model expects {coef.shape[0]}")
    comps = list(range(coef.shape[1])) if components is None else list(components)
    for kk in comps:
        if not 0 <= kk < coef.shape[1]:
            raise OracleError(f"component {kk} out of range")
    out = np.empty((len(comps), h, w))
    spans = [(r, min(r + ROW_CHUNK, h)) for r in range(0, h, ROW_CHUNK)]
    if workers <= 1:
        for r0, r1 in spans:
            _project_block(planes, model, comps, out, r0, r1)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            for f in [pool.submit(_project_block, planes, model, comps, out, r0, r1)
                      for r0, r1 in spans]:
                f.result()
    return out


# --------------------------------------------------------------------------
# whole-path drivers used by bench.py's CPU arms
# --------------------------------------------------------------------------

def _workers(workers):
    return len(os.sched_getaffinity(0)) if workers is None else int(workers)


def cpu_cva_pipeline(planes, xs, ys, labels, k, ridge=RIDGE_DEFAULT, workers=None,
                     values=None):
    """assemble -> fit_cva -> project -> rescale_full per plane."""
    if values is None:
        values = assemble(planes, xs, ys)
    model = fit_cva(values, labels, k=k, ridge=ridge)
    scores = project(planes, model, workers=_workers(workers))
    codes = np.stack([rescale_full(s) for s in scores])
    return model, scores, codes


def cpu_pca_pipeline(planes, k, region=None, workers=None):
    """fit_pca_unsupervised -> project -> rescale_full per plane."""
    model = fit_pca_unsupervised(planes, region=region, k=k)
    scores = project(planes, model, workers=_workers(workers))
    codes = np.stack([rescale_full(s) for s in scores])
    return model, scores, codes
