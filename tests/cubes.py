"""Seeded host-side cube generator for the parity tests (small sizes only).

Follows the BASELINE.json generator recipe: class means
U[0.2, 0.8]; covariance A A^T/16 + 1e-3 I with A ~ N(0, 0.02^2) shared by all
classes (or A_c A_c^T/32 + 1e-3 I per class); class 0 background plus axis-aligned
rectangles for classes 1..C-1 (optionally elliptic "stain" blobs for the last
class); pixel = mean + L z, clipped to [0, 1], then cast -- uint16 as
round_half_away(4095 v).  Training pixels are drawn per class without
replacement.  The bench uses the CUDA generator in
``paper_1612_06457_b200.synthetic`` for the full-size configs; the tests here only
need *some* seeded input that both the oracle and the device see identically.
"""

from __future__ import annotations

import numpy as np


def class_map(h, w, classes, rng, blobs=False):
    cmap = np.zeros((h, w), dtype=np.int32)
    for c in range(1, classes):
        if blobs and c == classes - 1:
            yy, xx = np.mgrid[0:h, 0:w]
            for _ in range(3):
                cy, cx = rng.integers(0, h), rng.integers(0, w)
                ry, rx = max(2, h // 6), max(2, w // 5)
                inside = ((yy - cy) ** 2) * rx * rx + ((xx - cx) ** 2) * ry * ry <= (rx * ry) ** 2
                cmap[inside] = c
            continue
        for _ in range(4):
            rh, rw = max(1, int(h * 0.32)), max(1, int(w * 0.32))
            y0 = int(rng.integers(0, h - rh + 1))
            x0 = int(rng.integers(0, w - rw + 1))
            cmap[y0:y0 + rh, x0:x0 + rw] = c
    return cmap


def make_cube(h, w, bands, classes, dtype, seed, per_class, per_class_cov=False,
              blobs=False):
    rng = np.random.default_rng(seed)
    means = rng.uniform(0.2, 0.8, size=(classes, bands))
    if per_class_cov:
        chol = []
        for _ in range(classes):
            a = rng.normal(size=(bands, bands)) * 0.02
            chol.append(np.linalg.cholesky(a @ a.T / 32 + 1e-3 * np.eye(bands)))
    else:
        a = rng.normal(size=(bands, bands)) * 0.02
        chol = [np.linalg.cholesky(a @ a.T / 16 + 1e-3 * np.eye(bands))] * classes
    cmap = class_map(h, w, classes, rng, blobs=blobs)
    flat = cmap.reshape(-1)
    z = rng.normal(size=(h * w, bands))
    pix = means[flat].copy()
    for c in range(classes):
        sel = flat == c
        pix[sel] += z[sel] @ chol[c].T
    pix = np.clip(pix, 0.0, 1.0)
    cube = np.ascontiguousarray(pix.T.reshape(bands, h, w))
    if dtype == np.uint16:
        v = 4095.0 * cube
        cube = (np.sign(v) * np.floor(np.abs(v) + 0.5)).astype(np.uint16)
    else:
        cube = cube.astype(dtype)
    xs, ys, labels = [], [], []
    for c in range(classes):
        idx = np.flatnonzero(flat == c)
        take = rng.choice(idx, size=min(per_class, len(idx)), replace=False)
        ys += list(take // w)
        xs += list(take % w)
        labels += [c] * len(take)
    return (cube, np.array(xs, dtype=np.int32), np.array(ys, dtype=np.int32),
            np.array(labels, dtype=np.int32))
