"""Helpers shared by the parity tests: golden-fixture loading and the
comparison rules of SURVEY.md Appendix A."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def rel_close(got, want, rtol: float) -> bool:
    """max|got - want| <= rtol * max|want| (per-matrix relative bar)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.shape != want.shape:
        return False
    scale = float(np.abs(want).max()) if want.size else 0.0
    return float(np.abs(got - want).max(initial=0.0)) <= rtol * max(scale, 1e-300)


def align_signs(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """Flip columns of ``got`` (B x K) to the sign of ``want`` (Appendix A:
    near-ties in the largest-|entry| rule may flip a component)."""
    out = np.array(got, dtype=np.float64, copy=True)
    for j in range(out.shape[1]):
        if float(out[:, j] @ want[:, j]) < 0:
            out[:, j] = -out[:, j]
    return out


def plane_close(got, want, rtol: float = 1e-6) -> float:
    """Worst per-plane error / (max - min of the reference plane)."""
    worst = 0.0
    for g, w in zip(got, want):
        rng = float(w.max() - w.min()) or 1.0
        worst = max(worst, float(np.abs(np.asarray(g, np.float64) - w).max()) / rng)
    return worst
