"""Regularized generalized symmetric eigensolver on the device.

Drop-in for /root/reference/pkg/src/undertext/eigen.py: ``solve_gen_eig_sym``
(:75-113) runs in one CTA (``ut_gen_eig_sym``, csrc/eig.cu): ridge (:63-72),
Cholesky, C = L^-1 A L^-T, parallel cyclic Jacobi, V = L^-T U, descending
sort, sign normalization (:40-52).  Error behaviour matches: NumericError for
shape mismatch, asymmetry beyond 1e-10, or an M' that is not positive definite
(with the eigenvalue range and condition estimate of M' in the message).

``regularize`` and ``sign_normalize`` are kept as small host utilities for API
compatibility; the device solver applies both rules itself.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import NumericError

DEFAULT_RIDGE = 1e-8
_SYMMETRY_RTOL = 1e-10


@dataclass(frozen=True)
class EigenSolution:
    """Eigenvalues in descending order; eigenvector k in column k."""

    eigenvalues: np.ndarray
    eigenvectors: np.ndarray

    def __post_init__(self):
        self.eigenvalues.setflags(write=False)
        self.eigenvectors.setflags(write=False)


def sign_normalize(vectors: np.ndarray) -> np.ndarray:
    """Flip each column so its first largest-|entry| is positive (utility)."""
    out = np.array(vectors, dtype=np.float64, copy=True)
    lead = np.argmax(np.abs(out), axis=0)
    flip = out[lead, np.arange(out.shape[1])] < 0
    out[:, flip] *= -1.0
    return out


def regularize(M: np.ndarray, ridge: float = DEFAULT_RIDGE) -> np.ndarray:
    """M + ridge*(trace(M)/B)*I, or ridge*I when trace(M) <= 0 (utility)."""
    b = M.shape[0]
    tr = float(np.trace(M))
    return M + (ridge * (tr / b if tr > 0.0 else 1.0)) * np.eye(b)


def raise_for_info(info: int, aux: np.ndarray | None) -> None:
    """Map the device solver's info word onto the reference's exceptions."""
    if info == _lib.INFO_OK:
        return
    if info == _lib.INFO_ASYM_A:
        raise NumericError(f"matrix A is not symmetric within {_SYMMETRY_RTOL}")
    if info == _lib.INFO_ASYM_M:
        raise NumericError(f"matrix M is not symmetric within {_SYMMETRY_RTOL}")
    if info == _lib.INFO_NOT_PD:
        lo, hi = float(aux.min()), float(aux.max())
        cond = float("inf") if lo <= 0 else hi / lo
        raise NumericError(
            f"regularized M is not positive definite "
            f"(eigenvalue range [{lo:.3e}, {hi:.3e}], condition estimate {cond:.3e}); "
            f"increase the ridge or check the training data")
    if info == _lib.INFO_NO_CONVERGE:
        raise NumericError("eigensolver did not converge")
    raise NumericError(f"eigensolver failed with info {info}")


def solve_gen_eig_sym(A: np.ndarray, M: np.ndarray, ridge: float = DEFAULT_RIDGE) -> EigenSolution:
    """Solve A v = lambda M' v, M' = regularize(M, ridge) (eigen.py:75-113)."""
    A = np.asarray(A, dtype=np.float64)
    M = np.asarray(M, dtype=np.float64)
    if A.shape != M.shape or A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise NumericError(f"need square matrices of one size, got {A.shape} and {M.shape}")
    b = A.shape[0]
    if not 1 <= b <= 32:
        raise NumericError(f"device eigensolver handles 1..32 bands, got {b}")
    device = dev.require_cuda()
    a_d = dev.to_device(A, device)
    m_d = dev.to_device(M, device)
    out = torch.empty(b + b * b + b, dtype=torch.float64, device=device)
    info = torch.empty(1, dtype=torch.int32, device=device)
    evals, evecs, aux = out[:b], out[b:b + b * b], out[b + b * b:]
    _lib.check(_lib.lib().ut_gen_eig_sym(a_d.data_ptr(), m_d.data_ptr(), b, float(ridge),
                                         evals.data_ptr(), evecs.data_ptr(), aux.data_ptr(),
                                         info.data_ptr(), dev.stream_handle()), "ut_gen_eig_sym")
    host = out.cpu().numpy()
    raise_for_info(int(info.item()), host[b + b * b:])
    return EigenSolution(host[:b].copy(), host[b:b + b * b].reshape(b, b).copy())


def eigh_desc(C: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Standard symmetric problem, descending, sign-normalized orthonormal
    vectors (np.linalg.eigh + reverse + sign_normalize, projection.py:263-270)."""
    C = np.asarray(C, dtype=np.float64)
    b = C.shape[0]
    device = dev.require_cuda()
    c_d = dev.to_device(C, device)
    out = torch.empty(b + b * b, dtype=torch.float64, device=device)
    info = torch.empty(1, dtype=torch.int32, device=device)
    _lib.check(_lib.lib().ut_gen_eig_sym(c_d.data_ptr(), None, b, 0.0, out.data_ptr(),
                                         out[b:].data_ptr(), None, info.data_ptr(),
                                         dev.stream_handle()), "ut_gen_eig_sym")
    host = out.cpu().numpy()
    raise_for_info(int(info.item()), None)
    return host[:b].copy(), host[b:].reshape(b, b).copy()
