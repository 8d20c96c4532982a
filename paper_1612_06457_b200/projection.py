"""Scatter, CVA / PCA fits and the stack projector -- on the B200.

Drop-in for the hot-path functions of
/root/reference/pkg/src/undertext/projection.py with the same signatures,
return types and errors:

* ``compute_scatter(dm)``          (:172-201)  -> K1 ``ut_class_moments`` + ``ut_cva_solve``
* ``fit_cva(dm, k, ridge, prov)``  (:211-237)  -> K1 + K3 (one CTA eigensolve)
* ``fit_pca(dm, k, prov)``         (:273-295)  -> K2 over the design matrix + K3
* ``fit_pca_unsupervised(stack, region, k, prov)`` (:298-347) -> K2 + K3
* ``project_stack(stack, model, components, workers)`` (:391-439) -> K4
* ``standardize(dm)`` / ``fit_lda(dm, k, ridge, prov)`` (:152-169, :240-260) -> ``ut_standardize`` + K1 + K3
* ``fit(method, ...)``             (:350-368)

Host arrays in -> host arrays out (one H2D / D2H per call); ``DeviceStack`` /
device ``DesignMatrix`` inputs keep everything in HBM.  Inputs are duck-typed,
so the reference's own DesignMatrix / SpectralStack / ScorePlane objects are
accepted unchanged.  ``ProjectionModel`` and
``ScatterPair`` are the reference's types (JSON round trip included).
"""

from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _lib
from . import device as dev
from .annotations import DesignMatrix
from .eigen import DEFAULT_RIDGE, raise_for_info
from .errors import DataError, NumericError
from .rendering import DeviceScorePlane, ScorePlane
from .stack import DeviceStack, SpectralStack, on_device

METHOD_CVA = "cva"
METHOD_LDA = "lda"
METHOD_PCA = "pca"
METHOD_PCA_UNSUPERVISED = "pca_unsupervised"
SUPERVISED_METHODS = (METHOD_CVA, METHOD_LDA, METHOD_PCA)
ALL_METHODS = SUPERVISED_METHODS + (METHOD_PCA_UNSUPERVISED,)

MODEL_FORMAT = "undertext-projection-model"
MODEL_VERSION = 1

# Projector arithmetic: "fp64" (default) accumulates in fp64 like the
# reference; "fp32" is the centred-fp32 variant.
PRECISION = os.environ.get("UT_PRECISION", "fp64")


def _precision_flag(precision: str | None) -> int:
    p = PRECISION if precision is None else precision
    if p not in ("fp32", "fp64"):
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {p!r}")
    return 1 if p == "fp64" else 0


@dataclass(frozen=True)
class ScatterPair:
    """Pooled within-class and between-class scatter (projection.py:39-52)."""

    within: np.ndarray
    between: np.ndarray
    class_means: np.ndarray
    class_ids: tuple[int, ...]
    counts: np.ndarray
    grand_mean: np.ndarray


@dataclass(frozen=True)
class ProjectionModel:
    """A fitted linear projection (projection.py:55-149)."""

    method: str
    mean: np.ndarray
    std: np.ndarray | None
    coefficients: np.ndarray
    eigenvalues: np.ndarray
    training_scores: np.ndarray | None = None
    provenance: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.method not in ALL_METHODS:
            raise DataError(f"unknown method {self.method!r}")
        for arr in (self.mean, self.std, self.coefficients, self.eigenvalues,
                    self.training_scores):
            if arr is not None:
                arr.setflags(write=False)

    @property
    def band_count(self) -> int:
        return int(self.coefficients.shape[0])

    @property
    def component_count(self) -> int:
        return int(self.coefficients.shape[1])

    def apply(self, samples: np.ndarray) -> np.ndarray:
        """Project (n, B) samples onto all components -> (n, K) scores."""
        centered = np.asarray(samples, dtype=np.float64) - self.mean
        if self.std is not None:
            centered = centered / self.std
        return centered @ self.coefficients

    def to_dict(self) -> dict:
        return {
            "format": MODEL_FORMAT,
            "version": MODEL_VERSION,
            "method": self.method,
            "bands": self.band_count,
            "components": self.component_count,
            "mean": self.mean.tolist(),
            "std": None if self.std is None else self.std.tolist(),
            "eigenvalues": self.eigenvalues.tolist(),
            "coefficients": self.coefficients.tolist(),
            "training_scores": None if self.training_scores is None
            else self.training_scores.tolist(),
            "provenance": self.provenance,
        }

    def save(self, path) -> None:
        """JSON; floats serialize via repr, which round-trips binary64."""
        Path(path).write_text(json.dumps(self.to_dict(), indent=1) + "\n", encoding="utf-8")

    @classmethod
    def from_dict(cls, doc: dict) -> "ProjectionModel":
        if doc.get("format") != MODEL_FORMAT:
            raise DataError(f"not a projection model document: {doc.get('format')!r}")
        if doc.get("version") != MODEL_VERSION:
            raise DataError(f"unsupported model version {doc.get('version')!r}")
        f64 = lambda v: None if v is None else np.asarray(v, dtype=np.float64)  # noqa: E731
        return cls(method=doc["method"], mean=f64(doc["mean"]), std=f64(doc["std"]),
                   coefficients=f64(doc["coefficients"]), eigenvalues=f64(doc["eigenvalues"]),
                   training_scores=f64(doc["training_scores"]),
                   provenance=doc.get("provenance", {}))

    @classmethod
    def load(cls, path) -> "ProjectionModel":
        try:
            doc = json.loads(Path(path).read_text(encoding="utf-8"))
        except json.JSONDecodeError as exc:
            raise DataError(f"{path}: not a model file: {exc}") from exc
        return cls.from_dict(doc)


def _top_k(requested, band_count: int) -> int:
    k = band_count if requested is None else int(requested)
    if not 1 <= k <= band_count:
        raise DataError(f"requested {k} components from {band_count} bands")
    return k


def class_index(labels) -> tuple[tuple[int, ...], np.ndarray]:
    """Sorted unique label ids (projection.py:179) and each point's index into them."""
    labels = np.asarray(labels)
    ids = np.unique(labels)
    return tuple(int(c) for c in ids), np.searchsorted(ids, labels).astype(np.int32)


# --------------------------------------------------------------- device fits

class CvaDevice:
    """Device buffers of one CVA fit (moments -> scatter -> eigen)."""

    def __init__(self, bands: int, classes: int, device, groups: int = 1):
        self.b, self.c, self.groups = bands, classes, groups
        self.mlen = int(_lib.lib().ut_moment_len(bands))
        b, c = bands, classes
        self.moments = torch.zeros(groups * c * self.mlen, dtype=torch.float64, device=device)
        # sharded fits: this rank's record lives in its own buffer; as a slice of
        # `moments` it would overlap the all_gather output of rank 0's slot
        self._local = self.moments[: c * self.mlen] if groups == 1 else \
            torch.zeros(c * self.mlen, dtype=torch.float64, device=device)
        sizes = dict(within=b * b, between=b * b, class_means=c * b, counts=c, grand_mean=b,
                     evals=b, evecs=b * b, aux=b)
        total = sum(sizes.values())
        self.flat = torch.zeros(total, dtype=torch.float64, device=device)
        self.views, off = {}, 0
        for name, n in sizes.items():
            self.views[name] = self.flat[off:off + n]
            off += n
        self.info = torch.zeros(1, dtype=torch.int32, device=device)
        self.out = _lib.CvaOut(*(self.views[n].data_ptr() for n in sizes), self.info.data_ptr())

    def local_moments(self) -> torch.Tensor:
        return self._local

    def moments_from(self, values: torch.Tensor, ld: int, cls_d: torch.Tensor, n: int):
        L = _lib.lib()
        if n == 0:
            self.local_moments().zero_()
            return
        need = L.ut_class_moments_ws(n, self.b, self.c)
        ws = dev.workspace("class_moments", need, values.device)
        _lib.check(L.ut_class_moments(values.data_ptr(), ld, cls_d.data_ptr(), n, self.b, self.c,
                                      None, self._local.data_ptr(), ws.data_ptr(), ws.numel(),
                                      dev.stream_handle()), "ut_class_moments")

    def moments_from_cube(self, cube, xy_d: torch.Tensor, cls_d: torch.Tensor, n: int,
                          first_bad: torch.Tensor, pivots: torch.Tensor | None = None):
        """Fused K1: gather the n training pixels from the cube + class moments."""
        L = _lib.lib()
        if n == 0:
            self.local_moments().zero_()
            return
        ws = dev.workspace("class_moments", L.ut_class_moments_ws(n, self.b, self.c),
                           xy_d.device)
        _lib.check(L.ut_cube_class_moments(C.byref(cube), xy_d.data_ptr(), cls_d.data_ptr(), n,
                                           self.c, None if pivots is None else pivots.data_ptr(),
                                           self._local.data_ptr(), first_bad.data_ptr(),
                                           ws.data_ptr(), ws.numel(), dev.stream_handle()),
                   "ut_cube_class_moments")

    def solve(self, ridge: float, want: int = 0):
        """K3; ``want`` leading eigenvectors (0 = all B)."""
        _lib.check(_lib.lib().ut_cva_solve(self.moments.data_ptr(), self.groups, self.b, self.c,
                                           float(ridge), int(want), C.byref(self.out),
                                           dev.stream_handle()), "ut_cva_solve")

    def host(self) -> dict:
        flat = self.flat.cpu().numpy()
        info = int(self.info.item())
        out, off = {}, 0
        for name, v in self.views.items():
            out[name] = flat[off:off + v.numel()].copy()
            off += v.numel()
        b, c = self.b, self.c
        for name in ("within", "between", "evecs"):
            out[name] = out[name].reshape(b, b)
        out["class_means"] = out["class_means"].reshape(c, b)
        out["info"] = info
        return out


def _on_device(dm) -> bool:
    """Whether a design matrix's values live in HBM.  Duck-typed: the
    reference's DesignMatrix (annotations.py:69-103, numpy values, no
    ``on_device``) is accepted everywhere ours is."""
    return isinstance(dm.values, torch.Tensor)


def _design_device(dm):
    return dm.values.device if _on_device(dm) else dev.require_cuda()


def _design_on_device(dm, device):
    if _on_device(dm):
        v = dm.values
        if v.dtype != torch.float64:
            v = v.double()
        if v.stride(1) != 1:
            v = v.contiguous()
        return v, v.stride(0)
    v = dev.to_device(np.asarray(dm.values, dtype=np.float64), device)
    return v, v.shape[1]


def _scatter_device(dm: DesignMatrix, ridge: float, want: int = 0):
    ids, cls = class_index(dm.labels)
    if len(ids) < 2:
        raise DataError(f"scatter needs at least 2 classes with points, got {len(ids)}")
    if dm.band_count > 32:
        raise DataError(f"the device path supports up to 32 bands, got {dm.band_count}")
    device = _design_device(dm)
    with torch.cuda.device(device):
        values, ld = _design_on_device(dm, device)
        cls_d = dev.to_device(cls, device)
        fit = CvaDevice(dm.band_count, len(ids), device)
        fit.moments_from(values, ld, cls_d, dm.point_count)
        fit.solve(ridge, want)
        return ids, fit.host()


def compute_scatter(dm: DesignMatrix) -> ScatterPair:
    """Pooled within/between-class scatter, symmetrized (projection.py:172-201)."""
    ids, h = _scatter_device(dm, DEFAULT_RIDGE, want=1)
    return ScatterPair(h["within"], h["between"], h["class_means"], ids,
                       h["counts"].astype(np.intp), h["grand_mean"])


def _training_scores(dm: DesignMatrix, coeffs: np.ndarray, mean: np.ndarray):
    """coeffs^T (X - m) (projection.py:228); computed with the same numpy
    expression as ``ProjectionModel.apply`` so the two agree bit for bit
    (tests/test_projection.py:122-127) -- bookkeeping, not on the hot path."""
    if _on_device(dm):
        x = dm.values.double()
        c = torch.from_numpy(coeffs).to(x.device)
        m = torch.from_numpy(mean).to(x.device)
        return ((x - m[:, None]).T @ c).cpu().numpy()
    return (np.asarray(dm.values, dtype=np.float64).T - mean) @ coeffs


def fit_cva(dm: DesignMatrix, k: int | None = None, ridge: float = DEFAULT_RIDGE,
            provenance: dict | None = None) -> ProjectionModel:
    """Canonical variates on raw values (projection.py:211-237)."""
    k = _top_k(k, dm.band_count)
    ids, h = _scatter_device(dm, ridge, want=k)
    raise_for_info(h["info"], h["aux"])
    coeffs = np.ascontiguousarray(h["evecs"][:, :k])
    mean = h["grand_mean"]
    return ProjectionModel(method=METHOD_CVA, mean=mean, std=None, coefficients=coeffs,
                           eigenvalues=np.ascontiguousarray(h["evals"][:k]),
                           training_scores=np.ascontiguousarray(_training_scores(dm, coeffs, mean).T),
                           provenance=provenance or {})


def standardize(dm) -> tuple[DesignMatrix, np.ndarray, np.ndarray]:
    """Recentre each band row to mean 0 and sample standard deviation 1
    (projection.py:152-169): divisor N - 1, constant rows centred only with
    std 1; N >= 2.  One device pass per row (``ut_standardize``); a host matrix
    gives a host matrix, a device matrix stays in HBM."""
    if dm.point_count < 2:
        raise DataError("standardization needs at least 2 points")
    device = _design_device(dm)
    b, n = dm.band_count, dm.point_count
    with torch.cuda.device(device):
        values, ld = _design_on_device(dm, device)
        out = torch.empty((b, n), dtype=torch.float64, device=device)
        ms = torch.empty(2 * b, dtype=torch.float64, device=device)
        _lib.check(_lib.lib().ut_standardize(values.data_ptr(), ld, b, n, out.data_ptr(), n,
                                             ms.data_ptr(), ms[b:].data_ptr(),
                                             dev.stream_handle()), "ut_standardize")
        host_ms = ms.cpu().numpy()
        labels = np.array(dm.labels)
        names = tuple(dm.class_names)
        if _on_device(dm):
            return DesignMatrix(out, labels, names), host_ms[:b].copy(), host_ms[b:].copy()
        return (DesignMatrix(out.cpu().numpy(), labels, names), host_ms[:b].copy(),
                host_ms[b:].copy())


def fit_lda(dm, k: int | None = None, ridge: float = DEFAULT_RIDGE,
            provenance: dict | None = None) -> ProjectionModel:
    """Two-class discriminant: the CVA core (K1 + K3) on the standardized
    matrix (projection.py:240-260)."""
    present = np.unique(np.asarray(dm.labels))
    if len(present) != 2:
        raise DataError(f"LDA requires exactly 2 classes, got {len(present)}")
    sdm, mean, std = standardize(dm)
    core = fit_cva(sdm, k=k, ridge=ridge)
    return ProjectionModel(method=METHOD_LDA, mean=mean, std=std,
                           coefficients=core.coefficients, eigenvalues=core.eigenvalues,
                           training_scores=core.training_scores,
                           provenance=provenance or {})


class PcaDevice:
    """Device buffers of one PCA fit (region moments -> correlation -> eigen)."""

    def __init__(self, bands: int, device, groups: int = 1):
        self.b, self.groups = bands, groups
        self.mlen = int(_lib.lib().ut_moment_len(bands))
        b = bands
        self.moments = torch.zeros(groups * self.mlen, dtype=torch.float64, device=device)
        self._local = self.moments[: self.mlen] if groups == 1 else \
            torch.zeros(self.mlen, dtype=torch.float64, device=device)  # see CvaDevice
        sizes = dict(mean=b, std=b, corr=b * b, evals=b, evecs=b * b)
        self.flat = torch.zeros(sum(sizes.values()), dtype=torch.float64, device=device)
        self.views, off = {}, 0
        for name, n in sizes.items():
            self.views[name] = self.flat[off:off + n]
            off += n
        self.info = torch.zeros(1, dtype=torch.int32, device=device)
        self.out = _lib.PcaOut(*(self.views[n].data_ptr() for n in sizes), self.info.data_ptr())

    def local_moments(self) -> torch.Tensor:
        return self._local

    def moments_from(self, cube, x0, y0, w, h, device):
        L = _lib.lib()
        ws = dev.workspace("region_moments", L.ut_region_moments_ws(self.b), device)
        _lib.check(L.ut_region_moments(C.byref(cube), x0, y0, w, h, self._local.data_ptr(),
                                       ws.data_ptr(), ws.numel(), dev.stream_handle()),
                   "ut_region_moments")

    def region_path(self, device) -> tuple[int, int]:
        """(path of this thread's last region pass -- _lib.UT_REGION_PATH_*, the
        integer path's range flag: 1 if it handed the region to the fp64 path).
        Synchronizes; diagnostics for tests."""
        L = _lib.lib()
        ws = dev.workspace("region_moments", L.ut_region_moments_ws(self.b), device)
        off = int(L.ut_region_flag_offset())
        flag = int(ws[off:off + 4].view(torch.int32).item())
        return int(L.ut_region_last_path()), flag

    def solve(self):
        _lib.check(_lib.lib().ut_pca_solve(self.moments.data_ptr(), self.groups, self.b,
                                           C.byref(self.out), dev.stream_handle()), "ut_pca_solve")

    def host(self) -> dict:
        flat = self.flat.cpu().numpy()
        out, off = {}, 0
        for name, v in self.views.items():
            out[name] = flat[off:off + v.numel()].copy()
            off += v.numel()
        out["corr"] = out["corr"].reshape(self.b, self.b)
        out["evecs"] = out["evecs"].reshape(self.b, self.b)
        out["info"] = int(self.info.item())
        return out


def _pca_model(h: dict, k: int, method: str, provenance, training_scores=None):
    raise_for_info(h["info"], None)
    return ProjectionModel(method=method, mean=h["mean"], std=h["std"],
                           coefficients=np.ascontiguousarray(h["evecs"][:, :k]),
                           eigenvalues=np.ascontiguousarray(h["evals"][:k]),
                           training_scores=training_scores, provenance=provenance or {})


def fit_pca_unsupervised(stack, region: tuple[int, int, int, int] | None = None,
                         k: int | None = None, provenance: dict | None = None) -> ProjectionModel:
    """PCA over every pixel of a stack region (projection.py:298-347)."""
    if region is None:
        x0, y0, w, h = 0, 0, stack.width, stack.height
    else:
        x0, y0, w, h = (int(v) for v in region)
        if w <= 0 or h <= 0:
            raise DataError(f"empty region {region}")
        if x0 < 0 or y0 < 0 or x0 + w > stack.width or y0 + h > stack.height:
            raise DataError(f"region {region} outside {stack.width}x{stack.height} stack")
    if w * h < 2:
        raise DataError("unsupervised PCA needs at least 2 pixels")
    k = _top_k(k, stack.band_count)
    ds = on_device(stack)
    device = ds.planes.device
    with torch.cuda.device(device):
        fit = PcaDevice(ds.band_count, device)
        fit.moments_from(ds.cube(), x0, y0, w, h, device)
        fit.solve()
        hres = fit.host()
    return _pca_model(hres, k, METHOD_PCA_UNSUPERVISED, provenance)


def fit_pca(dm: DesignMatrix, k: int | None = None,
            provenance: dict | None = None) -> ProjectionModel:
    """Principal components of the standardized design matrix
    (projection.py:273-295): the design matrix is viewed as a (B, 1, N) cube
    and reduced by the same K2 + K3 kernels as the unsupervised fit."""
    if dm.point_count < 2:
        raise DataError("standardization needs at least 2 points")
    k = _top_k(k, dm.band_count)
    device = _design_device(dm)
    with torch.cuda.device(device):
        values, ld = _design_on_device(dm, device)
        cube = _lib.Cube(values.data_ptr(), _lib.UT_F64, dm.band_count, 1, dm.point_count, ld,
                         ld, 0)
        fit = PcaDevice(dm.band_count, device)
        fit.moments_from(cube, 0, 0, dm.point_count, 1, device)
        fit.solve()
        hres = fit.host()
    x = np.asarray(dm.values.cpu().numpy() if _on_device(dm) else dm.values, dtype=np.float64)
    coeffs = np.ascontiguousarray(hres["evecs"][:, :k])
    scores = coeffs.T @ ((x - hres["mean"][:, None]) / hres["std"][:, None])
    return _pca_model(hres, k, METHOD_PCA, provenance, training_scores=scores)


def fit(method: str, dm: DesignMatrix | None = None, stack=None, region=None, k=None,
        ridge: float = DEFAULT_RIDGE, provenance: dict | None = None) -> ProjectionModel:
    """Dispatch a fit by method tag (projection.py:350-368)."""
    if method == METHOD_CVA:
        return fit_cva(dm, k=k, ridge=ridge, provenance=provenance)
    if method == METHOD_LDA:
        return fit_lda(dm, k=k, ridge=ridge, provenance=provenance)
    if method == METHOD_PCA:
        return fit_pca(dm, k=k, provenance=provenance)
    if method == METHOD_PCA_UNSUPERVISED:
        return fit_pca_unsupervised(stack, region=region, k=k, provenance=provenance)
    raise DataError(f"unknown method {method!r}; expected one of {ALL_METHODS}")


# --------------------------------------------------------------- projector

def project_device(ds: DeviceStack, coef_d: torch.Tensor, mean_d: torch.Tensor,
                   std_d: torch.Tensor | None, components, precision=None,
                   scores: torch.Tensor | None = None, minmax: torch.Tensor | None = None,
                   nonfinite: torch.Tensor | None = None):
    """K4 on a device stack: (K, rows, W) fp32 scores + [-min.., max..] record."""
    k = len(components)
    device = ds.planes.device
    if scores is None:
        scores = torch.empty((k, ds.height, ds.width), dtype=torch.float32, device=device)
    if minmax is None:
        minmax = torch.empty(2 * k, dtype=torch.float32, device=device)
    if nonfinite is None:
        nonfinite = torch.empty(1, dtype=torch.int32, device=device)
    L = _lib.lib()
    ws = dev.workspace("project", L.ut_project_ws(), device)
    comps = (C.c_int32 * k)(*[int(c) for c in components])
    _lib.check(L.ut_project_minmax(C.byref(ds.cube()), coef_d.data_ptr(), coef_d.shape[1],
                                   C.cast(comps, C.c_void_p), k, mean_d.data_ptr(),
                                   None if std_d is None else std_d.data_ptr(),
                                   _precision_flag(precision), scores.data_ptr(),
                                   minmax.data_ptr(), nonfinite.data_ptr(), ws.data_ptr(),
                                   ws.numel(), dev.stream_handle()), "ut_project_minmax")
    return scores, minmax, nonfinite


def project_stack(stack, model: ProjectionModel, components: list[int] | None = None,
                  workers: int = 1, precision: str | None = None) -> list:
    """Project every pixel onto the model's coefficient columns
    (projection.py:391-439).  Host stack -> list[ScorePlane] (float64 values
    of the fp32 device planes); DeviceStack -> list[DeviceScorePlane].
    ``workers`` is accepted for signature compatibility: the device result does
    not depend on it (every pixel is summed in band order by one thread)."""
    if stack.band_count != model.band_count:
        raise DataError(f"stack has {stack.band_count} bands but model expects "
                        f"{model.band_count}")
    fitted_normalized = model.provenance.get("normalized_input")
    if fitted_normalized is not None and fitted_normalized != stack.normalized:
        raise DataError("model was fitted on normalized data" if fitted_normalized
                        else "model was fitted on unnormalized data")
    if components is None:
        components = list(range(model.component_count))
    for kk in components:
        if not 0 <= kk < model.component_count:
            raise DataError(f"component {kk} out of range")
    if not components:
        return []
    ds = on_device(stack)
    device = ds.planes.device
    planes = []
    with torch.cuda.device(device):
        coef_d = dev.to_device(np.ascontiguousarray(model.coefficients), device)
        mean_d = dev.to_device(np.ascontiguousarray(model.mean), device)
        std_d = None if model.std is None else dev.to_device(np.ascontiguousarray(model.std), device)
        # K4 handles up to 32 components per call
        for start in range(0, len(components), 32):
            chunk = components[start:start + 32]
            scores, minmax, bad = project_device(ds, coef_d, mean_d, std_d, chunk, precision)
            if int(bad.item()):
                raise DataError("score plane contains NaN or Inf")
            if isinstance(stack, DeviceStack):
                planes += [DeviceScorePlane(scores, minmax, i) for i in range(len(chunk))]
            else:
                host = scores.cpu().numpy().astype(np.float64)
                planes += [ScorePlane(host[i]) for i in range(len(chunk))]
    return planes
