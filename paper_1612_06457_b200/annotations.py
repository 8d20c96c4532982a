"""Training points and the design matrix gathered from them.

Mirrors the reference types (/root/reference/pkg/src/undertext/annotations.py:
ClassLabel :24-31, AnnotatedPoint :34-38, TrainingSet :41-66, DesignMatrix
:69-103) and replaces ``assemble_matrix``'s Python point loop (:195-215) with
the K1 gather kernel (``ut_gather``).  The CSV dialect (parse/serialize) is
host I/O outside the hot path and is not reimplemented.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import DataError
from .stack import DeviceStack, on_device


@dataclass(frozen=True)
class ClassLabel:
    name: str
    id: int

    def __post_init__(self):
        if not self.name:
            raise DataError("class name must be non-empty")


@dataclass(frozen=True)
class AnnotatedPoint:
    x: int
    y: int
    label: ClassLabel


@dataclass(frozen=True)
class TrainingSet:
    """Annotated points grouped by named classes, in declaration order."""

    classes: tuple[ClassLabel, ...]
    points: tuple[AnnotatedPoint, ...]
    provenance: dict = field(default_factory=dict)

    def counts(self) -> dict[str, int]:
        by_name = {c.name: 0 for c in self.classes}
        for p in self.points:
            by_name[p.label.name] += 1
        return by_name

    def arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(xs, ys, label ids) as int arrays, in point order."""
        n = len(self.points)
        xs = np.fromiter((p.x for p in self.points), dtype=np.int64, count=n)
        ys = np.fromiter((p.y for p in self.points), dtype=np.int64, count=n)
        ids = np.fromiter((p.label.id for p in self.points), dtype=np.int64, count=n)
        return xs, ys, ids

    @classmethod
    def from_arrays(cls, xs, ys, labels, names=None) -> "TrainingSet":
        ids = sorted({int(v) for v in labels})
        names = names or {c: f"class{c}" for c in ids}
        lab = {c: ClassLabel(names[c], c) for c in ids}
        pts = tuple(AnnotatedPoint(int(x), int(y), lab[int(l)]) for x, y, l in zip(xs, ys, labels))
        return cls(tuple(lab[c] for c in ids), pts)


@dataclass(frozen=True)
class DesignMatrix:
    """B x N spectral matrix plus labels (annotations.py:69-103).

    ``values`` is a float64 numpy array (host path) or a CUDA float64 tensor
    (device-resident path); ``labels`` is always a host integer array.
    """

    values: object
    labels: np.ndarray
    class_names: tuple[str, ...]

    def __post_init__(self):
        shape = tuple(self.values.shape)
        if len(shape) != 2:
            raise DataError("design matrix must be 2-D (bands x points)")
        if shape[1] != self.labels.shape[0]:
            raise DataError(f"{shape[1]} columns vs {self.labels.shape[0]} labels")
        if isinstance(self.values, np.ndarray):
            self.values.setflags(write=False)
        self.labels.setflags(write=False)

    @property
    def band_count(self) -> int:
        return int(self.values.shape[0])

    @property
    def point_count(self) -> int:
        return int(self.values.shape[1])

    @property
    def on_device(self) -> bool:
        return isinstance(self.values, torch.Tensor)

    def class_counts(self) -> dict[str, int]:
        return {name: int(np.sum(self.labels == cid)) for cid, name in enumerate(self.class_names)}


def point_arrays(ts) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(xs, ys, label ids) of any training set with ``points`` of (x, y, label.id)
    -- ours or the reference's TrainingSet (annotations.py:41-66)."""
    if isinstance(ts, TrainingSet):
        return ts.arrays()
    pts = ts.points
    n = len(pts)
    return (np.fromiter((p.x for p in pts), dtype=np.int64, count=n),
            np.fromiter((p.y for p in pts), dtype=np.int64, count=n),
            np.fromiter((p.label.id for p in pts), dtype=np.int64, count=n))


def check_points(xs, ys, width: int, row0: int, rows: int, names=None) -> None:
    """DataError for the first point outside the (shard of the) stack."""
    xs = np.asarray(xs)
    ys = np.asarray(ys)
    bad = (xs < 0) | (xs >= width) | (ys < row0) | (ys >= row0 + rows)
    if bad.any():
        j = int(np.argmax(bad))
        who = f" of class {names[j]!r}" if names is not None else ""
        raise DataError(f"point ({int(xs[j])}, {int(ys[j])}){who} outside "
                        f"{width}x{row0 + rows} stack")


def gather(stack: DeviceStack, xy: torch.Tensor, n: int) -> torch.Tensor:
    """K1 gather: (B, n) float64 device matrix of the samples at xy (2n int32)."""
    values = torch.empty((stack.band_count, max(n, 1)), dtype=torch.float64,
                         device=stack.planes.device)
    first_bad = torch.empty(1, dtype=torch.int64, device=stack.planes.device)
    cube = stack.cube()
    _lib.check(_lib.lib().ut_gather(cube, xy.data_ptr(), n, values.data_ptr(), values.shape[1],
                                    first_bad.data_ptr(), dev.stream_handle()), "ut_gather")
    return values[:, :n], first_bad


def assemble_matrix(stack, ts: TrainingSet) -> DesignMatrix:
    """Sample the stack at every annotated point, in point order
    (annotations.py:195-215).  Host stacks give a host matrix (as the
    reference); DeviceStacks keep it in HBM."""
    if not stack.normalized:
        raise DataError("assemble_matrix requires a normalized stack")
    if not ts.points:
        raise DataError("training set has no points")
    xs, ys, ids = point_arrays(ts)
    ds = on_device(stack)
    check_points(xs, ys, ds.width, ds.row0, ds.height, [p.label.name for p in ts.points])
    with torch.cuda.device(ds.planes.device):
        xy = dev.to_device(np.stack([xs, ys], axis=1).astype(np.int32), ds.planes.device)
        values, first_bad = gather(ds, xy, len(xs))
        names = tuple(c.name for c in ts.classes)
        if isinstance(stack, DeviceStack):
            return DesignMatrix(values, ids.astype(np.intp), names)
        host = values.cpu().numpy()
    if int(first_bad.item()) >= 0:  # cannot happen after check_points; ABI safety net
        raise DataError(f"point index {int(first_bad.item())} outside the stack")
    return DesignMatrix(np.ascontiguousarray(host), ids.astype(np.intp), names)
