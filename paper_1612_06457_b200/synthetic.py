"""Seeded synthetic cubes for the BASELINE.json configurations.

The reference ships no dataset for this path; BASELINE.json describes the
generator (see also SURVEY.md §8(d) and DESIGN.md §6):

* class means ~ U[0.2, 0.8] per band; covariance A A^T/16 + 1e-3 I with
  A ~ N(0, 0.02^2) shared by all classes (cfg 4: A_c A_c^T/32 + 1e-3 I per class);
* class 0 background plus axis-aligned rectangles of classes 1..C-1, ~10 % of
  the image each (4 rectangles of 16 % x 16 % of the sides); for the palimpsest
  configs the last class ("stains") is a union of 4 low-frequency ellipses;
* pixel = mean[class] + L z, clipped to [0, 1], cast to the config dtype
  (uint16: round_half_away(4095 v));
* ``per_class`` training pixels per class, uniform without replacement.

Host side (numpy ``default_rng(seed)``): means, Cholesky factors, the shape
list and the training points (rejection sampling against the same integer
class map).  Device side (``ut_synth_cube``): the pixels, from a counter hash
of (seed, pixel, band), so a 34 GB cube is generated in HBM in well under a
second and any row shard can be generated independently.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dev
from .stack import DeviceStack, default_bands


@dataclass(frozen=True)
class Config:
    name: str
    height: int
    width: int
    bands: int
    dtype: torch.dtype
    classes: int
    per_class: int
    k: int
    method: str = "cva"
    per_class_cov: bool = False
    blobs: bool = False
    seed: int = 0

    @property
    def pixels(self) -> int:
        return self.height * self.width

    @property
    def sample_bytes(self) -> int:
        return torch.empty((), dtype=self.dtype).element_size()

    def bytes_per_pixel(self) -> int:
        """Algorithmic bytes per pixel: one cube read per
        data-dependent pass plus the K uint8 codes written."""
        passes = 1 if self.method == "cva" else 2
        return passes * self.bands * self.sample_bytes + self.k


CONFIGS = {
    "cfg1": Config("cfg1_cva_512x512x16_f64", 512, 512, 16, torch.float64, 3, 500, 2, seed=1),
    "cfg2": Config("cfg2_pca_2048x2048x16_f32", 2048, 2048, 16, torch.float32, 3, 0, 3,
                   method="pca", seed=2),
    "cfg3": Config("cfg3_cva_7216x5412x23_u16", 7216, 5412, 23, torch.uint16, 4, 2000, 3,
                   blobs=True, seed=3),
    "cfg4": Config("cfg4_cva_16384x16384x32_f32", 16384, 16384, 32, torch.float32, 6, 10000, 5,
                   per_class_cov=True, seed=4),
    "cfg4pca": Config("cfg4_pca_16384x16384x32_f32", 16384, 16384, 32, torch.float32, 6, 0, 5,
                      method="pca", per_class_cov=True, seed=4),
    "cfg5": Config("cfg5_cva_folio_4096x3072x23_f16", 4096, 3072, 23, torch.float16, 4, 1000, 3,
                   blobs=True, seed=5),
}


def scaled(cfg: Config, height: int, width: int, per_class: int | None = None) -> Config:
    """The same generator at a smaller size (parity tests, CPU samples)."""
    from dataclasses import replace
    return replace(cfg, name=f"{cfg.name}@{height}x{width}", height=height, width=width,
                   per_class=cfg.per_class if per_class is None else per_class)


@dataclass
class Scene:
    """Everything the host knows about a generated cube."""

    cfg: Config
    means: np.ndarray       # (C, B)
    chol: np.ndarray        # (C, B, B)
    shapes: np.ndarray      # (S, 6) int64: kind, class, a, b, c, d
    xs: np.ndarray
    ys: np.ndarray
    labels: np.ndarray


def class_map_at(shapes: np.ndarray, ys, xs) -> np.ndarray:
    """Integer class map (same arithmetic as class_at in csrc/synth.cu)."""
    ys = np.asarray(ys, dtype=np.int64)
    xs = np.asarray(xs, dtype=np.int64)
    out = np.zeros(np.broadcast(ys, xs).shape, dtype=np.int32)
    for kind, cls, a, b, c, d in shapes.tolist():
        if kind == 0:
            inside = (ys >= a) & (xs >= b) & (ys < c) & (xs < d)
        else:
            dy, dx = ys - a, xs - b
            inside = (dy * d) ** 2 + (dx * c) ** 2 <= (c * d) ** 2
        out[inside] = cls
    return out


def make_scene(cfg: Config) -> Scene:
    rng = np.random.default_rng(cfg.seed)
    b, c = cfg.bands, cfg.classes
    means = rng.uniform(0.2, 0.8, size=(c, b))
    if cfg.per_class_cov:
        chol = []
        for _ in range(c):
            a = rng.normal(size=(b, b)) * 0.02
            chol.append(np.linalg.cholesky(a @ a.T / 32 + 1e-3 * np.eye(b)))
        chol = np.stack(chol)
    else:
        a = rng.normal(size=(b, b)) * 0.02
        chol = np.repeat(np.linalg.cholesky(a @ a.T / 16 + 1e-3 * np.eye(b))[None], c, axis=0)
    h, w = cfg.height, cfg.width
    shapes = []
    for cls in range(1, c):
        if cfg.blobs and cls == c - 1:
            for _ in range(4):
                cy, cx = int(rng.integers(0, h)), int(rng.integers(0, w))
                ry, rx = max(1, h // 10), max(1, w // 10)
                shapes.append((1, cls, cy, cx, ry, rx))
            continue
        rh, rw = max(1, int(0.16 * h)), max(1, int(0.16 * w))
        for _ in range(4):
            y0 = int(rng.integers(0, h - rh + 1))
            x0 = int(rng.integers(0, w - rw + 1))
            shapes.append((0, cls, y0, x0, y0 + rh, x0 + rw))
    shapes = np.array(shapes, dtype=np.int64).reshape(-1, 6)
    xs, ys, labels = _training_points(cfg, shapes, rng)
    return Scene(cfg, means, chol, shapes, xs, ys, labels)


def _training_points(cfg: Config, shapes, rng):
    if cfg.per_class <= 0:
        z = np.zeros(0, dtype=np.int64)
        return z, z, z
    xs, ys, labels = [], [], []
    npix = cfg.pixels
    for cls in range(cfg.classes):
        picked: list[int] = []
        seen: set[int] = set()
        tries = 0
        while len(picked) < cfg.per_class:
            cand = rng.integers(0, npix, size=max(4 * cfg.per_class, 1024))
            ok = class_map_at(shapes, cand // cfg.width, cand % cfg.width) == cls
            for p in cand[ok].tolist():
                if p not in seen:
                    seen.add(p)
                    picked.append(p)
                    if len(picked) == cfg.per_class:
                        break
            tries += 1
            if tries > 1000:
                raise RuntimeError(f"class {cls} too small for {cfg.per_class} points")
        arr = np.array(picked, dtype=np.int64)
        ys.append(arr // cfg.width)
        xs.append(arr % cfg.width)
        labels.append(np.full(len(arr), cls, dtype=np.int64))
    return np.concatenate(xs), np.concatenate(ys), np.concatenate(labels)


def generate(scene: Scene, device=None, row0: int = 0, rows: int | None = None) -> DeviceStack:
    """Generate rows [row0, row0+rows) of the scene's cube in HBM."""
    cfg = scene.cfg
    device = device or dev.require_cuda()
    rows = cfg.height - row0 if rows is None else rows
    with torch.cuda.device(device):
        planes = torch.empty((cfg.bands, rows, cfg.width), dtype=cfg.dtype, device=device)
        means = dev.to_device(scene.means.astype(np.float64), device)
        chol = dev.to_device(scene.chol.astype(np.float64), device)
        shp = np.ascontiguousarray(scene.shapes, dtype=np.int64)
        cube = dev.cube_desc(planes, row0)
        _lib.check(_lib.lib().ut_synth_cube(
            C.byref(cube), cfg.height, means.data_ptr(), chol.data_ptr(), cfg.classes,
            shp.ctypes.data_as(C.c_void_p), len(shp), C.c_uint64(cfg.seed * 0x9E3779B1 + 17),
            dev.stream_handle()), "ut_synth_cube")
    depth = 16 if cfg.dtype == torch.uint16 else 8
    return DeviceStack(default_bands(cfg.bands), planes, depth, True, row0, cfg.height)
