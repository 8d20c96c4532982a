"""Device-resident fused CVA / PCA pipelines (the measured hot path).

One ``run()`` enqueues the whole path on the current stream with no host
synchronization:

  CVA:  K1 gather -> K1 class moments -> [all_gather] -> K3 cva_solve
        -> K4 project+min/max -> [all_reduce MAX] -> K5 stretch
  PCA:  K2 region moments -> [all_gather] -> K3 pca_solve
        -> K4 project+min/max -> [all_reduce MAX] -> K5 stretch

Row sharding: each rank holds rows [row0, row0+rows) of the
cube; training points are routed to the rank owning their row; the only data
exchanged are the per-class moment records (all_gather, then a fixed
rank-order combine inside the K3 kernel -- deterministic for a given world
size) and the 2K min/max record (all_reduce MAX).  Errors found on the device
(bad point, non-PD scatter, NaN scores) are read back by ``check()``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import device as dev
from .annotations import check_points
from .eigen import DEFAULT_RIDGE, raise_for_info
from .errors import DataError, NumericError
from .projection import (CvaDevice, PcaDevice, ProjectionModel, METHOD_CVA,
                         METHOD_PCA_UNSUPERVISED, class_index, project_device, _top_k)
from .rendering import (CompositeRecipe, RenderSpec, _zeros_warning, compose_rgb, rescale,
                        stretch_planes)
from .stack import DeviceStack, on_device


def row_bounds(height: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block of ``rank``: [rank*H/G, (rank+1)*H/G)."""
    return (height * rank) // world, (height * (rank + 1)) // world


def route_points(ys, row0: int, rows: int) -> np.ndarray:
    """Indices (in original order) of the training points owned by a shard."""
    ys = np.asarray(ys)
    return np.flatnonzero((ys >= row0) & (ys < row0 + rows))


class _Sharded:
    """Exchange steps of a row-sharded pipeline: through ``comm`` (the library's
    NCCL collectives, comm.py) when given, else torch.distributed on ``group``."""

    def __init__(self, group, comm=None):
        self.group, self.comm = group, comm
        if comm is not None:
            self.world = comm.world
        else:
            self.world = dist.get_world_size(group) if group is not None else 1
        self.graph = None

    def capture(self):
        """Record run() as a CUDA graph: the path is a handful of short kernels at
        small sizes, so launch overhead matters.  Sharded pipelines capture too when
        their exchanges go through a ``Comm`` (NCCL collectives on the same stream);
        torch.distributed collectives (gloo) cannot be captured.  Call after one
        eager run (it sets up workspaces and kernel attributes)."""
        if self.world > 1 and self.comm is None:
            raise RuntimeError("graph capture of a sharded pipeline needs a Comm "
                               "(NCCL collectives through the library)")
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.run()  # warm the side stream's workspaces
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            self.run()
        torch.cuda.synchronize()
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()
        return self.codes

    def gather_moments(self, fit):
        if self.comm is not None:
            self.comm.allgather_f64(fit.local_moments(), fit.moments)
        elif self.world > 1:
            dist.all_gather_into_tensor(fit.moments, fit.local_moments(), group=self.group)

    def reduce_minmax(self, minmax):
        if self.comm is not None:
            self.comm.allreduce(minmax, "max")
        elif self.world > 1:
            dist.all_reduce(minmax, op=dist.ReduceOp.MAX, group=self.group)


class CvaPipeline(_Sharded):
    """CVA fit + projection + stretch of one (shard of a) device cube."""

    def __init__(self, stack: DeviceStack, xs, ys, labels, k: int | None = None,
                 ridge: float = DEFAULT_RIDGE, precision: str | None = None, depth: int = 8,
                 group=None, comm=None):
        super().__init__(group, comm)
        if not stack.normalized:
            raise DataError("assemble_matrix requires a normalized stack")
        self.ds = stack
        self.device = stack.planes.device
        xs, ys, labels = (np.asarray(a) for a in (xs, ys, labels))
        if len(xs) == 0:
            raise DataError("training set has no points")
        check_points(xs, ys, stack.width, 0, stack.full_height)
        self.class_ids, cls = class_index(labels)
        if len(self.class_ids) < 2:
            raise DataError(f"scatter needs at least 2 classes with points, got {len(self.class_ids)}")
        self.k = _top_k(k, stack.band_count)
        self.ridge, self.precision, self.depth = float(ridge), precision, depth
        own = route_points(ys, stack.row0, stack.height) if self.world > 1 else np.arange(len(xs))
        # K1 visits the points grouped by class and, within a class, in raster
        # order: class runs keep its Gram loop branch-free and row order keeps
        # the random gather TLB-/sector-friendly (the sums' order is fixed by
        # this permutation, so results stay deterministic)
        own = own[np.lexsort((xs[own], ys[own], cls[own]))]
        self.own = own            # K1 order -> caller's point index (error reports)
        self.n = len(own)
        b = stack.band_count
        with torch.cuda.device(self.device):
            xy = np.stack([xs[own], ys[own]], axis=1).astype(np.int32) if self.n else \
                np.zeros((1, 2), np.int32)
            self.xy = dev.to_device(xy, self.device)
            self.cls = dev.to_device(cls[own] if self.n else np.zeros(1, np.int32), self.device)
            # first local point of each class: the per-class shift of K1
            piv = np.full(len(self.class_ids), -1, dtype=np.int32)
            if self.n:
                local = cls[own]
                for c in range(len(self.class_ids)):
                    hit = np.flatnonzero(local == c)
                    if len(hit):
                        piv[c] = hit[0]
            self.pivots = dev.to_device(piv, self.device)
            self.fit = CvaDevice(b, len(self.class_ids), self.device, groups=self.world)
            self.cube = stack.cube()
            self.first_bad = torch.full((1,), -1, dtype=torch.int64, device=self.device)
            self.scores = torch.empty((self.k, stack.height, stack.width), dtype=torch.float32,
                                      device=self.device)
            self.minmax = torch.empty(2 * self.k, dtype=torch.float32, device=self.device)
            self.nonfinite = torch.zeros(1, dtype=torch.int32, device=self.device)
            self.codes = torch.empty((self.k, stack.height, stack.width),
                                     dtype=torch.uint8 if depth == 8 else torch.uint16,
                                     device=self.device)
            self.evecs = self.fit.views["evecs"].view(b, b)
            self.mean = self.fit.views["grand_mean"]

    @staticmethod
    def training_arrays(xs, ys, labels, class_ids=None):
        """Host-side K1 inputs for an unsharded pipeline: (xy int32 [n,2],
        class index int32 [n], first point of each class int32 [C]) in K1's
        class-then-raster order -- precomputed per folio by streaming callers."""
        xs, ys, labels = (np.asarray(a) for a in (xs, ys, labels))
        ids, cls = class_index(labels) if class_ids is None else \
            (class_ids, np.searchsorted(np.asarray(class_ids), labels).astype(np.int32))
        order = np.lexsort((xs, ys, cls))
        xy = np.stack([xs[order], ys[order]], axis=1).astype(np.int32)
        cls = cls[order].astype(np.int32)
        piv = np.full(len(ids), -1, dtype=np.int32)
        for c in range(len(ids)):
            hit = np.flatnonzero(cls == c)
            if len(hit):
                piv[c] = hit[0]
        return xy, cls, piv

    def load_training(self, xy: torch.Tensor, cls: torch.Tensor, pivots: torch.Tensor):
        """Swap in another training set of the same size (non-blocking copies on
        the current stream, e.g. from pinned host tensors): streaming folios."""
        if tuple(xy.shape) != tuple(self.xy.shape) or len(pivots) != len(self.pivots):
            raise DataError(f"training set shape {tuple(xy.shape)}/{len(pivots)} classes does "
                            f"not match the pipeline's {tuple(self.xy.shape)}/{len(self.pivots)}")
        self.xy.copy_(xy, non_blocking=True)
        self.cls.copy_(cls, non_blocking=True)
        self.pivots.copy_(pivots, non_blocking=True)
        self.own = None           # the swapped-in set is already in K1 order

    # -- the hot path -------------------------------------------------------
    def fit_only(self):
        self.fit.moments_from_cube(self.cube, self.xy, self.cls, self.n, self.first_bad,
                                   self.pivots)
        self.gather_moments(self.fit)
        self.fit.solve(self.ridge, self.k)

    def project_kernel(self):
        project_device(self.ds, self.evecs, self.mean, None, range(self.k), self.precision,
                       self.scores, self.minmax, self.nonfinite)

    def project_only(self):
        self.project_kernel()
        self.reduce_minmax(self.minmax)

    def stretch_only(self):
        stretch_planes(self.scores, self.minmax, self.depth, out=self.codes)

    def run(self):
        with torch.cuda.device(self.device):
            self.fit_only()
            self.project_only()
            self.stretch_only()
        return self.codes

    # -- results ------------------------------------------------------------
    def bad_point_message(self, k1_index: int) -> str:
        """A K1-order point index (first_bad) in the caller's terms."""
        x, y = (int(v) for v in self.xy[k1_index].cpu())
        if self.own is not None and k1_index < len(self.own):
            return f"training point {int(self.own[k1_index])} at ({x}, {y}) outside the stack"
        return f"training point at ({x}, {y}) outside the stack"

    def check(self):
        """Synchronize and raise the reference's errors for device-side failures."""
        bad = int(self.first_bad.item())
        if bad >= 0:
            raise DataError(self.bad_point_message(bad))
        h = self.fit.host()
        raise_for_info(h["info"], h["aux"])
        if int(self.nonfinite.item()):
            raise DataError("score plane contains NaN or Inf")
        return h

    def model(self) -> ProjectionModel:
        h = self.check()
        return ProjectionModel(method=METHOD_CVA, mean=h["grand_mean"], std=None,
                               coefficients=np.ascontiguousarray(h["evecs"][:, :self.k]),
                               eigenvalues=np.ascontiguousarray(h["evals"][:self.k]))

    def launches(self) -> int:
        """Our kernels per run(): moments + merge, solve, K4 groups, stretch."""
        return (2 if self.n else 0) + 1 + (self.k + 7) // 8 + 1


class PcaPipeline(_Sharded):
    """Unsupervised PCA fit + projection + stretch of one (shard of a) device cube."""

    def __init__(self, stack: DeviceStack, k: int | None = None, precision: str | None = None,
                 depth: int = 8, group=None, comm=None):
        super().__init__(group, comm)
        self.ds = stack
        self.device = stack.planes.device
        self.k = _top_k(k, stack.band_count)
        if stack.full_height * stack.width < 2:
            raise DataError("unsupervised PCA needs at least 2 pixels")
        self.precision, self.depth = precision, depth
        b = stack.band_count
        with torch.cuda.device(self.device):
            self.fit = PcaDevice(b, self.device, groups=self.world)
            self.scores = torch.empty((self.k, stack.height, stack.width), dtype=torch.float32,
                                      device=self.device)
            self.minmax = torch.empty(2 * self.k, dtype=torch.float32, device=self.device)
            self.nonfinite = torch.zeros(1, dtype=torch.int32, device=self.device)
            self.codes = torch.empty((self.k, stack.height, stack.width),
                                     dtype=torch.uint8 if depth == 8 else torch.uint16,
                                     device=self.device)
            self.evecs = self.fit.views["evecs"].view(b, b)

    def fit_only(self):
        if self.ds.height:
            self.fit.moments_from(self.ds.cube(), 0, 0, self.ds.width, self.ds.height, self.device)
        else:
            self.fit.local_moments().zero_()
        self.gather_moments(self.fit)
        self.fit.solve()

    def project_kernel(self):
        project_device(self.ds, self.evecs, self.fit.views["mean"], self.fit.views["std"],
                       range(self.k), self.precision, self.scores, self.minmax, self.nonfinite)

    def project_only(self):
        self.project_kernel()
        self.reduce_minmax(self.minmax)

    def stretch_only(self):
        stretch_planes(self.scores, self.minmax, self.depth, out=self.codes)

    def run(self):
        with torch.cuda.device(self.device):
            self.fit_only()
            self.project_only()
            self.stretch_only()
        return self.codes

    def check(self):
        h = self.fit.host()
        raise_for_info(h["info"], None)
        if int(self.nonfinite.item()):
            raise DataError("score plane contains NaN or Inf")
        return h

    def model(self) -> ProjectionModel:
        h = self.check()
        return ProjectionModel(method=METHOD_PCA_UNSUPERVISED, mean=h["mean"], std=h["std"],
                               coefficients=np.ascontiguousarray(h["evecs"][:, :self.k]),
                               eigenvalues=np.ascontiguousarray(h["evals"][:self.k]))

    def launches(self) -> int:
        """shift + region moments + merge, solve, K4 groups, stretch."""
        return 3 + 1 + (self.k + 7) // 8 + 1


class FolioStream:
    """A batch of independent folios (each its own cube and training set, same
    shape) streamed through CVA on one GPU: the next folio's cube and training
    set are copied host->HBM on a copy stream while the current one is fitted,
    projected and stretched; its codes are copied back to the host.  Two device
    buffers ping-pong.  Host tensors should be pinned for the copies to overlap.

    cubes: list of host (B, H, W) tensors; training: list of
    CvaPipeline.training_arrays() tuples as host tensors; outs: list of host
    (k, H, W) code tensors the results land in."""

    def __init__(self, cubes, training, outs, k: int, precision: str | None = None,
                 depth: int = 8, device=None):
        from .stack import default_bands

        if not cubes:
            raise DataError("no folios")
        self.cubes, self.training, self.outs = cubes, training, outs
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        shape = tuple(cubes[0].shape)
        if any(tuple(c.shape) != shape or c.dtype != cubes[0].dtype for c in cubes):
            raise DataError("all folios of a stream must share shape and sample type")
        # every folio's points are validated here, on the host: K1 drops an
        # out-of-range point (flagging it), and a later folio would overwrite the flag
        for i, tr in enumerate(training):
            xy = np.asarray(tr[0].cpu() if torch.is_tensor(tr[0]) else tr[0])
            if xy.ndim != 2 or xy.shape[1] != 2:
                raise DataError(f"folio {i}: training xy must be (n, 2), got {xy.shape}")
            try:
                check_points(xy[:, 0], xy[:, 1], shape[2], 0, shape[1])
            except DataError as exc:
                raise DataError(f"folio {i}: {exc}") from None
        self.bufs, self.pipes = [], []
        xy0, cls0, _ = (t.numpy() for t in training[0])
        for _ in range(2):
            planes = torch.empty(shape, dtype=cubes[0].dtype, device=self.device)
            ds = DeviceStack(default_bands(shape[0]), planes, depth, True)
            # placeholder labels with the same classes; load_training swaps in each folio's
            self.bufs.append(ds)
            self.pipes.append(CvaPipeline(ds, xy0[:, 0], xy0[:, 1], cls0, k=k,
                                          precision=precision, depth=depth))
        self.copy_stream = torch.cuda.Stream(self.device)
        # per-folio device status, copied out of the pipeline after each folio
        # (each run resets first_bad / info / nonfinite): [first_bad, info, nonfinite]
        b = shape[0]
        self.status = torch.zeros((len(cubes), 3), dtype=torch.int64, device=self.device)
        self.aux = torch.zeros((len(cubes), b), dtype=torch.float64, device=self.device)

    def launches(self) -> int:
        return self.pipes[0].launches() * len(self.cubes)

    def run(self):
        """Enqueue the whole batch on the current stream (+ the copy stream)."""
        comp = torch.cuda.current_stream(self.device)
        done = [None, None]
        for i in range(len(self.cubes)):
            j = i % 2
            ready = torch.cuda.Event()
            with torch.cuda.stream(self.copy_stream):
                if done[j] is not None:
                    self.copy_stream.wait_event(done[j])
                self.bufs[j].planes.copy_(self.cubes[i], non_blocking=True)
                self.pipes[j].load_training(*self.training[i])
                ready.record(self.copy_stream)
            comp.wait_event(ready)
            p = self.pipes[j]
            p.run()
            self.outs[i].copy_(p.codes, non_blocking=True)
            self.status[i, 0:1].copy_(p.first_bad)
            self.status[i, 1:2].copy_(p.fit.info)
            self.status[i, 2:3].copy_(p.nonfinite)
            self.aux[i].copy_(p.fit.views["aux"])
            done[j] = torch.cuda.Event()
            done[j].record(comp)
        # the copy stream must not run ahead into buffers the caller reuses
        self.copy_stream.wait_stream(comp)

    def check(self):
        """Raise the first failing folio's error (with its index)."""
        status = self.status.cpu().numpy()
        for i, (bad, info, nonfinite) in enumerate(status):
            try:
                if bad >= 0 and self.training[i][0].shape[0] > int(bad):
                    x, y = (int(v) for v in self.training[i][0][int(bad)])
                    raise DataError(f"training point at ({x}, {y}) outside the stack")
                raise_for_info(int(info), self.aux[i].cpu().numpy())
                if nonfinite:
                    raise DataError("score plane contains NaN or Inf")
            except (DataError, NumericError) as exc:
                raise type(exc)(f"folio {i}: {exc}") from None


# ------------------------------------------------------------ render_planes
# Components projected per K4 pass: up to 32 (the kernel's limit, one cube read
# for all of them) when their fp32 score planes and codes fit in half the free
# HBM; fewer otherwise.  The reference batches 8 planes at a time to bound host
# memory (pipeline.py:44), re-reading the cube once per batch.
_RENDER_BATCH = 32
_ENCODES_IN_FLIGHT = 4   # planes encoding on the device while earlier files are written
_WRITERS = 4             # host threads waiting on finished encodes and writing files


def _render_batch(ds, n_specs: int, depth_bytes: int = 2) -> int:
    npix = ds.height * ds.width
    per_component = npix * (4 + n_specs * depth_bytes)
    free, _ = torch.cuda.mem_get_info(ds.planes.device)
    return int(max(1, min(_RENDER_BATCH, (free // 2) // max(per_component, 1))))


@dataclass
class RenderResult:
    """Artifact paths written by render_planes, in deterministic order
    (pipeline.py:120-125)."""

    plane_paths: list[Path] = field(default_factory=list)
    composite_path: Path | None = None


def plane_filename(run_name: str, k: int, spec: RenderSpec, fmt: str) -> str:
    return f"{run_name}_plane{k:02d}{spec.suffix()}.{fmt}"


def composite_filename(run_name: str, recipe: CompositeRecipe) -> str:
    return f"{run_name}{recipe.suffix()}.png"


def render_planes(stack, model: ProjectionModel, specs: list[RenderSpec], out_dir,
                  run_name: str = "run", components: list[int] | None = None,
                  recipe: CompositeRecipe | None = None, workers: int = 1, fmt: str = "png",
                  compression: str = "none") -> RenderResult:
    """Project, rescale per spec, and write one grayscale image per plane per
    spec, plus the optional composite (pipeline.py:136-190), entirely on the
    device: one K4 pass projects every requested component (score planes stay
    in HBM), each spec renders codes on the device (full range from the
    projector's min/max, training range, percentile select), compose_rgb
    interleaves the recipe's planes, and the PNG / TIFF bytes are encoded on
    the device; the host writes finished files -- a few encodes stay in flight
    and a small thread pool writes finished files while the next planes encode.
    Same files, names and order as the reference; ``workers`` is accepted for
    signature compatibility."""
    from collections import deque
    from concurrent.futures import ThreadPoolExecutor

    from .image_io import save_image, save_image_start
    from .projection import project_stack

    if fmt not in ("png", "tif"):
        raise DataError(f"format must be png or tif, got {fmt!r}")
    if not specs:
        raise DataError("at least one render spec required")
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    if components is None:
        components = list(range(model.component_count))
    ds = on_device(stack)
    result = RenderResult()
    needed = set() if recipe is None else {recipe.red, recipe.green, recipe.blue}
    recipe_planes: dict = {}
    step = _render_batch(ds, len(specs))
    inflight: deque = deque()     # encodes enqueued on the device, oldest first
    writes = []
    with ThreadPoolExecutor(max_workers=_WRITERS) as pool:
        for i in range(0, len(components), step):
            batch = components[i:i + step]
            planes = project_stack(ds, model, components=batch, workers=workers)
            ranges = planes[0].minmax.cpu().numpy()   # [-min_0.., max_0..] of the batch
            nb = len(batch)
            for j, (k, plane) in enumerate(zip(batch, planes)):
                for s_i, spec in enumerate(specs):
                    if spec.mode == "full" and -ranges[j] == ranges[nb + j]:
                        _zeros_warning("constant score plane")   # rendering.py:128-129
                    img = rescale(plane, spec, model=model, k=k)
                    path = out_dir / plane_filename(run_name, k, spec, fmt)
                    inflight.append(save_image_start(img, path, compression=compression))
                    if len(inflight) > _ENCODES_IN_FLIGHT:
                        writes.append(pool.submit(inflight.popleft()))
                    result.plane_paths.append(path)
                    if s_i == 0 and k in needed:
                        recipe_planes[k] = img
        while inflight:
            writes.append(pool.submit(inflight.popleft()))
        for w in writes:
            w.result()            # re-raises a writer's DataError
    if recipe is not None:
        missing = sorted(needed - set(recipe_planes))
        if missing:
            raise DataError(f"recipe needs planes {missing}, not rendered")
        trio = [recipe_planes[recipe.red], recipe_planes[recipe.green], recipe_planes[recipe.blue]]
        composite = compose_rgb(trio, CompositeRecipe(0, 1, 2, swap=recipe.swap))
        path = out_dir / composite_filename(run_name, recipe)
        save_image(composite, path)
        result.composite_path = path
    return result


# ------------------------------------------------- staged entry points
# The composed stages the reference's CLI and service call (pipeline.py:56-117,
# :193-199), on the device path.

def load_normalized(manifest, crop_rect: tuple[int, int, int, int] | None = None,
                    scope: str = "per-band"):
    """Manifest -> loaded (device decode), optionally cropped, normalized stack
    (pipeline.py:56-65).  Returns a DeviceStack: the cube stays in HBM for the
    fit and projection that follow."""
    from .stack import crop, load_device_stack, normalize_stack

    stack = load_device_stack(manifest)
    if crop_rect is not None:
        stack = crop(stack, *crop_rect)
    return normalize_stack(stack, scope)


def model_provenance(stack_meta: dict, annotations_text: str | None, method: str,
                     k: int | None, ridge: float) -> dict:
    """The provenance dict embedded in a model file, in the reference's key
    order (pipeline.py:68-93)."""
    import hashlib

    prov = {key: stack_meta[key] for key in ("manifest", "manifest_sha256", "crop", "scope")
            if key in stack_meta}
    if annotations_text is not None:
        prov["annotations_sha256"] = hashlib.sha256(annotations_text.encode("utf-8")).hexdigest()
    prov["method"] = method
    prov["k"] = k if k is not None else "all"
    prov["ridge"] = ridge
    return prov


def fit_model(stack, training, method: str, k: int | None = None, ridge: float = DEFAULT_RIDGE,
              region: tuple[int, int, int, int] | None = None,
              provenance: dict | None = None) -> ProjectionModel:
    """Fit any method against a normalized stack (pipeline.py:96-117):
    supervised methods sample the stack at the training points (device
    gather), the unsupervised PCA uses every pixel of ``region``."""
    from .annotations import assemble_matrix
    from .projection import METHOD_PCA_UNSUPERVISED, fit

    provenance = dict(provenance or {})
    provenance.setdefault("normalized_input", stack.normalized)
    if method == METHOD_PCA_UNSUPERVISED:
        return fit(method, stack=stack, region=region, k=k, provenance=provenance)
    if training is None:
        raise DataError(f"method {method!r} needs annotations")
    dm = assemble_matrix(stack, training)
    return fit(method, dm=dm, k=k, ridge=ridge, provenance=provenance)


def project_single(stack, model: ProjectionModel, k: int, workers: int = 1):
    """One component's score plane (pipeline.py:193-199)."""
    from .projection import project_stack

    return project_stack(stack, model, components=[k], workers=workers)[0]
