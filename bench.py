#!/usr/bin/env python
"""Benchmark of the CVA hot path (BASELINE.json metric: CVA Mpixel/s,
scatter + eigen + projection, at 1/2/4/8 B200, and % of HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
  python bench.py --impl reference ...     # the reference algorithm on host cores

A step is one full pass of the hot path over the synthetic cube already in
HBM: K1 gather + class moments -> K3 scatter/eigen -> K4 projection + min/max
-> K5 uint8 stretch (for N > 1 plus the moment all_gather and the min/max
all_reduce over NCCL).  Rank 0 prints one JSON line.  See DESIGN.md §7.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def hbm_peak():
    try:
        doc = json.loads(PEAKS_FILE.read_text())
        return float(doc["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback 6.65 TB/s (B200_PROFILING.md)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--rows", type=int, default=None, help="override image height (profiling)")
    ap.add_argument("--precision", default=None, choices=[None, "fp32", "fp64"])
    ap.add_argument("--e2e-steps", type=int, default=7)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stream-e2e", action="store_true", help="serial e2e only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-pca", action="store_true",
                    help="skip the PCA companion measurement on the same cube")
    ap.add_argument("--folios", type=int, default=64, help="cfg5: folios in the batch")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU work for the cpu_baseline sample")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="seconds for the whole --impl reference run")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/ut_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3]) if v.lower() == "active"})
        loaded = [r for r in rows if r[2] > 250.0] or rows
        return {"sm_mhz": float(np.median([r[0] for r in loaded])),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(r[2] for r in rows)}


# ------------------------------------------------------------------ helpers

def dist_setup(n):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # UT_BENCH_BACKEND=gloo (with ranks sharing the GPUs there are) is the
        # functional check of this multi-rank path on a one-GPU box; timing
        # runs use NCCL, one GPU per rank
        backend = os.environ.get("UT_BENCH_BACKEND", "nccl")
        dev_id = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
        torch.cuda.set_device(dev_id)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_id))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def pipe_precision(args):
    from paper_1612_06457_b200 import projection

    return args.precision or projection.PRECISION


def cfg_of(args):
    from paper_1612_06457_b200 import synthetic

    cfg = synthetic.CONFIGS[args.config]
    if args.rows:
        cfg = synthetic.scaled(cfg, args.rows, cfg.width)
    return cfg


def host_cube(stack):
    """Pinned host copy of the device cube (setup; used by e2e and the CPU arms)."""
    import torch

    host = torch.empty(stack.planes.shape, dtype=stack.planes.dtype, pin_memory=True)
    host.copy_(stack.planes)
    return host


def cpu_reference(sample, train_values, scene, cfg, workers):
    """One bounded sample of the workload through the oracle port of the
    reference: fit_cva on the full training matrix (B x N, already gathered),
    then project + rescale_full of the ``sample`` rows (B, rows, W).  PCA fits
    on the sample rows (its covariance is a per-pixel pass).  Returns
    (seconds, pixels)."""
    import oracle

    t0 = time.perf_counter()
    if cfg.method == "cva":
        model = oracle.fit_cva(train_values, scene.labels, k=cfg.k)
    else:
        model = oracle.fit_pca_unsupervised(sample, k=cfg.k)
    scores = oracle.project(sample, model, workers=workers)
    _ = [oracle.rescale_full(s) for s in scores]
    return time.perf_counter() - t0, sample.shape[1] * sample.shape[2]


def cpu_threads():
    n = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_info

        blas = max((i.get("num_threads", 0) for i in threadpool_info()), default=n)
    except Exception:
        blas = n
    return n, blas


def pick_rows(probe_sample, train_values, scene, cfg, workers, seconds):
    """Rows so that one sample step takes about ``seconds`` of CPU time."""
    t, px = cpu_reference(probe_sample, train_values, scene, cfg, workers)
    t_fit, _ = cpu_reference(probe_sample[:, :2], train_values, scene, cfg, workers)
    per_row = max((t - t_fit) / probe_sample.shape[1], 1e-6)
    return int(max(16, min(cfg.height, (seconds - t_fit) / per_row)))


def bench_config(cfg, world, args, n_train):
    """The ``config`` object of the JSON line -- identical for both arms."""
    cube_bytes = cfg.pixels * cfg.bands * cfg.sample_bytes // max(world, 1)
    use_graph = world == 1 and cfg.pixels <= (1 << 24) and not args.no_graph
    return {"workload": cfg.name, "height": cfg.height, "width": cfg.width,
            "bands": cfg.bands, "sample": str(cfg.dtype).replace("torch.", ""),
            "classes": cfg.classes, "training_px": int(n_train), "components": cfg.k,
            "parallelism": f"rows{world}",
            "l2": "inputs > L2 (cube %.1f GB per GPU)" % (cube_bytes / 1e9)
                  if cube_bytes > 126e6 else
                  "cube fits L2 (%.1f MB); no flush: a repeated step re-reads the same "
                  "cube, as a resident-data service would" % (cube_bytes / 1e6),
            "cuda_graph": use_graph}


def repo_libs_mapped():
    """In-tree shared objects mapped into this process (the reference arm must
    map none)."""
    try:
        maps = Path("/proc/self/maps").read_text()
    except OSError:
        return []
    return sorted({ln.split()[-1] for ln in maps.splitlines()
                   if str(ROOT) in ln and ln.rstrip().endswith(".so")})


# ------------------------------------------------------------------ arms

def run_reference(args):
    """--impl reference: the reference algorithm (the numpy port in oracle/; the
    reference itself is Python and cannot travel to the box) on this box's
    host cores.  Inputs come from oracle/synth.py, the host restatement of the
    device generator (bit-identical samples), so this arm never maps the
    repo's CUDA library or touches the GPU."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import synth as host_synth
    from paper_1612_06457_b200 import synthetic

    cfg = cfg_of(args)
    scene = synthetic.make_scene(cfg)
    cores, blas = cpu_threads()
    t_gen = time.perf_counter()
    train = host_synth.pixels(scene, scene.ys, scene.xs).astype(np.float64) \
        if cfg.method == "cva" else None
    probe = host_synth.rows(scene, 0, min(cfg.height, 64), procs=cores)
    steps = args.steps + args.warmup
    rows = pick_rows(probe, train, scene, cfg, cores, args.ref_budget / max(steps, 1))
    r0 = (cfg.height - rows) // 2            # a block from the middle of the image
    sample = host_synth.rows(scene, r0, r0 + rows, procs=cores)
    t_gen = time.perf_counter() - t_gen
    times = []
    for i in range(steps):
        t, px = cpu_reference(sample, train, scene, cfg, cores)
        if i >= args.warmup:
            times.append(t)
    sec = float(np.mean(times))
    value = px / sec / 1e6
    libs = repo_libs_mapped()
    if libs:
        raise RuntimeError(f"reference arm mapped repo libraries: {libs}")
    fit = (f"fit_cva on all {len(scene.xs)} training px (gathered during setup)"
           if cfg.method == "cva" else f"PCA fit on the {rows} sampled rows")
    sample_txt = (f"{fit} + project/stretch of rows {r0}..{r0 + rows} of {cfg.height} "
                  f"({px} px) per step; numpy port of the reference (oracle/cva_pca.py), "
                  f"workers={cores}, BLAS threads={blas}; inputs from oracle/synth.py "
                  f"(host restatement of the device generator, {t_gen:.1f} s setup)")
    line = {
        "metric": "CVA Mpixel/s (scatter+eigen+projection)" if cfg.method == "cva"
        else "PCA Mpixel/s (covariance+eigen+projection)",
        "value": round(value, 3), "unit": "Mpixel/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json generator, host restatement; seed %d)" % cfg.seed,
        "config": bench_config(cfg, world, args, len(scene.xs)),
        "cpu_baseline": {"value": round(value, 3), "unit": "Mpixel/s", "cores": cores,
                         "kind": "port", "sample": sample_txt},
        "e2e": {"value": round(value, 3), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "repo_libs_mapped": libs,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_folios(args):
    """cfg 5: a batch of independent folios (distinct seeds and training sets)
    streamed through CVA (FolioStream), round-robin over the ranks (replicas, no
    collective).  Each folio is copied from pinned host memory to HBM on a copy
    stream while the previous one is processed and its uint8 planes are copied
    back, so the aggregate Mpixel/s includes the staging (BASELINE.json cfg 5)."""
    import torch

    import paper_1612_06457_b200 as ut
    from paper_1612_06457_b200 import synthetic
    from dataclasses import replace

    world, rank, local = dist_setup(args.gpus)
    base = cfg_of(args)
    mine = [f for f in range(args.folios) if f % world == rank]
    cubes, train, outs = [], [], []
    for f in mine:  # setup: generate each folio in HBM, keep it in pinned host memory
        sc = synthetic.make_scene(replace(base, seed=base.seed * 1000 + f))
        st = synthetic.generate(sc)
        cubes.append(host_cube(st))
        del st
        arrs = ut.CvaPipeline.training_arrays(sc.xs, sc.ys, sc.labels)
        train.append(tuple(torch.from_numpy(a).pin_memory() for a in arrs))
        outs.append(torch.empty((base.k, base.height, base.width), dtype=torch.uint8,
                                pin_memory=True))
    torch.cuda.empty_cache()
    fs = ut.FolioStream(cubes, train, outs, k=base.k, precision=args.precision)
    for _ in range(max(1, args.warmup // 3)):
        fs.run()
    torch.cuda.synchronize()
    fs.check()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier(world)
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            fs.run()
        stop.record()
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(start.elapsed_time(stop) / args.steps, world)
    px = base.pixels * args.folios
    h2d = sum(c.numel() * c.element_size() + sum(t.numel() * 4 for t in tr)
              for c, tr in zip(cubes, train))
    d2h = sum(o.numel() for o in outs)
    h2d, d2h = (int(max_over_ranks(float(x), world)) * world for x in (h2d, d2h))
    value = px / (ms * 1e-3) / 1e6
    if rank == 0:
        line = {
            "metric": "CVA Mpixel/s incl. H2D staging (folio batch)", "value": round(value, 3),
            "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if pipe_precision(args) == "fp64" else "f32",
            "data": "synthetic (BASELINE.json cfg 5 generator, one seed per folio)",
            "config": {"workload": f"{base.name}x{args.folios}", "folios": args.folios,
                       "parallelism": f"replicas{world}",
                       "staging": "pinned host -> HBM on a copy stream, double-buffered",
                       "l2": "each folio (> L2) is freshly copied in"},
            "e2e": {"value": round(value, 3), "unit": "Mpixel/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "clocks": clocks.summary(),
            "gpu_launches": fs.launches() * world,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def pca_companion(ut, stack, cfg, args, group, world, stream, comm=None):
    import torch

    pipe = ut.PcaPipeline(stack, k=cfg.k, precision=args.precision, group=group, comm=comm)
    for _ in range(3):
        pipe.run()
    torch.cuda.synchronize()
    pipe.check()
    steps = max(3, min(args.steps, 20))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    for e in ev:
        e[0].record(stream)
        pipe.fit_only()
        e[1].record(stream)
        pipe.project_kernel()
        e[2].record(stream)
        pipe.reduce_minmax(pipe.minmax)
        pipe.stretch_only()
        e[3].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    pipe.check()
    ms = max_over_ranks(float(np.mean([e[0].elapsed_time(e[3]) for e in ev])), world)
    fit_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    k4_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    tail_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    per_px = 2 * cfg.bands * cfg.sample_bytes + cfg.k       # PCA 2*B*s + K
    peak, _ = hbm_peak()
    step_gbs = per_px * stack.pixels / (ms * 1e-3) / 1e9
    out = {"metric": "PCA Mpixel/s (covariance+eigen+projection)",
           "workload": cfg.name.replace("_cva_", "_pca_"),
           "value": round(cfg.pixels / (ms * 1e-3) / 1e6, 3), "unit": "Mpixel/s",
           "ms_per_step": round(ms, 4), "steps": steps,
           "split_ms": {"fit": round(fit_ms, 4), "project": round(k4_ms, 4),
                        "minmax+stretch": round(tail_ms, 4)},
           "roofline_step": {"bytes_per_px": per_px, "achieved": round(step_gbs, 1),
                             "frac": round(step_gbs / peak, 4)}}
    del pipe
    torch.cuda.empty_cache()
    return out


def sharded_self_check(ut, synthetic, base, group, comm, world, rank):
    """N > 1, before timing: this run's sharded pipelines and collectives on a
    small cube of the workload's generator vs an unsharded fit of the same cube
    on rank 0.  Models to SURVEY Appendix A (eigenvalues 1e-9 relative, kept
    vectors 1e-6 after sign alignment), uint8 codes of rank 0's rows within 1
    (global min/max through the MAX exchange).  Every rank exits if it fails:
    no number is printed for a wrong multi-GPU result."""
    import torch
    import torch.distributed as dist

    cfg = synthetic.scaled(base, 64 * world, 384, per_class=400)
    scene = synthetic.make_scene(cfg)
    r0, r1 = ut.row_bounds(cfg.height, world, rank)
    shard = synthetic.generate(scene, row0=r0, rows=r1 - r0)
    full = synthetic.generate(scene) if rank == 0 else None
    report, ok_all = {}, True
    for method in ("cva", "pca"):
        def make(st, sharded):
            kw = dict(group=group, comm=comm) if sharded else {}
            if method == "cva":
                return ut.CvaPipeline(st, scene.xs, scene.ys, scene.labels, k=cfg.k, **kw)
            return ut.PcaPipeline(st, k=cfg.k, **kw)

        sp = make(shard, True)
        codes = sp.run()
        torch.cuda.synchronize()
        m = sp.model()
        ok, detail = True, {}
        if rank == 0:
            up = make(full, False)
            want = up.run()
            um = up.model()
            lam = float(np.abs(m.eigenvalues - um.eigenvalues).max() /
                        max(np.abs(um.eigenvalues).max(), 1e-300))
            sign = np.sign(np.sum(m.coefficients * um.coefficients, axis=0))
            vec = float(np.abs(m.coefficients * sign - um.coefficients).max() /
                        max(np.abs(um.coefficients).max(), 1e-300))
            diff = int((codes.int() - want[:, r0:r1].int()).abs().max().item())
            ok = lam <= 1e-9 and vec <= 1e-6 and diff <= 1
            detail = {"eigenvalue_rel": lam, "vector_rel": vec, "codes_max_diff": diff,
                      "ok": bool(ok)}
            del up, want
        flag = torch.tensor([0 if ok else 1], dtype=torch.int32, device="cuda")
        dist.broadcast(flag, src=0, group=group)
        ok_all = ok_all and int(flag.item()) == 0
        report[method] = detail
        del sp, codes
    del shard, full
    torch.cuda.empty_cache()
    report["collectives"] = "ut_comm (NCCL via the C ABI)" if comm is not None else \
        f"torch.distributed ({dist.get_backend(group)})"
    report["cube"] = f"{cfg.height}x{cfg.width}x{cfg.bands}, {world} row shards"
    if not ok_all:
        if rank == 0:
            sys.stderr.write(f"sharded self-check FAILED: {json.dumps(report)}\n")
        raise SystemExit(3)
    return report


def run_b200(args):
    import torch

    import paper_1612_06457_b200 as ut
    from paper_1612_06457_b200 import synthetic

    world, rank, local = dist_setup(args.gpus)
    group = comm = None
    self_check = None
    if world > 1:
        import torch.distributed as dist

        group = dist.group.WORLD
        # the exchange steps go through the library's NCCL collectives (C ABI)
        # unless UT_BENCH_COMM=torch; gloo runs (one-GPU functional checks) use
        # torch.distributed
        if dist.get_backend(group) == "nccl" and os.environ.get("UT_BENCH_COMM", "ut") != "torch":
            from paper_1612_06457_b200.comm import Comm

            comm = Comm.from_group(group)
        self_check = sharded_self_check(ut, synthetic, cfg_of(args), group, comm, world, rank)
    cfg = cfg_of(args)
    scene = synthetic.make_scene(cfg)
    r0, r1 = ut.row_bounds(cfg.height, world, rank)
    stack = synthetic.generate(scene, row0=r0, rows=r1 - r0)
    if cfg.method == "cva":
        pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k,
                              precision=args.precision, group=group, comm=comm)
    else:
        pipe = ut.PcaPipeline(stack, k=cfg.k, precision=args.precision, group=group,
                              comm=comm)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        pipe.run()
    torch.cuda.synchronize()
    pipe.check()
    # launch-bound sizes: replay the whole path as one CUDA graph (1 GPU only)
    use_graph = world == 1 and cfg.pixels <= (1 << 24) and not args.no_graph
    if use_graph:
        pipe.capture()

    # ---- timed region: K full steps, events on the launching stream
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier(world)
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            e = ev[i]
            if use_graph:  # whole step as one graph; per-kernel split from an eager pass
                e[0].record(stream)
                pipe.replay()
                e[3].record(stream)
                continue
            e[0].record(stream)
            pipe.fit_only()
            e[1].record(stream)
            pipe.project_kernel()
            e[2].record(stream)
            pipe.reduce_minmax(pipe.minmax)
            pipe.stretch_only()
            e[3].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    pipe.check()
    total_ms = start.elapsed_time(stop)
    ms_step = max_over_ranks(total_ms / args.steps, world)
    if use_graph:  # split the step with an eager, event-bracketed pass
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(10)]
        for e in ev:
            e[0].record(stream)
            pipe.fit_only()
            e[1].record(stream)
            pipe.project_kernel()
            e[2].record(stream)
            pipe.reduce_minmax(pipe.minmax)
            pipe.stretch_only()
            e[3].record(stream)
        torch.cuda.synchronize()
    k4_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    fit_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    tail_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    k4_ms = max_over_ranks(k4_ms, world)

    pixels = cfg.pixels
    value = pixels / (ms_step * 1e-3) / 1e6
    peak, peak_src = hbm_peak()
    local_px = stack.pixels
    per_px = cfg.bytes_per_pixel()
    # K4's own algorithmic bytes: one read of the cube (B * s per pixel); the
    # K uint8 codes of the step's 133 B/px are written by K5, not K4
    k4_px = cfg.bands * cfg.sample_bytes
    achieved = k4_px * local_px / (k4_ms * 1e-3) / 1e9
    step_achieved = per_px * local_px / (ms_step * 1e-3) / 1e9

    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            doc = json.loads(prof.read_text())
            ent = doc.get(cfg.name.split("@")[0]) or {}
            if "bytes_per_pixel" in ent:
                traffic = round(ent["bytes_per_pixel"] * local_px / 1e9, 3)
        except Exception:
            traffic = None

    # ---- PCA companion (north-star second path): the unsupervised PCA step on
    # the same resident cube (cfg 4's generator, so this is the cfg4pca
    # workload): covariance (K2) + eigen + projection (K4) + stretch (K5)
    pca = None
    if cfg.method == "cva" and not args.no_pca:
        pca = pca_companion(ut, stack, cfg, args, group, world, stream, comm)

    # ---- e2e: host (pinned) cube in, uint8 planes out, through the same API
    e2e = None
    if not args.no_e2e:
        host = host_cube(stack)
        codes_host = torch.empty(pipe.codes.shape, dtype=pipe.codes.dtype, pin_memory=True)
        # the step's inputs: the cube and (CVA) the training set, from pinned host memory
        train = tuple(t.cpu().pin_memory() for t in (pipe.xy, pipe.cls, pipe.pivots)) \
            if cfg.method == "cva" else ()
        h2d = host.numel() * host.element_size() + sum(t.numel() * t.element_size() for t in train)
        d2h = codes_host.numel() * codes_host.element_size()
        times = []
        for i in range(args.e2e_steps + 1):
            barrier(world)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            stack.planes.copy_(host, non_blocking=True)
            if train:
                pipe.load_training(*train)
            pipe.run()
            codes_host.copy_(pipe.codes, non_blocking=True)
            b.record(stream)
            torch.cuda.synchronize()
            if i:
                times.append(a.elapsed_time(b))
        e2e_ms = max_over_ranks(float(np.mean(times)), world)
        e2e = {"value": round(pixels / (e2e_ms * 1e-3) / 1e6, 3), "unit": "Mpixel/s",
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
               "ms_per_step": round(e2e_ms, 3), "mode": "serial: H2D, fit, project, stretch, D2H"}
        pipe.check()
        if world == 1 and cfg.method == "cva" and not args.no_stream_e2e:
            # the same steps through FolioStream: step i+1's cube and training set
            # copy in on a copy stream while step i computes and copies its codes
            # out (PCIe is full duplex); throughput over e2e_steps + 1 back-to-back
            # steps, every step's full H2D and D2H inside the timed region
            import paper_1612_06457_b200 as ut

            nstep = args.e2e_steps + 1
            outs = [codes_host] + [torch.empty_like(codes_host, pin_memory=True)
                                   for _ in range(nstep - 1)]
            fs = ut.FolioStream([host] * nstep, [train] * nstep, outs, k=cfg.k,
                                precision=args.precision)
            fs.run()  # warm-up
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fs.run()
            b.record()
            torch.cuda.synchronize()
            fs.check()
            s_ms = a.elapsed_time(b) / nstep
            if s_ms < e2e_ms:
                e2e = {"value": round(pixels / (s_ms * 1e-3) / 1e6, 3), "unit": "Mpixel/s",
                       "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                       "ms_per_step": round(s_ms, 3),
                       "mode": f"streamed (FolioStream, {nstep} steps back to back, "
                               f"H2D of step i+1 overlaps compute + D2H of step i)",
                       "serial_ms_per_step": round(e2e_ms, 3)}
            del fs
            torch.cuda.empty_cache()
    else:
        host = None

    # ---- CPU baseline (rank 0, N = 1): oracle port on a bounded sample
    cpu = None
    if world == 1 and not args.no_cpu:
        if host is None:
            host = host_cube(stack)
        cube_np = host.numpy()
        cores, blas = cpu_threads()
        train = None
        if cfg.method == "cva":
            import oracle

            train = oracle.assemble(cube_np, scene.xs, scene.ys)
        rows = pick_rows(cube_np[:, :64], train, scene, cfg, cores, args.cpu_seconds)
        t, px = cpu_reference(cube_np[:, :rows], train, scene, cfg, cores)
        cpu = {"value": round(px / t / 1e6, 3), "unit": "Mpixel/s", "cores": cores,
               "kind": "port",
               "sample": (f"fit on all {len(scene.xs)} training px + project/stretch of "
                          f"{rows}/{cfg.height} rows ({px} px), numpy port of the reference "
                          f"(oracle/), workers={cores}, BLAS threads={blas}, {t:.1f} s")}

    if rank == 0:
        launches = pipe.launches() * args.steps
        line = {
            "metric": "CVA Mpixel/s (scatter+eigen+projection)" if cfg.method == "cva"
            else "PCA Mpixel/s (covariance+eigen+projection)",
            "value": round(value, 3), "unit": "Mpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64" if pipe_precision(args) == "fp64" else "f32 (fit f64)",
            "data": "synthetic (BASELINE.json generator, generated in HBM; seed %d)" % cfg.seed,
            "config": bench_config(cfg, world, args, len(scene.xs)),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "kernel": "project_kernel (K4)",
                         "kernel_ms": round(k4_ms, 4), "bytes_per_px": k4_px,
                         "peak_source": peak_src},
            "roofline_step": {"bytes_per_px": per_px, "achieved": round(step_achieved, 1),
                              "frac": round(step_achieved / peak, 4),
                              "split_ms": {"fit": round(fit_ms, 4), "project": round(k4_ms, 4),
                                           "minmax+stretch": round(tail_ms, 4)}},
            "clocks": clocks.summary(),
            "e2e": e2e,
            "pca": pca,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        if self_check is not None:
            line["self_check"] = self_check
        print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "cfg5":
        return run_folios(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
