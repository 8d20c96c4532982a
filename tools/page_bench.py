"""End-to-end page harness: the reference's ``undertext bench`` (cli.py:384-425)
on the device path -- normalize -> fit CVA -> project + render PNG files -- with
the same stages timed for the CPU port of the reference (oracle/ + cv2.imwrite,
the reference's codec) on the same page.

    python tools/page_bench.py [--size 2000x2000] [--bands 23] [--k all] [--cpu]

The page is the BASELINE palimpsest generator (cfg 3 recipe: 12-bit uint16, 4
classes with stains, 2000 training pixels per class) at the requested size,
unnormalized, so the normalize stage has work (the reference bench normalizes
its uint8 page the same way).  Stages are wall-clock with a device sync (they
include file writes).  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def write_bands(raw, band_dir):
    """The page as band files + manifest, as the reference's CLI reads them
    (deflate TIFFs written by cv2 with the reference's save_image parameters)."""
    import cv2

    band_dir.mkdir(parents=True, exist_ok=True)
    planes = raw.planes.cpu().numpy()
    lines = []
    for b in range(planes.shape[0]):
        name = f"band{b:02d}.tif"
        cv2.imwrite(str(band_dir / name), planes[b], [cv2.IMWRITE_TIFF_COMPRESSION, 8])
        lines.append(f"{name},{400 + 20 * b},visible")
    (band_dir / "manifest.txt").write_text("\n".join(lines) + "\n")
    return band_dir / "manifest.txt"


def gpu_arm(cfg, scene, k, depth, fmt, out_dir, reps, manifest=None):
    raw = synthetic.generate(scene)
    raw = ut.DeviceStack(raw.bands, raw.planes, 16, False)
    ts = ut.TrainingSet.from_arrays(scene.xs, scene.ys, scene.labels)
    best = None
    for _ in range(reps):
        stages = {}
        if manifest is not None:
            raw, stages["load"] = timed(lambda: ut.load_device_stack(manifest))
        norm, stages["normalize"] = timed(lambda: ut.normalize_stack(raw))
        model, stages["fit"] = timed(lambda: ut.fit_cva(ut.assemble_matrix(norm, ts), k=k))
        res, stages["project+render"] = timed(lambda: ut.render_planes(
            norm, model, [ut.RenderSpec(out_depth=depth)], out_dir, run_name="gpu", fmt=fmt))
        stages["total"] = sum(stages.values())
        if best is None or stages["total"] < best["total"]:
            best = stages
    sizes = [p.stat().st_size for p in res.plane_paths]
    return best, len(res.plane_paths), int(np.sum(sizes)), raw


def cpu_arm(raw, scene, k, depth, out_dir, workers, manifest=None):
    import cv2

    import oracle

    cube = raw.planes.cpu().numpy()
    stages = {}
    if manifest is not None:   # the reference's load_stack: cv2.imread per band
        t0 = time.perf_counter()
        names = [ln.split(",")[0] for ln in manifest.read_text().splitlines() if ln]
        cube = np.stack([cv2.imread(str(manifest.parent / n), cv2.IMREAD_UNCHANGED)
                         for n in names])
        stages["load"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    codes, _ = oracle.normalize_stack(cube)
    stages["normalize"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    model = oracle.fit_cva(oracle.assemble(codes, scene.xs, scene.ys), scene.labels, k=k)
    stages["fit"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    planes = oracle.project(codes, model, workers=workers)
    sizes = 0
    for j in range(planes.shape[0]):
        img = oracle.rescale_full(planes[j], depth)
        p = out_dir / f"cpu_plane{j:02d}_full.png"
        cv2.imwrite(str(p), img)
        sizes += p.stat().st_size
    stages["project+render"] = time.perf_counter() - t0
    stages["total"] = sum(stages.values())
    return stages, sizes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="2000x2000")
    ap.add_argument("--bands", type=int, default=23)
    ap.add_argument("--k", default="all")
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--format", default="png")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--from-files", action="store_true",
                    help="start from band TIFF files + manifest (load_stack timed)")
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    w, h = (int(v) for v in args.size.lower().split("x"))
    base = synthetic.CONFIGS["cfg3"]
    cfg = replace(base, name=f"page_{w}x{h}x{args.bands}_u16", height=h, width=w,
                  bands=args.bands)
    k = None if args.k == "all" else int(args.k)
    torch.cuda.set_device(0)
    scene = synthetic.make_scene(cfg)
    with tempfile.TemporaryDirectory() as tmp:
        out_dir = Path(tmp)
        manifest = None
        if args.from_files:
            manifest = write_bands(synthetic.generate(scene), out_dir / "bands")
        g, nplanes, gbytes, raw = gpu_arm(cfg, scene, k, args.depth, args.format, out_dir,
                                          args.reps, manifest)
        line = {"workload": cfg.name, "planes": nplanes, "gpu_s": {s: round(v, 4) for s, v in g.items()},
                "gpu_png_bytes": gbytes}
        if args.cpu:
            c, cbytes = cpu_arm(raw, scene, k, args.depth, out_dir, args.workers, manifest)
            line["cpu_s"] = {s: round(v, 4) for s, v in c.items()}
            line["cpu_png_bytes"] = cbytes
            line["cpu"] = f"oracle/ port of the reference + cv2.imwrite, workers={args.workers}"
            line["speedup_total"] = round(c["total"] / g["total"], 1)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
