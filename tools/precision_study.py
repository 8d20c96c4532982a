"""Projector precision study: fp32 vs fp64 score planes against the oracle.

For each BASELINE generator config (scaled where the oracle would be slow),
fit the model on the device, project with both precisions and compare with the
oracle's float64 projection of the same cube and model (the reference's
_project_rows arithmetic).  Reports the worst |delta| / (max - min) per config
and the uint8 disagreement count; writes profiles/<round>/precision.json.

    python tools/precision_study.py [--out profiles/r1/precision.json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402
from paper_1612_06457_b200.projection import project_device  # noqa: E402
from paper_1612_06457_b200.rendering import stretch_planes  # noqa: E402

CASES = [
    ("cfg1", 512, 512, None),
    ("cfg2", 1024, 1024, None),
    ("cfg3", 1804, 1353, 2000),
    ("cfg4", 2048, 2048, 10000),
    ("cfg4pca", 1024, 1024, None),
    ("cfg5", 1024, 768, 1000),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r1" / "precision.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    report = {}
    for name, h, w, per in CASES:
        cfg = synthetic.scaled(synthetic.CONFIGS[name], h, w, per)
        scene = synthetic.make_scene(cfg)
        stack = synthetic.generate(scene)
        cube = stack.planes.cpu().numpy()
        if cfg.method == "cva":
            pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
        else:
            pipe = ut.PcaPipeline(stack, k=cfg.k)
        pipe.run()
        model = pipe.model()
        ref = oracle.project(cube, {"mean": model.mean, "std": model.std,
                                    "coefficients": model.coefficients}, workers=8)
        ref_codes = np.stack([oracle.rescale_full(p) for p in ref])
        row = {"pixels": cfg.pixels, "bands": cfg.bands, "k": cfg.k, "dtype": str(cfg.dtype)}
        for prec in ("fp32", "fp64"):
            mean = pipe.mean if cfg.method == "cva" else pipe.fit.views["mean"]
            std = None if cfg.method == "cva" else pipe.fit.views["std"]
            scores, mm, _ = project_device(stack, pipe.evecs, mean, std, range(cfg.k), prec)
            codes = stretch_planes(scores, mm).cpu().numpy()
            got = scores.double().cpu().numpy()
            err = max(float(np.abs(got[j] - ref[j]).max() / (ref[j].max() - ref[j].min()))
                      for j in range(cfg.k))
            diff = np.abs(codes.astype(int) - ref_codes.astype(int))
            row[prec] = {"max_err_over_range": err, "u8_max_diff": int(diff.max()),
                         "u8_pixels_differing": int((diff > 0).sum())}
        report[cfg.name] = row
        print(cfg.name, json.dumps(row), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(report, indent=1) + "\n")


if __name__ == "__main__":
    main()
