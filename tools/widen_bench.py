"""Throughput of the §8(f) rows on one GPU (CUDA events, hot), JSON lines:

    python tools/widen_bench.py > profiles/r1/widen.jsonl

* normalize_stack of a raw cfg 3-shaped cube (7216 x 5412 x 23 uint16, 1.80 GB):
  algorithmic bytes = 2 reads of the cube + 1 byte per sample written;
* rescale_percentile on one cfg 4 score plane (16384^2 fp32): algorithmic
  bytes = one read of the plane to find the window + linear_to_codes (read 4 B,
  write 1 B per pixel) = 9 B/px;
* the oracle (numpy, this host) on the same inputs for scale.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1612_06457_b200 as ut  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6455.9) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6455.9
    g = torch.Generator(device="cuda").manual_seed(3)
    raw = torch.randint(0, 4096, (23, 7216, 5412), dtype=torch.int32, device="cuda",
                        generator=g).to(torch.uint16)
    ds = ut.DeviceStack(ut.stack.default_bands(23), raw, 16, False)
    ms = timed(lambda: ut.normalize_stack(ds))
    n = raw.numel()
    gb = (2 * 2 * n + n) / 1e9
    line = {"row": "normalize_stack", "workload": "7216x5412x23 u16 raw, per-band",
            "ms": round(ms, 3), "GB/s": round(gb / ms * 1e3, 1), "roofline_frac": round(gb / ms * 1e3 / peak, 3),
            "algorithmic_bytes": int(gb * 1e9)}
    sub = raw[:, :512].cpu().numpy()
    import oracle
    t0 = time.perf_counter()
    oracle.normalize_stack(sub)
    cpu = time.perf_counter() - t0
    line["oracle_ms_full_cube_est"] = round(cpu * 1e3 * 7216 / 512, 1)
    print(json.dumps(line), flush=True)
    del raw, ds
    torch.cuda.empty_cache()

    plane = torch.randn((16384, 16384), dtype=torch.float32, device="cuda", generator=g)
    mm = torch.stack([-plane.min(), plane.max()]).float()
    dp = ut.DeviceScorePlane(plane[None], mm, 0)
    ms = timed(lambda: ut.rescale_percentile(dp, 1.0))
    n = plane.numel()
    gb = (4 * n + 5 * n) / 1e9
    print(json.dumps({"row": "rescale_percentile", "workload": "16384^2 fp32 plane, p=1",
                      "ms": round(ms, 3), "GB/s": round(gb / ms * 1e3, 1),
                      "roofline_frac": round(gb / ms * 1e3 / peak, 3)}), flush=True)


if __name__ == "__main__":
    main()
