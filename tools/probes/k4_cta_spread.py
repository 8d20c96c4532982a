"""Per-CTA finish times of project_dmma_kernel (K4) at cfg 4: how much of the kernel
is the tail of its slowest CTAs (static round-robin tiles)?  Needs a -DUT_K4_PROBE
variant: python tools/build_variant.py project "-DUT_K4_PROBE" k4probe;
UT_LIB_PATH=scratch/lib_k4probe.so python tools/probes/k4_cta_spread.py"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402

cfg = synthetic.CONFIGS["cfg4"]
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
for _ in range(3):
    pipe.run()
torch.cuda.synchronize()
L = ut._lib.lib()
f = L.ut_debug_k4_probe
f.argtypes = [C.c_void_p]
for rep in range(4):
    for _ in range(10 if rep else 1):   # rep 0: one fresh launch; later reps: sustained
        pipe.project_kernel()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 2048)()
    f(C.cast(buf, C.c_void_p))
    t = np.array(list(buf), dtype=np.float64).reshape(1024, 2)[:296]
    t0 = t[:, 0].min()
    end = (t[:, 1] - t0) / 1e3
    start = (t[:, 0] - t0) / 1e3
    print(f"rep {rep}: CTA start spread {start.max():.1f} us; main-loop end (us): min {end.min():.0f} "
          f"p10 {np.percentile(end, 10):.0f} median {np.median(end):.0f} p90 {np.percentile(end, 90):.0f} "
          f"max {end.max():.0f}; tail (max - median) = {100 * (end.max() - np.median(end)) / end.max():.2f}% "
          f"(max - min) = {100 * (end.max() - end.min()) / end.max():.2f}%")
