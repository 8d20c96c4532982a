"""Per-CTA finish times of region_imma_kernel (K2) at cfg 4 (static round-robin tiles).
Needs a -DUT_K2_PROBE variant: python tools/build_variant.py region "-DUT_K2_PROBE" k2probe;
UT_LIB_PATH=scratch/lib_k2probe.so python tools/probes/k2_cta_spread.py"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402
from paper_1612_06457_b200.projection import PcaDevice  # noqa: E402

cfg = synthetic.CONFIGS["cfg4pca"]
st = synthetic.generate(synthetic.make_scene(cfg))
pd = PcaDevice(cfg.bands, st.planes.device)
cube = st.cube()
for _ in range(3):
    pd.moments_from(cube, 0, 0, cfg.width, cfg.height, st.planes.device)
torch.cuda.synchronize()
time.sleep(3)
L = ut._lib.lib()
f = L.ut_debug_k2_probe
f.argtypes = [C.c_void_p]
for rep in range(4):
    for _ in range(20 if rep else 1):   # rep 0: one launch after idle; later: sustained
        pd.moments_from(cube, 0, 0, cfg.width, cfg.height, st.planes.device)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 320)()
    f(C.cast(buf, C.c_void_p))
    t = np.array(list(buf), dtype=np.float64).reshape(160, 2)[:148]
    t0 = t[:, 0].min()
    end = (t[:, 1] - t0) / 1e3
    print(f"rep {rep}: CTA end (us): min {end.min():.0f} p10 {np.percentile(end, 10):.0f} median {np.median(end):.0f} "
          f"p90 {np.percentile(end, 90):.0f} max {end.max():.0f}; (max - median) = {100 * (end.max() - np.median(end)) / end.max():.2f}% "
          f"(max - min) = {100 * (end.max() - end.min()) / end.max():.2f}%; mean rate time {len(end) / np.sum(1.0 / end):.0f} us")
