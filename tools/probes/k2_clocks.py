"""SM clock / power under a sustained K2 loop (dev probe): is the MMA's cost in
region_imma_kernel a clock effect (power cap) or cycles?  Run once per setting of
UT_IMMA_DEBUG (0 = shipped, 1 = no MMA); prints per-call ms (first / last calls)
and the nvidia-smi samples taken during the loop."""
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1612_06457_b200 import synthetic  # noqa: E402
from paper_1612_06457_b200.projection import PcaDevice  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cfg = synthetic.CONFIGS["cfg4pca"]
st = synthetic.generate(synthetic.make_scene(cfg))
pd = PcaDevice(cfg.bands, st.planes.device)
cube = st.cube()
for _ in range(3):
    pd.moments_from(cube, 0, 0, cfg.width, cfg.height, st.planes.device)
torch.cuda.synchronize()
time.sleep(3)
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap",
                      "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
evs = []
for _ in range(calls):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pd.moments_from(cube, 0, 0, cfg.width, cfg.height, st.planes.device)
    b.record()
    evs.append((a, b))
torch.cuda.synchronize()
time.sleep(0.1)
p.terminate()
out = p.stdout.read().strip().splitlines()
ms = [a.elapsed_time(b) for a, b in evs]
rows = [[x.strip() for x in l.split(",")] for l in out if l.count(",") >= 3]
sm = [float(r[0]) for r in rows]
pw = [float(r[2]) for r in rows]
busy = [s for s, w in zip(sm, pw) if w > 300]
print(f"UT_IMMA_DEBUG={os.environ.get('UT_IMMA_DEBUG', '0')} calls={calls} "
      f"first5={np.round(ms[:5], 3).tolist()} last5={np.round(ms[-5:], 3).tolist()} mean={np.mean(ms):.3f}")
print(f"  smi samples={len(rows)} sm_mhz under load: median={np.median(busy) if busy else None} "
      f"min={min(busy) if busy else None} max={max(busy) if busy else None} power max={max(pw) if pw else None} "
      f"power_cap_flags={sum(1 for r in rows if 'Active' == r[3])}")
