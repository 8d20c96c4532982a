"""Time ut_region_moments on a cfg4pca-shaped cube (dev probe; env toggles:
UT_REGION_IMMA=0, UT_IMMA_DEBUG=1 (no MMA) / 2 (no conversion))."""
import os
import sys

import torch

import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import synthetic
from paper_1612_06457_b200.projection import PcaDevice

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cfg = synthetic.scaled(synthetic.CONFIGS["cfg4pca"], rows, 16384, 0)
st = synthetic.generate(synthetic.make_scene(cfg))
pd = PcaDevice(cfg.bands, st.planes.device)
cube = st.cube()
for _ in range(3):
    pd.moments_from(cube, 0, 0, cfg.width, cfg.height, st.planes.device)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    pd.moments_from(cube, 0, 0, cfg.width, cfg.height, st.planes.device)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
gb = cfg.pixels * cfg.bands * 4 / 1e9
print(f"{os.environ.get('UT_REGION_IMMA', '1')}/{os.environ.get('UT_IMMA_DEBUG', '0')}: "
      f"{ms:.3f} ms  {gb / ms:.1f} TB/s  m[1]={pd.local_moments()[1].item():.12f}")
