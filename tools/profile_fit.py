"""One warm + one measured fit of a scaled config (for ncu -s/-c windows).

    python tools/profile_fit.py [cfg4] [rows] [cols]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
h = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
w = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
cfg = synthetic.scaled(synthetic.CONFIGS[name], h, w)
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
for _ in range(2):
    pipe.fit_only()
torch.cuda.synchronize()
pipe.check()
print("ok", cfg.name)
