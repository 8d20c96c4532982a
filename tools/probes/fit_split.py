"""In-step split of the CVA fit at cfg 4 (dev probe): moments (K1 + merge) vs
solve (K3), CUDA events, hot."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402

torch.cuda.set_device(0)
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cfg = synthetic.scaled(synthetic.CONFIGS["cfg4"], rows, 16384)
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
for _ in range(5):
    pipe.run()
torch.cuda.synchronize()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(20)]
for e in ev:
    pipe.project_kernel()          # evict the fit's data like a real step
    e[0].record()
    pipe.fit.moments_from_cube(pipe.cube, pipe.xy, pipe.cls, pipe.n, pipe.first_bad, pipe.pivots)
    e[1].record()
    pipe.fit.solve(pipe.ridge, pipe.k)
    e[2].record()
torch.cuda.synchronize()
m = np.mean([e[0].elapsed_time(e[1]) for e in ev]) * 1e3
s = np.mean([e[1].elapsed_time(e[2]) for e in ev]) * 1e3
print(f"moments (K1 + merge): {m:.1f} us   solve (K3): {s:.1f} us   n = {pipe.n}")
