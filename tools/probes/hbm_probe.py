"""This box's streaming bandwidth next to K4 (dev probe): torch copy (read +
write), a read-mostly reduction over the cfg4 cube, and the K4 projector on it."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


torch.cuda.set_device(0)
x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x)
ms = t(lambda: y.copy_(x))
print(f"copy 2 GiB -> 2 GiB: {ms:.3f} ms  {4 * (1 << 30) / ms / 1e6:.0f} GB/s")
del x, y
cfg = synthetic.CONFIGS["cfg4"]
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
flat = stack.planes.view(-1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
ms = t(lambda: torch.sum(flat, dim=0, out=out[0]))
print(f"sum over cube {flat.numel() * 4 / 1e9:.1f} GB: {ms:.3f} ms  {flat.numel() * 4 / ms / 1e6:.0f} GB/s")
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
pipe.run()
ms = t(lambda: pipe.project_kernel())
print(f"K4 fp64: {ms:.3f} ms  {148 * cfg.pixels / ms / 1e6:.0f} GB/s real (148 B/px)")
ms = t(lambda: pipe.stretch_only())
print(f"K5: {ms:.3f} ms  {25 * cfg.pixels / ms / 1e6:.0f} GB/s (25 B/px)")
