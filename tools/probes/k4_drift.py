"""Dev probe: K4 (projection), K5 and the fit timed alone and back to back on the
cfg 4 cube, then K4 again after 2 s idle -- shows the sustained-load drift
(DESIGN.md §10.3).  Run on the GPU box with PYTHONPATH=."""
import torch, numpy as np, time
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import synthetic
cfg = synthetic.CONFIGS["cfg4"]
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
for _ in range(5): pipe.run()
torch.cuda.synchronize()
def t(fn, n=30):
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/n
for rep in range(2):
    print("K4 alone x30", round(t(pipe.project_kernel),4))
    print("K5 alone x30", round(t(pipe.stretch_only),4))
    print("fit alone x30", round(t(pipe.fit_only),4))
    print("full step x30", round(t(pipe.run),4))
    print("K4+K5 x30", round(t(lambda: (pipe.project_kernel(), pipe.stretch_only())),4))
    time.sleep(2)
    print("after 2s idle: K4 x5", round(t(pipe.project_kernel, 5),4))
