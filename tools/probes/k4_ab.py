import torch, time, sys
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import synthetic
cfg = synthetic.CONFIGS["cfg4"]
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
for _ in range(3): pipe.run()
torch.cuda.synchronize()
def t(fn, n):
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/n
time.sleep(3)
fresh = [round(t(pipe.project_kernel, 1), 3) for _ in range(3)]
sus = [round(t(pipe.project_kernel, 5), 3) for _ in range(10)]
time.sleep(3)
step = [round(t(pipe.run, 5), 3) for _ in range(6)]
print(sys.argv[1] if len(sys.argv) > 1 else "", "K4 fresh", fresh, "sustained", sus, "step", step)
