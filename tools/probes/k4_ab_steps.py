import torch, time, sys
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import synthetic
cfg = synthetic.CONFIGS["cfg4"]
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
for _ in range(5): pipe.run()
torch.cuda.synchronize()
a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): pipe.run()
b.record(); torch.cuda.synchronize()
print(sys.argv[1], round(a.elapsed_time(b)/50, 4))
