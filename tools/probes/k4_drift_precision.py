import torch, time, os
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import synthetic
cfg = synthetic.CONFIGS["cfg4"]
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
def t(fn, n):
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/n
for prec in ("fp64", "fp32"):
    pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k, precision=prec)
    for _ in range(3): pipe.run()
    torch.cuda.synchronize(); time.sleep(3)
    seq = [round(t(pipe.project_kernel, 5), 3) for _ in range(12)]
    print(prec, "K4 x5 blocks:", seq)
    del pipe; torch.cuda.empty_cache()
# plain copy of the cube (device memcpy, read+write) to see HBM drift alone
src = stack.planes.view(-1)
dst = torch.empty(src.numel() // 4, dtype=src.dtype, device="cuda")
time.sleep(3)
seq = [round(t(lambda: dst.copy_(src[:dst.numel()]), 20), 3) for _ in range(12)]
print("copy 8.6GB x20 blocks:", seq)
# read-only reduction over the cube (sum) 
time.sleep(3)
seq = [round(t(lambda: src.sum(), 3), 3) for _ in range(12)]
print("sum 34GB x3 blocks:", seq)
