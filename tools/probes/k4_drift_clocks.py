import torch, time, subprocess, os
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import synthetic
cfg = synthetic.CONFIGS["cfg4"]
scene = synthetic.make_scene(cfg)
stack = synthetic.generate(scene)
pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
for _ in range(3): pipe.run()
torch.cuda.synchronize(); time.sleep(3)
fh = open("gpurun_out/smi.csv", "w")
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.hw_thermal_slowdown", "--format=csv,noheader", "-lms", "20"], stdout=fh)
time.sleep(0.5)
evs = []
for i in range(60):
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); pipe.project_kernel(); b.record(); evs.append((a,b))
torch.cuda.synchronize()
time.sleep(0.5)
p.terminate(); fh.close()
print([round(a.elapsed_time(b),2) for a,b in evs])
