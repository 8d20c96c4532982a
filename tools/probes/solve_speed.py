"""Time the PCA solve (B = 32 Jacobi) and the general CVA solve on small images
where the moments are cheap (dev probe)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402


def t(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


torch.cuda.set_device(0)
cfg = synthetic.scaled(synthetic.CONFIGS["cfg4pca"], 128, 128, 0)
st = synthetic.generate(synthetic.make_scene(cfg))
pca = ut.PcaPipeline(st, k=5)
print(f"pca fit (128x128x32 moments + B=32 solve): {t(pca.fit_only):.1f} us  evals[0]={pca.model().eigenvalues[0]:.12f}")
cfg = synthetic.scaled(synthetic.CONFIGS["cfg4"], 256, 256, 200)
sc = synthetic.make_scene(cfg)
st = synthetic.generate(sc)
cva = ut.CvaPipeline(st, sc.xs, sc.ys, sc.labels, k=32)
print(f"cva fit, all 32 components (general path): {t(cva.fit_only):.1f} us")
cva5 = ut.CvaPipeline(st, sc.xs, sc.ys, sc.labels, k=5)
print(f"cva fit, k = 5 (low-rank path): {t(cva5.fit_only):.1f} us")
