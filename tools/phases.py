"""Phase timing of cva_solve_kernel (needs a -DUT_PHASES build:
UT_NVCC_FLAGS=-DUT_PHASES python -m paper_1612_06457_b200.build --force)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402

L = ut._lib.lib()
f = L.ut_debug_eig_phases
f.argtypes = [C.c_void_p]
for name, h, w in (("cfg1", 512, 512), ("cfg4", 1024, 1024)):
    cfg = synthetic.scaled(synthetic.CONFIGS[name], h, w)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
    for _ in range(3):
        pipe.fit_only()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 32)()
    f(C.cast(buf, C.c_void_p))
    t = np.array(list(buf), dtype=np.float64)
    t0 = t[0]
    print(cfg.name, [round((t[i] - t0) / 1000, 1) for i in range(11)], "us")
    print("   jacobi sweeps (C x C team32, full team128):", int(t[30]), int(t[31]))
# full path (general / PCA) sweeps
import paper_1612_06457_b200.projection as pj  # noqa: E402
cfg = synthetic.scaled(synthetic.CONFIGS["cfg4pca"], 512, 512)
stack = synthetic.generate(synthetic.make_scene(cfg))
for _ in range(2):
    pm = ut.fit_pca_unsupervised(stack, k=5)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 32)()
f(C.cast(buf, C.c_void_p))
print("PCA B=32 full Jacobi sweeps:", int(buf[31]))
