"""Per-kernel microbenchmarks of the fit path (CUDA events, hot, averaged).

    python tools/microbench.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import synthetic  # noqa: E402


def timed(fn, reps=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    torch.cuda.set_device(0)
    for name, h, w in (("cfg1", 512, 512), ("cfg3", 1024, 1024), ("cfg4", 1024, 1024)):
        cfg = synthetic.scaled(synthetic.CONFIGS[name], h, w)
        scene = synthetic.make_scene(cfg)
        stack = synthetic.generate(scene)
        pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k)
        pipe.run()
        pipe.check()
        f = pipe.fit
        t_mom = timed(lambda: f.moments_from_cube(pipe.cube, pipe.xy, pipe.cls, pipe.n,
                                                  pipe.first_bad, pipe.pivots))
        t_fast = timed(lambda: f.solve(1e-8, cfg.k))
        t_full = timed(lambda: f.solve(1e-8, 0))
        t_proj = timed(pipe.project_kernel)
        t_str = timed(pipe.stretch_only)
        t_run = timed(pipe.run)
        print(f"{cfg.name}: N={pipe.n} B={cfg.bands} C={cfg.classes} | moments {t_mom:.1f} us | "
              f"solve low-rank {t_fast:.1f} us | solve full {t_full:.1f} us | "
              f"project {t_proj:.1f} us | stretch {t_str:.1f} us | run {t_run:.1f} us", flush=True)
    for b in (16, 32):
        rng = np.random.default_rng(0)
        a = rng.normal(size=(b, b))
        m = a @ a.T + b * np.eye(b)
        cm = (a + a.T) / 2
        A = torch.from_numpy(cm).cuda()
        M = torch.from_numpy(m).cuda()
        out = torch.empty(b + b * b + b, dtype=torch.float64, device="cuda")
        info = torch.empty(1, dtype=torch.int32, device="cuda")
        L = ut._lib.lib()
        s = torch.cuda.current_stream().cuda_stream
        t_gen = timed(lambda: L.ut_gen_eig_sym(A.data_ptr(), M.data_ptr(), b, 1e-8, out.data_ptr(),
                                               out[b:].data_ptr(), out[b + b * b:].data_ptr(),
                                               info.data_ptr(), s))
        t_std = timed(lambda: L.ut_gen_eig_sym(A.data_ptr(), None, b, 0.0, out.data_ptr(),
                                               out[b:].data_ptr(), None, info.data_ptr(), s))
        print(f"gen_eig B={b}: generalized {t_gen:.1f} us, standard {t_std:.1f} us", flush=True)


if __name__ == "__main__":
    main()
