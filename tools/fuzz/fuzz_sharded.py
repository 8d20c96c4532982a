"""Row-sharded CVA on ONE GPU against the unsharded run: random world sizes (2-8), heights not
divisible by them, shards without training points.  Every rank's row block is fitted /
projected exactly as that rank would (its own CvaPipeline with a fake process group); the
all-gather is replaced by copies of the ranks' real moment records and the all-reduce(MAX)
by a maximum over the ranks' min/max records.  Training sets are kept well conditioned
(n >= 2 B + C): with fewer points than bands W' is the ridge alone and the two combine orders
differ by more than 1e-9 in the (then meaningless) eigenvalues (dev tool; python tools/fuzz/fuzz_sharded.py [seed])."""
import sys, traceback
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch
import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import pipeline
from golden_util import align_signs, rel_close
from test_gpu_edges import cube_of, pick_points, DTYPES


class _Fake:
    pass


rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 21)
real_ws = pipeline.dist.get_world_size
fails = 0
for it in range(60):
    try:
        g = int(rng.integers(2, 9)); b = int(rng.integers(2, 33)); classes = int(rng.integers(2, 7))
        h = int(rng.integers(g, 160)); w = int(rng.integers(8, 200))
        dtype = DTYPES[int(rng.integers(0, len(DTYPES)))]
        cube, cmap = cube_of(rng, b, h, w, dtype, classes=classes)
        xs, ys, ls = pick_points(rng, cmap, int(rng.integers(b + 3, b + 60)))   # W well conditioned (n >> B)
        if it % 3 == 0:                       # all points in the top third: some ranks own none
            keep = ys < max(2, h // 3)
            if len(np.unique(ls[keep])) >= 2:
                xs, ys, ls = xs[keep], ys[keep], ls[keep]
        if len(np.unique(ls)) < 2 or len(ls) < 2 * b + classes:
            continue
        k = int(rng.integers(1, min(b, len(np.unique(ls)) - 1) + 1))
        depth = 16 if dtype == np.uint16 else 8
        whole = ut.DeviceStack(ut.stack.default_bands(b), torch.from_numpy(cube).cuda(), depth, True)
        ref = ut.CvaPipeline(whole, xs, ys, ls, k=k)
        ref_codes = ref.run().cpu().numpy()
        ref_h = ref.check()
        pipes = []
        for r in range(g):
            r0, r1 = ut.row_bounds(h, g, r)
            part = ut.DeviceStack(ut.stack.default_bands(b),
                                  torch.from_numpy(np.ascontiguousarray(cube[:, r0:r1])).cuda(),
                                  depth, True, row0=r0, full_height=h)
            fake = _Fake()
            pipeline.dist.get_world_size = lambda grp=None, _f=fake, _g=g: _g if grp is _f else real_ws(grp)
            try:
                p = ut.CvaPipeline(part, xs, ys, ls, k=k, group=fake)
            finally:
                pipeline.dist.get_world_size = real_ws
            pipes.append(p)
        recs = []
        for p in pipes:
            if p.n:
                p.fit.moments_from_cube(p.cube, p.xy, p.cls, p.n, p.first_bad, p.pivots)
            else:
                p.fit.local_moments().zero_()
            recs.append(p.fit.local_moments().clone())
        full = torch.stack(recs)
        mms = []
        for p in pipes:
            p.fit.moments.view(g, -1).copy_(full)
            p.fit.solve(p.ridge, p.k)
            p.project_kernel()
            mms.append(p.minmax.clone())
        mm = torch.stack(mms).max(dim=0).values
        codes = []
        for p in pipes:
            p.minmax.copy_(mm)
            p.stretch_only()
            codes.append(p.codes.cpu().numpy())
        codes = np.concatenate(codes, axis=1)
        hh = pipes[0].check()
        lam = ref_h["evals"][:k]
        assert np.all(np.abs(hh["evals"][:k] - lam) <= 1e-9 * np.abs(lam).max()), ("evals", g, b, h, w)
        v = align_signs(hh["evecs"][:, :k], ref_h["evecs"][:, :k])
        assert rel_close(v, ref_h["evecs"][:, :k], 1e-6), ("evecs", g, b, h, w)
        s = np.sign(np.sum(hh["evecs"][:, :k] * ref_h["evecs"][:, :k], axis=0))
        for j in range(k):
            a = codes[j].astype(int) if s[j] > 0 else (np.iinfo(codes.dtype).max - codes[j].astype(int))
            assert np.abs(a - ref_codes[j].astype(int)).max() <= 1, ("codes", g, j, b, h, w)
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:220], traceback.format_exc().splitlines()[-3][:150], flush=True)
print("fuzz sharded done, fails:", fails)
