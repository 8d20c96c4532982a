"""FolioStream (the streamed e2e path: pinned host cubes, double-buffered H2D, per-folio
training sets) against stand-alone pipelines and the oracle: random folio counts, shapes,
dtypes, band and class counts (dev tool; python tools/fuzz/fuzz_folios.py [seed])."""
import sys, traceback
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch
import oracle
import paper_1612_06457_b200 as ut
from test_gpu_edges import cube_of, pick_points, DTYPES
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 31)
fails = 0
for it in range(40):
    try:
        nf = int(rng.integers(1, 6)); b = int(rng.integers(2, 33)); classes = int(rng.integers(2, 6))
        h = int(rng.integers(8, 150)); w = int(rng.integers(8, 200))
        dtype = DTYPES[int(rng.integers(0, len(DTYPES)))]
        depth = 16 if dtype == np.uint16 else 8
        k = int(rng.integers(1, min(b, classes - 1) + 1))
        cubes, train, outs, want, host = [], [], [], [], []
        ok = True
        per = int(rng.integers(b + 3, b + 50))   # one training-set size per stream (FolioStream's contract)
        for f in range(nf):
            cube, cmap = cube_of(rng, b, h, w, dtype, classes=classes)
            xs, ys, ls = pick_points(rng, cmap, per)
            if len(np.unique(ls)) != classes or len(ls) != per * classes:
                ok = False
                break
            host.append((cube, xs, ys, ls))
            cubes.append(torch.from_numpy(cube).pin_memory())
            arrs = ut.CvaPipeline.training_arrays(xs, ys, ls)
            train.append(tuple(torch.from_numpy(a).pin_memory() for a in arrs))
            outs.append(torch.empty((k, h, w), dtype=torch.uint8, pin_memory=True))
            ds = ut.DeviceStack(ut.stack.default_bands(b), torch.from_numpy(cube).cuda(), depth, True)
            want.append(ut.CvaPipeline(ds, xs, ys, ls, k=k).run().cpu().numpy())
        if not ok:
            continue
        fs = ut.FolioStream(cubes, train, outs, k=k)
        for _ in range(2):
            fs.run()
            torch.cuda.synchronize()
            fs.check()
            for f in range(nf):
                assert np.array_equal(outs[f].numpy(), want[f]), ("folio vs pipeline", it, f, nf, b, h, w)
        cube, xs, ys, ls = host[-1]
        ref = oracle.fit_cva(oracle.assemble(cube, xs, ys), ls, k=k)
        planes = oracle.project(cube, {"mean": ref["mean"], "std": None, "coefficients": ref["coefficients"]})
        for j in range(k):
            a = oracle.rescale_full(planes[j]).astype(int)
            got = outs[-1].numpy()[j].astype(int)
            assert min(np.abs(got - a).max(), np.abs(255 - got - a).max()) <= 1, ("folio vs oracle", it, j)
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:220], traceback.format_exc().splitlines()[-3][:150], flush=True)
print("fuzz folios done, fails:", fails)
