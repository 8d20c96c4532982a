"""render_planes with random specs (full / percentile / training, 8 / 16 bit), formats,
compressions, component subsets and composites: every written file is read back with cv2 and
compared with the device's rescale of the same plane (dev tool; python tools/fuzz/fuzz_render.py [seed])."""
import sys, tempfile, traceback, warnings
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np, torch, cv2
import paper_1612_06457_b200 as ut
from test_gpu_edges import cube_of, pick_points
warnings.simplefilter("ignore")
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 51)
fails = done = 0
def tonp(x): return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
for it in range(40):
    try:
        b = int(rng.integers(3, 25)); classes = int(rng.integers(3, 7))
        h = int(rng.integers(8, 160)); w = int(rng.integers(8, 240))
        cube, cmap = cube_of(rng, b, h, w, np.uint8, classes=classes)
        xs, ys, ls = pick_points(rng, cmap, b + 20)
        if len(np.unique(ls)) < 3:
            continue
        stack = ut.SpectralStack(ut.stack.default_bands(b), cube, 8, True)
        ts = ut.TrainingSet.from_arrays(xs, ys, ls)
        k = int(rng.integers(2, min(b, len(np.unique(ls)) - 1) + 1))
        model = ut.fit_cva(ut.assemble_matrix(stack, ts), k=k)
        pool = [ut.RenderSpec(), ut.RenderSpec(out_depth=16), ut.RenderSpec("training"),
                ut.RenderSpec("percentile", float(rng.choice([0.01, 0.1, 1.0, 5.0])), out_depth=int(rng.choice([8, 16])))]
        specs = [pool[i] for i in sorted(set(int(v) for v in rng.integers(0, len(pool), size=int(rng.integers(1, 4)))))]
        names = {s.suffix() for s in specs}
        if len(names) != len(specs):
            specs = specs[:1]
        fmt = str(rng.choice(["png", "tif"])); comp = str(rng.choice(["none", "deflate"]))
        comps = sorted(set(int(v) for v in rng.integers(0, k, size=int(rng.integers(1, k + 1)))))
        recipe = None
        if len(comps) >= 2 and it % 2:
            recipe = ut.CompositeRecipe(comps[0], comps[1], comps[0])
        out = tempfile.mkdtemp()
        res = ut.render_planes(stack, model, specs, out, run_name="f", components=comps, recipe=recipe,
                               fmt=fmt, compression=comp)
        planes = ut.project_stack(ut.stack.on_device(stack), model, components=comps)
        i = 0
        first = {}
        for kk, plane in zip(comps, planes):
            for s_i, spec in enumerate(specs):
                want = tonp(ut.rescale(plane, spec, model=model, k=kk))
                got = cv2.imread(str(res.plane_paths[i]), cv2.IMREAD_UNCHANGED)
                assert got is not None and got.dtype == want.dtype and np.array_equal(got, want), ("plane", kk, spec, fmt, comp)
                if s_i == 0:
                    first[kk] = want
                i += 1
        if recipe is not None and specs[0].out_depth == 8:
            comp_img = cv2.imread(str(res.composite_path), cv2.IMREAD_UNCHANGED)[:, :, ::-1]
            want = np.stack([first[recipe.red], first[recipe.green], first[recipe.blue]], -1)
            assert np.array_equal(comp_img, want), ("composite",)
        done += 1
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:240], traceback.format_exc().splitlines()[-3][:140], flush=True)
print("fuzz render done:", done, "pages, fails:", fails)
