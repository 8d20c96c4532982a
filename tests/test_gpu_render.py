"""render_planes and compose_rgb on the device (pipeline.py:136-190,
rendering.py:206-225): the written files decode to exactly
the codes the per-plane API renders, full-range codes are within one level of
the oracle's, composites follow the recipe, names and order match the
reference's RenderResult."""

import warnings

import numpy as np
import pytest

import oracle
from cubes import make_cube

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
cv2 = pytest.importorskip("cv2")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402


def load(path):
    img = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    assert img is not None
    return np.ascontiguousarray(img[:, :, ::-1]) if img.ndim == 3 else img


@pytest.fixture(scope="module")
def case():
    cube, xs, ys, labels = make_cube(96, 130, 16, 3, np.float64, seed=21, per_class=60)
    stack = ut.SpectralStack(ut.stack.default_bands(16), cube, 8, True)
    model = ut.fit_cva(ut.assemble_matrix(stack, ut.TrainingSet.from_arrays(xs, ys, labels)), k=2)
    return cube, stack, model


@pytest.mark.parametrize("fmt,compression", [("png", "none"), ("tif", "none"), ("tif", "deflate")])
def test_render_planes_files(tmp_path, case, fmt, compression):
    cube, stack, model = case
    specs = [ut.RenderSpec(), ut.RenderSpec("percentile", 1.0, out_depth=16),
             ut.RenderSpec("training")]
    recipe = ut.CompositeRecipe(0, 1, 1, swap=(0, 2))
    res = ut.render_planes(stack, model, specs, tmp_path, run_name="pg", recipe=recipe, fmt=fmt,
                           compression=compression)
    names = [p.name for p in res.plane_paths]
    assert names == [f"pg_plane{k:02d}{s.suffix()}.{fmt}" for k in range(2) for s in specs]
    assert res.composite_path.name == "pg_R0G1B1_swap02.png"
    planes = ut.project_stack(ut.stack.on_device(stack), model)
    first = []
    for k in range(2):
        for s, spec in enumerate(specs):
            want = ut.rescale(planes[k], spec, model=model, k=k)
            want = want.cpu().numpy() if isinstance(want, torch.Tensor) else want
            got = load(tmp_path / ut.plane_filename("pg", k, spec, fmt))
            assert got.dtype == want.dtype and np.array_equal(got, want)
            if s == 0:
                first.append(want)
    # full-range codes against the oracle's projection + stretch (sign-aligned)
    ref = oracle.project(cube, {"mean": model.mean, "std": None,
                                "coefficients": model.coefficients}, workers=1)
    for k in range(2):
        codes = oracle.rescale_full(ref[k])
        assert int(np.abs(first[k].astype(int) - codes.astype(int)).max()) <= 1
    comp = load(res.composite_path)
    want = np.stack([first[0], first[1], first[1]], -1)[:, :, [2, 1, 0]]
    assert np.array_equal(comp, want)


def test_render_planes_write_failure_is_a_data_error(tmp_path, case):
    """A file that cannot be written surfaces as the reference's DataError even
    though the writes run on the writer pool, and the other planes are written."""
    cube, stack, model = case
    (tmp_path / "run_plane01_full.png").mkdir()        # a directory where plane 1 should go
    with pytest.raises(ut.DataError, match="failed to write image"):
        ut.render_planes(stack, model, [ut.RenderSpec()], tmp_path)
    assert (tmp_path / "run_plane00_full.png").is_file()


def test_pending_encodes_finish_in_any_order(case):
    """encode_*_start keeps encodes in flight; their bytes do not depend on when or
    where (another thread) they are collected."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1612_06457_b200 import image_io

    cube, stack, model = case
    planes = ut.project_stack(ut.stack.on_device(stack), model)
    imgs = [ut.rescale_full(p) for p in planes]
    want = [image_io.encode_png(i) for i in imgs] + [image_io.encode_tiff(i, "deflate") for i in imgs]
    pend = [image_io.encode_png_start(i) for i in imgs] + \
           [image_io.encode_tiff_start(i, "deflate") for i in imgs]
    with ThreadPoolExecutor(max_workers=3) as pool:
        got = list(pool.map(lambda q: q.bytes(), reversed(pend)))[::-1]
    assert got == want


def test_render_planes_device_stack_and_subset(tmp_path, case):
    cube, stack, model = case
    ds = ut.stack.on_device(stack)
    res = ut.render_planes(ds, model, [ut.RenderSpec()], tmp_path, components=[1])
    assert [p.name for p in res.plane_paths] == ["run_plane01_full.png"]
    with pytest.raises(ut.DataError, match="recipe needs planes"):
        ut.render_planes(ds, model, [ut.RenderSpec()], tmp_path, components=[1],
                         recipe=ut.CompositeRecipe(0, 1, 1))


def test_render_constant_plane_warns(tmp_path):
    cube = np.full((3, 8, 9), 0.5)
    stack = ut.SpectralStack(ut.stack.default_bands(3), cube, 8, True)
    model = ut.fit_pca_unsupervised(stack, k=1)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        res = ut.render_planes(stack, model, [ut.RenderSpec()], tmp_path)
    assert any(issubclass(x.category, ut.UndertextWarning) for x in w)
    assert not load(res.plane_paths[0]).any()


class TestComposite:
    """rendering.py:206-225 and the reference's tests (test_rendering.py:207-248)."""

    def planes(self, device=False, dtype=np.uint8):
        ps = [np.full((4, 4), v, dtype=dtype) for v in (10, 20, 30)]
        return [torch.from_numpy(p.astype(np.int32)).to(torch.uint8 if dtype == np.uint8 else torch.uint16).cuda()
                for p in ps] if device else ps

    @pytest.mark.parametrize("device", [False, True])
    def test_assignment_repeats_swap(self, device):
        def px(img):
            img = img.cpu().numpy() if isinstance(img, torch.Tensor) else img
            assert img.shape == (4, 4, 3)
            return img[0, 0].tolist()
        p = self.planes(device)
        assert px(ut.compose_rgb(p, ut.CompositeRecipe(0, 1, 2))) == [10, 20, 30]
        assert px(ut.compose_rgb(p, ut.CompositeRecipe(2, 2, 0))) == [30, 30, 10]
        assert px(ut.compose_rgb(p, ut.CompositeRecipe(0, 1, 2, swap=(1, 2)))) == [10, 30, 20]

    def test_errors(self):
        p = self.planes()
        with pytest.raises(ut.DataError):
            ut.compose_rgb(p, ut.CompositeRecipe(0, 1, 3))
        q = list(p)
        q[1] = np.zeros((5, 4), dtype=np.uint8)
        with pytest.raises(ut.DataError):
            ut.compose_rgb(q, ut.CompositeRecipe(0, 1, 2))
        q = list(p)
        q[2] = np.zeros((4, 4), dtype=np.uint16)
        with pytest.raises(ut.DataError):
            ut.compose_rgb(q, ut.CompositeRecipe(0, 1, 2))

    @pytest.mark.parametrize("shape", [(1, 1), (3, 5), (517, 1023)])
    @pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
    def test_large_and_ragged(self, shape, dtype):
        rng = np.random.default_rng(3)
        ps = [rng.integers(0, np.iinfo(dtype).max, size=shape).astype(dtype) for _ in range(3)]
        got = ut.compose_rgb(ps, ut.CompositeRecipe(2, 0, 1))
        assert np.array_equal(got, np.stack([ps[2], ps[0], ps[1]], -1))
