"""The reference's staged flow on the device, end to end from band files to
image files (pipeline.py:56-190: load_normalized -> fit_model -> render_planes),
against the oracle run on the same band files (cv2.imread, the oracle's
normalize / fit / project / stretch): codes within one level, models to the
parity bars."""

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


@pytest.fixture(scope="module")
def page(tmp_path_factory):
    d = tmp_path_factory.mktemp("page")
    cube, xs, ys, labels = make_cube(120, 160, 12, 4, np.uint16, seed=31, per_class=80, blobs=True)
    lines = []
    for b in range(cube.shape[0]):
        name = f"b{b:02d}.tif"
        assert cv2.imwrite(str(d / name), cube[b], [cv2.IMWRITE_TIFF_COMPRESSION, 8])
        lines.append(f"{name},{400 + 30 * b},visible")
    (d / "manifest.txt").write_text("\n".join(lines) + "\n")
    return d, cube, xs, ys, labels


def test_cli_flow_cva(tmp_path, page):
    d, cube, xs, ys, labels = page
    stack = ut.load_normalized(d / "manifest.txt")
    assert stack.normalized and stack.planes.dtype == torch.uint8
    codes_ref, _ = oracle.normalize_stack(cube)
    assert np.array_equal(stack.planes.cpu().numpy(), codes_ref)
    ts = ut.TrainingSet.from_arrays(xs, ys, labels)
    model = ut.fit_model(stack, ts, ut.METHOD_CVA, k=3)
    ref = oracle.fit_cva(oracle.assemble(codes_ref, xs, ys), labels, k=3)
    assert np.allclose(model.eigenvalues, ref["eigenvalues"], rtol=1e-9)
    res = ut.render_planes(stack, model, [ut.RenderSpec()], tmp_path, run_name="cli")
    planes = oracle.project(codes_ref, ref)
    for k, path in enumerate(res.plane_paths):
        got = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
        sign = np.sign(model.coefficients[:, k] @ ref["coefficients"][:, k])
        want = oracle.rescale_full(sign * planes[k])
        assert int(np.abs(got.astype(int) - want.astype(int)).max()) <= 1
    single = ut.project_single(stack, model, 1)
    assert tuple(single.values.shape) == cube.shape[1:]


def test_cli_flow_pca_and_crop(page):
    d, cube, *_ = page
    stack = ut.load_normalized(d / "manifest.txt", crop_rect=(10, 20, 100, 80))
    assert (stack.width, stack.height) == (100, 80)
    model = ut.fit_model(stack, None, ut.METHOD_PCA_UNSUPERVISED, k=2)
    codes_ref, _ = oracle.normalize_stack(cube[:, 20:100, 10:110])
    ref = oracle.fit_pca_unsupervised(codes_ref, k=2)
    assert np.allclose(model.eigenvalues, ref["eigenvalues"], rtol=1e-9)
    with pytest.raises(ut.DataError, match="needs annotations"):
        ut.fit_model(stack, None, ut.METHOD_CVA)


def test_model_provenance_order():
    prov = ut.model_provenance({"scope": "per-band", "manifest": "m.txt", "crop": None}, "x,y",
                               "cva", None, 1e-8)
    assert list(prov) == ["manifest", "crop", "scope", "annotations_sha256", "method", "k", "ridge"]
    assert prov["k"] == "all"
