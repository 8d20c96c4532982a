"""INTEGRATION.md's recipe end to end on the GPU, with objects shaped like the
reference's own types.

/root/reference does not travel to the GPU box, so these stand-ins reproduce
the reference's public fields (annotations.py:23-103 ClassLabel /
AnnotatedPoint / TrainingSet / DesignMatrix, stack.py:22-98 BandMeta /
SpectralStack, rendering.py:39-60 ScorePlane, projection.py:55-96
ProjectionModel) as plain frozen dataclasses -- none of this package's types.
The drop-ins must accept them (duck typing, round-1 VERDICT weak #5) and give
the oracle's results: fits to the Appendix-A bars, planes to 1e-6 of their
range, codes bit-exact against the oracle's stretch of the device planes.
LDA (projection.py:240-260) is checked against golden vectors of the real
reference (tests/golden/lda.npz).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import pytest

import oracle
from golden_util import align_signs, load, rel_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as b  # noqa: E402
from paper_1612_06457_b200 import pipeline as bp  # noqa: E402


# -- stand-ins with the reference's field names (no methods beyond those used) --
@dataclass(frozen=True)
class RefBandMeta:
    band_id: int
    wavelength_nm: float
    illumination: str
    filter: str | None = None


@dataclass(frozen=True)
class RefStack:
    bands: tuple
    planes: np.ndarray = field(repr=False)
    bit_depth: int
    normalized: bool = False

    @property
    def band_count(self):
        return len(self.bands)

    @property
    def width(self):
        return int(self.planes.shape[2])

    @property
    def height(self):
        return int(self.planes.shape[1])


@dataclass(frozen=True)
class RefLabel:
    name: str
    id: int


@dataclass(frozen=True)
class RefPoint:
    x: int
    y: int
    label: RefLabel


@dataclass(frozen=True)
class RefTraining:
    classes: tuple
    points: tuple
    provenance: dict = field(default_factory=dict)


@dataclass(frozen=True)
class RefDesign:
    values: np.ndarray
    labels: np.ndarray
    class_names: tuple

    @property
    def band_count(self):
        return int(self.values.shape[0])

    @property
    def point_count(self):
        return int(self.values.shape[1])


@dataclass(frozen=True)
class RefPlane:
    values: np.ndarray

    @property
    def height(self):
        return int(self.values.shape[0])

    @property
    def width(self):
        return int(self.values.shape[1])


@dataclass(frozen=True)
class RefModel:
    method: str
    mean: np.ndarray
    std: np.ndarray | None
    coefficients: np.ndarray
    eigenvalues: np.ndarray
    training_scores: np.ndarray | None = None
    provenance: dict = field(default_factory=dict)

    @property
    def band_count(self):
        return int(self.coefficients.shape[0])

    @property
    def component_count(self):
        return int(self.coefficients.shape[1])


def page(seed=21, b=12, h=96, w=128, classes=3, per=40):
    rng = np.random.default_rng(seed)
    means = rng.uniform(0.2, 0.8, size=(classes, b))
    cmap = (np.arange(w)[None, :] * classes // w).repeat(h, 0)
    x = np.clip(means[cmap] + rng.normal(scale=0.04, size=(h, w, b)), 0, 1)
    planes = np.ascontiguousarray(x.transpose(2, 0, 1))
    stack = RefStack(tuple(RefBandMeta(i, 400.0 + 10 * i, "uv") for i in range(b)), planes, 8,
                     normalized=True)
    labels = [RefLabel(f"class{c}", c) for c in range(classes)]
    pts = []
    for c in range(classes):
        ys = rng.integers(0, h, per)
        xs = rng.integers(c * w // classes, (c + 1) * w // classes, per)
        pts += [RefPoint(int(xx), int(yy), labels[c]) for xx, yy in zip(xs, ys)]
    return stack, RefTraining(tuple(labels), tuple(pts))


def host_design(stack, training):
    xs = np.array([p.x for p in training.points])
    ys = np.array([p.y for p in training.points])
    lab = np.array([p.label.id for p in training.points], dtype=np.intp)
    return RefDesign(stack.planes[:, ys, xs].astype(np.float64), lab,
                     tuple(c.name for c in training.classes))


def test_assemble_matrix_with_reference_types():
    stack, training = page()
    dm = b.assemble_matrix(stack, training)
    want = host_design(stack, training)
    got = dm.values.cpu().numpy() if torch.is_tensor(dm.values) else np.asarray(dm.values)
    assert np.array_equal(got, want.values)
    assert np.array_equal(np.asarray(dm.labels), want.labels)


def test_fits_accept_reference_design_matrix():
    stack, training = page()
    dm = host_design(stack, training)
    sp = b.compute_scatter(dm)
    ref = oracle.scatter(dm.values, dm.labels)
    assert np.array_equal(np.asarray(sp.counts), ref["counts"])
    for got, key in ((sp.within, "within"), (sp.between, "between"),
                     (sp.class_means, "class_means"), (sp.grand_mean, "grand_mean")):
        assert rel_close(got, ref[key], 1e-9), key
    m = b.fit_cva(dm, k=2)
    r = oracle.fit_cva(dm.values, dm.labels, k=2)
    assert rel_close(m.eigenvalues, r["eigenvalues"], 1e-9)
    assert rel_close(align_signs(m.coefficients, r["coefficients"]), r["coefficients"], 1e-6)
    # apply == training_scores (test_projection.py:122-127's contract)
    assert np.array_equal(m.apply(dm.values.T).T, m.training_scores)


def test_lda_and_standardize_vs_reference_golden():
    g = load("lda")
    for i in range(int(g["n"])):
        dm = RefDesign(g[f"{i}_values"], g[f"{i}_labels"].astype(np.intp), tuple())
        sdm, mean, std = b.standardize(dm)
        assert rel_close(np.asarray(sdm.values), g[f"{i}_std_values"], 1e-12), i
        assert rel_close(mean, g[f"{i}_mean"], 1e-12), i
        assert rel_close(std, g[f"{i}_std"], 1e-12), i
        m = b.fit_lda(dm, k=1)
        assert m.method == "lda"
        assert rel_close(m.eigenvalues, g[f"{i}_evals"], 1e-9), i
        coef = align_signs(m.coefficients, g[f"{i}_coef"])
        assert rel_close(coef, g[f"{i}_coef"], 1e-6), i
        sign = np.sign(np.sum(m.coefficients * g[f"{i}_coef"]))
        assert rel_close(sign * m.training_scores, g[f"{i}_scores"], 1e-6), i
    with pytest.raises(b.DataError, match="exactly 2"):
        b.fit_lda(RefDesign(np.zeros((3, 6)), np.array([0, 1, 2, 0, 1, 2]), tuple()))


def test_project_and_rescale_with_reference_types():
    stack, training = page()
    dm = host_design(stack, training)
    r = oracle.fit_cva(dm.values, dm.labels, k=2)
    model = RefModel("cva", r["mean"], None, r["coefficients"], r["eigenvalues"],
                     provenance={"normalized_input": True})
    planes = b.project_stack(stack, model)
    want = oracle.project(stack.planes, r)
    for j, plane in enumerate(planes):
        got = np.asarray(plane.values, dtype=np.float64) if not torch.is_tensor(plane.values) \
            else plane.values.double().cpu().numpy()
        rng = float(want[j].max() - want[j].min())
        assert float(np.abs(got - want[j]).max()) <= 1e-6 * rng, j
        # a reference ScorePlane of those planes -> drop-in rescale_full
        codes = b.rescale_full(RefPlane(got))
        assert np.array_equal(np.asarray(codes), oracle.rescale_full(got)), j


def test_pipeline_fit_model_and_render_planes_end_to_end(tmp_path):
    import cv2

    stack, training = page()
    model = bp.fit_model(stack, training, "cva", k=2)
    dm = host_design(stack, training)
    r = oracle.fit_cva(dm.values, dm.labels, k=2)
    assert rel_close(model.eigenvalues, r["eigenvalues"], 1e-9)
    spec = b.RenderSpec()
    res = bp.render_planes(stack, model, [spec], tmp_path, run_name="page")
    assert [p.name for p in res.plane_paths] == [bp.plane_filename("page", k, spec, "png")
                                                 for k in range(2)]
    assert res.plane_paths[0].name == "page_plane00_full.png"   # pipeline.py:120-125 names
    planes = b.project_stack(stack, model)
    for p, plane in zip(res.plane_paths, planes):
        img = cv2.imread(str(p), cv2.IMREAD_UNCHANGED)
        assert np.array_equal(img, np.asarray(b.rescale_full(plane)))


def test_lda_at_bench_scale_vs_oracle():
    """fit_lda on a device design matrix of the cfg 4 shape (B = 32, two classes,
    20,000 points each) against the oracle's standardize + CVA (projection.py:240-260)."""
    from paper_1612_06457_b200 import synthetic

    cfg = synthetic.scaled(synthetic.CONFIGS["cfg4"], 2048, 2048, per_class=20_000)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)
    keep = scene.labels < 2
    xy = torch.from_numpy(np.stack([scene.xs[keep], scene.ys[keep]], 1).astype(np.int32)).cuda()
    values, bad = b.annotations.gather(stack, xy, int(keep.sum()))
    assert int(bad.item()) == -1
    labels = scene.labels[keep].astype(np.intp)
    dm = b.DesignMatrix(values, labels, ("c0", "c1"))
    m = b.fit_lda(dm, k=1)
    ref = oracle.fit_lda(values.cpu().numpy(), labels, k=1)
    assert rel_close(m.mean, ref["mean"], 1e-9) and rel_close(m.std, ref["std"], 1e-9)
    assert rel_close(m.eigenvalues, ref["eigenvalues"], 1e-9)
    assert rel_close(align_signs(m.coefficients, ref["coefficients"]), ref["coefficients"], 1e-6)
