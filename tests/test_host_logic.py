"""Host-side logic that needs no GPU: sharding arithmetic, point routing,
class indexing, the synthetic scene (class map, training points), the model
JSON contract, input validation that happens before any device work, and the
no-fallback rule."""

import numpy as np
import pytest

import paper_1612_06457_b200 as ut
from paper_1612_06457_b200 import synthetic
from paper_1612_06457_b200.projection import class_index


def test_row_bounds_partition():
    for h in (1, 7, 512, 16384):
        for g in (1, 2, 3, 4, 8):
            spans = [ut.row_bounds(h, g, r) for r in range(g)]
            assert spans[0][0] == 0 and spans[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_route_points_covers_each_point_once():
    rng = np.random.default_rng(0)
    ys = rng.integers(0, 1000, 5000)
    seen = np.zeros(5000, int)
    for g in range(8):
        r0, r1 = ut.row_bounds(1000, 8, g)
        own = ut.route_points(ys, r0, r1 - r0)
        assert np.all(np.diff(own) > 0)  # original order kept
        seen[own] += 1
    assert np.all(seen == 1)


def test_class_index_sorted_unique():
    ids, idx = class_index(np.array([7, 2, 9, 2, 7]))
    assert ids == (2, 7, 9)
    assert idx.tolist() == [1, 0, 2, 0, 1]


def test_scene_training_points_respect_class_map():
    cfg = synthetic.scaled(synthetic.CONFIGS["cfg3"], 400, 300, per_class=100)
    sc = synthetic.make_scene(cfg)
    assert len(sc.xs) == 4 * 100
    assert np.array_equal(synthetic.class_map_at(sc.shapes, sc.ys, sc.xs), sc.labels)
    flat = sc.ys * cfg.width + sc.xs
    for c in range(4):
        sel = flat[sc.labels == c]
        assert len(np.unique(sel)) == len(sel)  # without replacement
    again = synthetic.make_scene(cfg)
    assert np.array_equal(again.xs, sc.xs) and np.array_equal(again.shapes, sc.shapes)


def test_scene_class_coverage():
    cfg = synthetic.scaled(synthetic.CONFIGS["cfg1"], 256, 256, per_class=10)
    sc = synthetic.make_scene(cfg)
    yy, xx = np.mgrid[0:256, 0:256]
    cmap = synthetic.class_map_at(sc.shapes, yy, xx)
    frac = np.bincount(cmap.ravel(), minlength=3) / cmap.size
    assert 0.04 < frac[1] < 0.2 and 0.04 < frac[2] < 0.2  # "~10% each"


def test_config_bytes_per_pixel():
    assert synthetic.CONFIGS["cfg4"].bytes_per_pixel() == 32 * 4 + 5
    assert synthetic.CONFIGS["cfg1"].bytes_per_pixel() == 16 * 8 + 2
    assert synthetic.CONFIGS["cfg2"].bytes_per_pixel() == 2 * 16 * 4 + 3
    assert synthetic.CONFIGS["cfg3"].bytes_per_pixel() == 23 * 2 + 3


def test_model_json_round_trip(tmp_path):
    m = ut.ProjectionModel("cva", np.array([0.1, 0.2]), None, np.array([[1.0], [2.0 / 3.0]]),
                           np.array([3.5]), np.array([[0.25, -1e-300]]), {"a": "b"})
    m.save(tmp_path / "m.json")
    again = ut.ProjectionModel.load(tmp_path / "m.json")
    assert np.array_equal(again.coefficients, m.coefficients)
    assert np.array_equal(again.training_scores, m.training_scores)
    assert again.std is None and again.provenance == {"a": "b"}
    doc = m.to_dict()
    doc["version"] = 99
    with pytest.raises(ut.DataError, match="version"):
        ut.ProjectionModel.from_dict(doc)
    with pytest.raises(ut.DataError):
        ut.ProjectionModel("nope", m.mean, None, m.coefficients, m.eigenvalues)


def test_validation_before_device_work():
    st = ut.SpectralStack(ut.stack.default_bands(2), np.zeros((2, 6, 6), np.uint8), 8, True)
    with pytest.raises(ut.DataError, match="empty region"):
        ut.fit_pca_unsupervised(st, region=(0, 0, 0, 2))
    with pytest.raises(ut.DataError, match="outside"):
        ut.fit_pca_unsupervised(st, region=(4, 4, 5, 5))
    with pytest.raises(ut.DataError, match="at least 2 pixels"):
        ut.fit_pca_unsupervised(st, region=(0, 0, 1, 1))
    with pytest.raises(ut.DataError, match="components"):
        ut.fit_pca_unsupervised(st, k=3)
    with pytest.raises(ut.DataError):
        ut.SpectralStack(ut.stack.default_bands(2), np.zeros((2, 6, 6), np.uint16) + 300, 8)


def test_no_cpu_fallback(monkeypatch):
    """Without CUDA the compute entry points raise instead of computing."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    st = ut.SpectralStack(ut.stack.default_bands(2), np.ones((2, 6, 6), np.uint8), 8, True)
    with pytest.raises(RuntimeError, match="CUDA|fallback"):
        ut.fit_pca_unsupervised(st)
    with pytest.raises(RuntimeError, match="CUDA|fallback"):
        ut.solve_gen_eig_sym(np.eye(2), np.eye(2))
    with pytest.raises(RuntimeError, match="CUDA|fallback"):
        ut.rescale_full(ut.ScorePlane(np.array([[0.0, 1.0]])))


def test_product_never_imports_oracle():
    import pathlib

    pkg = pathlib.Path(ut.__file__).parent
    for src in pkg.rglob("*.py"):
        text = src.read_text()
        assert "import oracle" not in text and "from oracle" not in text, src


def test_sharded_local_record_does_not_alias_gather_output():
    """all_gather_into_tensor(moments, local): with NCCL an input that overlaps
    another rank's output slot is a race, so a sharded fit keeps its own record
    in a separate buffer (an unsharded fit writes slot 0 directly)."""
    from paper_1612_06457_b200.projection import CvaDevice, PcaDevice

    for fit in (CvaDevice(8, 3, "cpu", groups=4), PcaDevice(8, "cpu", groups=4)):
        loc, out = fit.local_moments(), fit.moments
        assert loc.numel() * 4 == out.numel()
        lo, hi = loc.data_ptr(), loc.data_ptr() + loc.numel() * 8
        assert hi <= out.data_ptr() or lo >= out.data_ptr() + out.numel() * 8
    for fit in (CvaDevice(8, 3, "cpu"), PcaDevice(8, "cpu")):
        assert fit.local_moments().data_ptr() == fit.moments.data_ptr()


def test_render_batch_sized_to_free_memory(monkeypatch):
    """render_planes projects up to 32 components per pass only when
    their fp32 planes and codes fit in half the free HBM (the reference batches
    8 to bound memory); otherwise fewer, never 0."""
    import types

    import torch

    from paper_1612_06457_b200 import pipeline

    ds = types.SimpleNamespace(height=16384, width=16384, planes=types.SimpleNamespace(device="cuda:0"))
    per_comp = 16384 * 16384 * (4 + 2 * 1)           # one spec, 16-bit codes bound
    for free, want in ((10**12, 32), (20 * per_comp, 10), (per_comp, 1), (0, 1)):
        monkeypatch.setattr(torch.cuda, "mem_get_info", lambda device=None, f=free: (f, 2 * f + 1))
        assert pipeline._render_batch(ds, 1) == want, (free, want)
