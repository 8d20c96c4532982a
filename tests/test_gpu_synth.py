"""The device generator (csrc/synth.cu) against its host restatement
(oracle/synth.py), bit for bit.

bench.py's reference arm builds its inputs with oracle/synth.py so that it
never maps the repo's CUDA library; these tests are what lets that arm claim
it measures the same cube the device arm measures.
"""

import numpy as np
import pytest

from oracle import synth as host_synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1612_06457_b200 import synthetic  # noqa: E402


def _bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_small_cubes_bit_identical(name):
    cfg = synthetic.scaled(synthetic.CONFIGS[name], 96, 80,
                           per_class=20 if synthetic.CONFIGS[name].per_class else 0)
    scene = synthetic.make_scene(cfg)
    dev = synthetic.generate(scene).planes.cpu().numpy()
    host = host_synth.rows(scene, 0, cfg.height)
    assert dev.dtype == host.dtype
    assert np.array_equal(_bits(dev), _bits(host))


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
def test_full_size_rows_and_training_pixels_bit_identical(name):
    """Row blocks of the full-size cubes (generated as row shards on the
    device) and every training pixel of the scene."""
    cfg = synthetic.CONFIGS[name]
    scene = synthetic.make_scene(cfg)
    for r0 in (0, cfg.height // 2 - 1, cfg.height - 3):
        dev = synthetic.generate(scene, row0=r0, rows=3).planes.cpu().numpy()
        host = host_synth.rows(scene, r0, r0 + 3)
        assert np.array_equal(_bits(dev), _bits(host)), r0
    pick = np.random.default_rng(0).choice(len(scene.xs), 2000, replace=False)
    ys, xs = scene.ys[pick], scene.xs[pick]
    host = host_synth.pixels(scene, ys, xs)
    dev = np.stack([synthetic.generate(scene, row0=int(y), rows=1).planes[:, 0, int(x)]
                    .cpu().numpy() for y, x in zip(ys[:40], xs[:40])], axis=1)
    assert np.array_equal(_bits(dev), _bits(host[:, :40]))


def test_generator_statistics():
    """The generator draws what BASELINE.json describes: per class,
    mean + L z with z ~ N(0, I) (clipping is rare at these means)."""
    cfg = synthetic.scaled(synthetic.CONFIGS["cfg4"], 512, 512, per_class=0)
    scene = synthetic.make_scene(cfg)
    cube = synthetic.generate(scene).planes.double().cpu().numpy()
    cls = synthetic.class_map_at(scene.shapes, *np.meshgrid(np.arange(512), np.arange(512),
                                                              indexing="ij"))
    for c in range(cfg.classes):
        x = cube[:, cls == c]
        if x.shape[1] < 5000:
            continue
        want_cov = scene.chol[c] @ scene.chol[c].T
        assert np.allclose(x.mean(axis=1), scene.means[c], atol=5 * np.sqrt(want_cov.max()
                                                                              / x.shape[1]) + 1e-4)
        got_cov = np.cov(x)
        assert np.abs(got_cov - want_cov).max() <= 0.1 * np.abs(want_cov).max()
