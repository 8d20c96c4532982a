"""The library's own collectives (include/undertext_b200.h: ut_comm_*,
ut_allgather_f64, ut_allreduce_f32/f64 over NCCL) on one rank, and the
sharded pipeline code path driven through them: identical results to the
unsharded pipeline, and the step (kernels + NCCL collectives on one stream)
captured into a CUDA graph replays bit-identically.  N > 1 runs on the
driver's multi-GPU bench, which self-checks against an unsharded fit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_06457_b200 as ut  # noqa: E402
from paper_1612_06457_b200 import comm as ucomm, synthetic  # noqa: E402


@pytest.fixture(scope="module")
def comm():
    assert ucomm.available() > 0, "NCCL (torch's libnccl.so.2) not loadable by the library"
    c = ucomm.Comm.single()
    yield c
    c.close()


def test_single_rank_collectives(comm):
    x = torch.randn(1000, dtype=torch.float64, device="cuda")
    for op in ("sum", "min", "max"):
        y = x.clone()
        comm.allreduce(y, op)
        assert torch.equal(x, y)
    f = torch.randn(10, dtype=torch.float32, device="cuda")
    g = f.clone()
    comm.allreduce(g, "max")
    assert torch.equal(f, g)
    out = torch.empty_like(x)
    comm.allgather_f64(x, out)
    assert torch.equal(out, x)
    with pytest.raises(TypeError):
        comm.allreduce(torch.zeros(3, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        comm.allgather_f64(x, torch.empty(10, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("method", ["cva", "pca"])
def test_pipeline_through_comm_and_graph(comm, method):
    cfg = synthetic.scaled(synthetic.CONFIGS["cfg4"], 256, 192, per_class=80)
    scene = synthetic.make_scene(cfg)
    stack = synthetic.generate(scene)

    def make(c):
        if method == "cva":
            return ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k, comm=c)
        return ut.PcaPipeline(stack, k=cfg.k, comm=c)

    ref = make(None)
    want = ref.run().clone()
    pipe = make(comm)
    got = pipe.run().clone()
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    np.testing.assert_array_equal(pipe.model().eigenvalues, ref.model().eigenvalues)
    pipe.capture()
    pipe.codes.zero_()
    pipe.replay()
    torch.cuda.synchronize()
    assert torch.equal(pipe.codes, want)
    pipe.check()
