"""The row-sharded pipelines end to end: two processes on cuda:0 with a gloo
process group (host-mediated collectives, so no kernel of one rank waits on
another's), each generating and projecting its own row block.  The combined
result must match the unsharded pipeline: identical class counts, eigenvalues
to 1e-10, score planes to 1e-6 of range, codes within +-1 (and the codes of every
shard bit-exact against the oracle's stretch of its own planes with the
all-reduced min/max).  This exercises the same code path as NCCL on 2-8 GPUs."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, method, out):
    import paper_1612_06457_b200 as ut
    from paper_1612_06457_b200 import synthetic

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name = "cfg4" if method == "cva" else "cfg2"
    cfg = synthetic.scaled(synthetic.CONFIGS[name], 250, 192, 150 if method == "cva" else 0)
    scene = synthetic.make_scene(cfg)
    r0, r1 = ut.row_bounds(cfg.height, world, rank)
    shard = synthetic.generate(scene, row0=r0, rows=r1 - r0)
    if method == "cva":
        pipe = ut.CvaPipeline(shard, scene.xs, scene.ys, scene.labels, k=cfg.k,
                              group=dist.group.WORLD)
    else:
        pipe = ut.PcaPipeline(shard, k=cfg.k, group=dist.group.WORLD)
    codes = pipe.run()
    model = pipe.model()
    out.put((rank, r0, r1, codes.cpu().numpy(), pipe.scores.cpu().numpy(),
             pipe.minmax.cpu().numpy(), model.eigenvalues, model.coefficients,
             pipe.fit.host().get("counts")))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("method", ["cva", "pca"])
def test_two_rank_pipeline_matches_unsharded(method):
    import oracle
    import paper_1612_06457_b200 as ut
    from paper_1612_06457_b200 import synthetic

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, method, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    torch.cuda.set_device(0)
    name = "cfg4" if method == "cva" else "cfg2"
    cfg = synthetic.scaled(synthetic.CONFIGS[name], 250, 192, 150 if method == "cva" else 0)
    scene = synthetic.make_scene(cfg)
    whole = synthetic.generate(scene)
    if method == "cva":
        ref = ut.CvaPipeline(whole, scene.xs, scene.ys, scene.labels, k=cfg.k)
    else:
        ref = ut.PcaPipeline(whole, k=cfg.k)
    ref.run()
    ref_model = ref.model()
    ref_scores = ref.scores.cpu().numpy()
    ref_codes = ref.codes.cpu().numpy()
    if method == "cva":
        assert np.array_equal(parts[0][8], ref.fit.host()["counts"])
    for rank, r0, r1, codes, scores, mm, evals, coef, _ in parts:
        assert np.allclose(evals, ref_model.eigenvalues, rtol=1e-10, atol=0)
        assert np.allclose(coef, ref_model.coefficients, rtol=0, atol=1e-9)
        rng = ref_scores.max(axis=(1, 2)) - ref_scores.min(axis=(1, 2))
        err = np.abs(scores - ref_scores[:, r0:r1]).max(axis=(1, 2)) / rng
        assert (err <= 1e-6).all(), err
        assert int(np.abs(codes.astype(int) - ref_codes[:, r0:r1].astype(int)).max()) <= 1
        k = scores.shape[0]
        for j in range(k):
            lo, hi = -float(mm[j]), float(mm[k + j])
            assert np.array_equal(codes[j], oracle.linear_to_codes(scores[j].astype(np.float64),
                                                                    lo, hi))
    # the all-reduced record equals the extrema over both shards
    mm0 = parts[0][5]
    allsc = np.concatenate([p[4] for p in parts], axis=1)
    k = allsc.shape[0]
    assert np.array_equal(mm0[:k], -allsc.min(axis=(1, 2)))
    assert np.array_equal(mm0[k:], allsc.max(axis=(1, 2)))
