"""Multi-process (gloo, world_size 2, CPU) test of the row-sharded exchange.

Each rank owns a contiguous row block, routes the training points of its rows,
computes per-class (count, mean, centred M2) records for them and
all-gathers the records -- exactly the exchange CvaPipeline performs over NCCL.
The records are combined in rank order with the parallel-axis rule the K3
kernel applies (csrc/eig.cu: cva_solve_kernel) and must reproduce the
oracle's unsharded scatter.  The [-min, max] record all-reduced with MAX must
equal the whole-image extrema.  (The per-rank reductions here are numpy test
code; on the GPU they are K1 / K4.)
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1612_06457_b200 import route_points, row_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    rng = np.random.default_rng(42)
    b, h, w, c = 6, 40, 30, 3
    cube = rng.normal(size=(b, h, w)) + 3.0
    ys = rng.integers(0, h, 90)
    xs = rng.integers(0, w, 90)
    labels = np.repeat(np.arange(c), 30)
    return cube, xs, ys, labels, c


def _local_records(values, cls, c):
    b = values.shape[0]
    rec = np.zeros((c, 1 + b + b * b))
    for k in range(c):
        pts = values[:, cls == k]
        if pts.shape[1] == 0:
            continue
        m = pts.mean(axis=1)
        d = pts - m[:, None]
        rec[k, 0] = pts.shape[1]
        rec[k, 1:1 + b] = m
        rec[k, 1 + b:] = (d @ d.T).ravel()
    return rec


def _combine(records, b):
    """Parallel-axis combine in rank order (mirror of cva_solve_kernel)."""
    g, c, _ = records.shape
    counts = records[:, :, 0].sum(axis=0)
    means = np.zeros((c, b))
    within = np.zeros((b, b))
    for k in range(c):
        acc = np.zeros(b)
        for r in range(g):
            if records[r, k, 0] > 0:
                acc += records[r, k, 0] * records[r, k, 1:1 + b]
        means[k] = acc / counts[k]
        wk = np.zeros((b, b))
        for r in range(g):
            n = records[r, k, 0]
            wk += records[r, k, 1 + b:].reshape(b, b)
            if n > 0:
                d = records[r, k, 1:1 + b] - means[k]
                wk += n * np.outer(d, d)
        within += wk
    grand = (counts[:, None] * means).sum(axis=0) / counts.sum()
    between = sum(counts[k] * np.outer(means[k] - grand, means[k] - grand) for k in range(c))
    return counts, means, within, between


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cube, xs, ys, labels, c = _data()
    b, h, _ = cube.shape
    r0, r1 = row_bounds(h, world, rank)
    own = route_points(ys, r0, r1 - r0)
    local = cube[:, r0:r1]
    values = oracle.assemble(local, xs[own], ys[own] - r0)
    rec = torch.from_numpy(_local_records(values, labels[own], c)).reshape(-1)
    gathered = torch.empty(world * rec.numel(), dtype=rec.dtype)  # flat, as CvaPipeline
    dist.all_gather_into_tensor(gathered, rec)
    gathered = gathered.reshape(world, c, -1)
    # min/max exchange of a "score plane" = band 0 of the shard
    mm = torch.tensor([-local[0].min(), local[0].max()])
    dist.all_reduce(mm, op=dist.ReduceOp.MAX)
    if rank == 0:
        out.put((gathered.numpy(), mm.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_scatter_and_minmax_exchange():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    records, mm = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cube, xs, ys, labels, c = _data()
    ref = oracle.scatter(oracle.assemble(cube, xs, ys), labels)
    counts, means, within, between = _combine(records, cube.shape[0])
    assert np.array_equal(counts.astype(np.intp), ref["counts"])
    assert np.abs(within - ref["within"]).max() <= 1e-12 * np.abs(ref["within"]).max()
    assert np.abs(between - ref["between"]).max() <= 1e-12 * np.abs(ref["between"]).max()
    assert np.abs(means - ref["class_means"]).max() <= 1e-12 * np.abs(ref["class_means"]).max()
    assert -mm[0] == cube[0].min() and mm[1] == cube[0].max()

