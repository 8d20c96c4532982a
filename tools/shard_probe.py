"""Per-rank work of the row-sharded cfg-4 path at G = 1/2/4/8, measured on ONE GPU.

Only one B200 is reachable per call, so the NCCL collectives of the sharded path
cannot run here.  This probe measures everything else a rank does at world size
G: it generates rank r's row block of the cfg-4 cube (rows [rH/G, (r+1)H/G)),
routes the training points exactly as a rank would (pipeline.route_points), and
times fit / project / stretch with CUDA events on the launching stream.  The two
collectives are replaced by their local effect: the all_gather by a device copy
of every rank's moment record into its slot (the other ranks' records are
computed beforehand from their own shards, so K3 merges the same G records it
merges under NCCL), the all_reduce(MAX) of 40 bytes by nothing.
The whole-job figure printed is therefore an upper bound that excludes NCCL
latency (two small collectives per step).

usage: python tools/shard_probe.py [--gpus 1 2 4 8] [--steps 20] [--rank last]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class _FakeGroup:
    pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--rank", default="last", help="'last', 'first' or an index")
    args = ap.parse_args()

    import torch

    import paper_1612_06457_b200 as ut
    from paper_1612_06457_b200 import pipeline, synthetic

    torch.cuda.set_device(0)
    cfg = synthetic.CONFIGS[args.config]
    scene = synthetic.make_scene(cfg)
    sizes = {}
    real_ws = pipeline.dist.get_world_size
    def build(g, rank):
        r0, r1 = ut.row_bounds(cfg.height, g, rank)
        stack = synthetic.generate(scene, row0=r0, rows=r1 - r0)
        fake = _FakeGroup()
        pipeline.dist.get_world_size = lambda grp=None: g if grp is fake else real_ws(grp)
        try:
            pipe = ut.CvaPipeline(stack, scene.xs, scene.ys, scene.labels, k=cfg.k, group=fake)
        finally:
            pipeline.dist.get_world_size = real_ws
        return pipe, stack, (r0, r1)

    for g in args.gpus:
        rank = g - 1 if args.rank == "last" else 0 if args.rank == "first" else int(args.rank)
        # the other ranks' moment records, computed for real from their shards
        recs = [None] * g
        for other in range(g):
            if other == rank:
                continue
            p, st, _ = build(g, other)
            if p.n:
                p.fit.moments_from_cube(p.cube, p.xy, p.cls, p.n, p.first_bad, p.pivots)
            else:
                p.fit.local_moments().zero_()
            recs[other] = p.fit.local_moments().clone()
            del p, st
            torch.cuda.empty_cache()
        pipe, stack, (r0, r1) = build(g, rank)
        recs[rank] = torch.zeros_like(pipe.fit.local_moments())
        full = torch.stack(recs)

        def gather(fit, _g=g, _r=rank, _full=full):  # local effect of all_gather_into_tensor
            if _g == 1:
                return
            slots = fit.moments.view(_g, -1)
            slots.copy_(_full)
            slots[_r].copy_(fit.local_moments())

        pipe.gather_moments = gather
        pipe.reduce_minmax = lambda mm: None
        stream = torch.cuda.current_stream()
        for _ in range(args.warmup):
            pipe.run()
        torch.cuda.synchronize()
        pipe.check()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record(stream)
        for e in ev:
            e[0].record(stream)
            pipe.fit.moments_from_cube(pipe.cube, pipe.xy, pipe.cls, pipe.n, pipe.first_bad,
                                       pipe.pivots)
            pipe.gather_moments(pipe.fit)
            e[1].record(stream)
            pipe.fit.solve(pipe.ridge, pipe.k)
            e[2].record(stream)
            pipe.project_kernel()
            e[3].record(stream)
            pipe.stretch_only()
            e[4].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
        pipe.check()
        ms = start.elapsed_time(stop) / args.steps
        split = {k: round(float(np.mean([e[i].elapsed_time(e[i + 1]) for e in ev])), 4)
                 for i, k in enumerate(("moments", "solve", "project", "stretch"))}
        line = {"world": g, "rank": rank, "rows": r1 - r0, "points": int(pipe.n),
                "ms_per_step": round(ms, 4), "split_ms": split,
                "whole_job_mpx_s_excl_nccl": round(cfg.pixels / (ms * 1e-3) / 1e6, 1)}
        sizes[g] = ms
        print(json.dumps(line), flush=True)
        del pipe, stack
        torch.cuda.empty_cache()
    if 1 in sizes:
        for g, ms in sizes.items():
            print(json.dumps({"world": g, "efficiency_excl_nccl": round(sizes[1] / (g * ms), 3)}))


if __name__ == "__main__":
    main()
