"""N > 1 path on CPU: world_size 2 over gloo.

Each rank takes its equal-count spatial slab (rbg_partition_slabs), builds its
partial system (here with the CPU oracle standing in for the per-rank GPU
assembly, which cannot run without a GPU), and the partial [values | rhs |
hits] are summed with the same allreduce helper the bench uses.  The sum must
equal the single-rank system: B and A^T h are sums over points.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as po
        from paper_1806_07884_b200 import configs, distributed

        cfg = configs.CONFIGS["cfg1"]
        xy, h = configs.points("cfg1", n=20_000)
        refs = configs.centres("cfg1")
        bounds, slab = distributed.partition_slabs(xy, world)
        mine = slab == rank
        rp, cols = po.pattern(refs, cfg.alpha)
        vals, rhs, hits = po.assemble(xy[mine], h[mine], refs, 1, cfg.alpha, rp, cols)
        buf = np.concatenate([vals, rhs, hits.astype(np.float64)])
        distributed.allreduce_host([buf])
        if rank == 0:
            fv, fr, fh = po.assemble(xy, h, refs, 1, cfg.alpha, rp, cols)
            nv = len(vals)
            result_q.put({
                "dv": float(np.max(np.abs(buf[:nv] - fv)) / np.max(np.abs(fv))),
                "dr": float(np.max(np.abs(buf[nv:nv + 1000] - fr)) / np.max(np.abs(fr))),
                "hits_equal": bool(np.array_equal(buf[nv + 1000:].astype(np.uint64), fh)),
                "slab_sizes": np.bincount(slab, minlength=world).tolist(),
            })
    finally:
        dist.destroy_process_group()


def test_two_rank_slab_allreduce_equals_single():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = q.get(timeout=10)
    assert res["dv"] < 1e-12 and res["dr"] < 1e-12
    assert res["hits_equal"]
    assert abs(res["slab_sizes"][0] - res["slab_sizes"][1]) <= 1


def test_weak_scaling_shards_are_independent_draws():
    from paper_1806_07884_b200 import configs

    a, _ = configs.points("cfg2", n=1000, seed_offset=0)
    b, _ = configs.points("cfg2", n=1000, seed_offset=1)
    assert not np.array_equal(a, b)
    c, _ = configs.points("cfg5", n=1000, seed_offset=1)
    d, _ = configs.points("cfg5", n=1000, start=configs.CONFIGS["cfg5"].n)
    assert np.array_equal(c, d)  # Halton shard r continues the sequence
