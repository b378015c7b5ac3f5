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
    """Each rank takes its slab exactly as bench.py does (configs.slab_points:
    dyadic Halton slabs for cfg5, rbg_partition_slabs for cfg2), assembles it
    (the CPU oracle standing in for the per-rank GPU assembly) and the partial
    [values | rhs | hits] are summed with the bench's gloo/NCCL helper."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as po
        from paper_1806_07884_b200 import configs, distributed

        out = {}
        for name, n, refs in (("cfg5", 60_000, configs.grid_refs(60, 60)), ("cfg2", 20_000, None)):
            cfg = configs.CONFIGS[name]
            refs = configs.centres(name) if refs is None else refs
            alpha = cfg.alpha if name == "cfg2" else 60.0
            xy, h = configs.slab_points(name, rank, world, n=n)
            rp, cols = po.pattern(refs, alpha)
            vals, rhs, hits = po.assemble(xy, h, refs, 1, alpha, rp, cols)
            buf = np.concatenate([vals, rhs, hits.astype(np.float64)])
            distributed.allreduce_host([buf])
            counts = np.array([len(h)], dtype=np.float64)
            distributed.allreduce_host([counts])
            if rank == 0:
                fxy, fh = configs.points(name, n=n)
                fv, fr, fhits = po.assemble(fxy, fh, refs, 1, alpha, rp, cols)
                nv, m = len(vals), len(refs)
                out[name] = {
                    "dv": float(np.max(np.abs(buf[:nv] - fv)) / np.max(np.abs(fv))),
                    "dr": float(np.max(np.abs(buf[nv:nv + m] - fr)) / np.max(np.abs(fr))),
                    "hits_equal": bool(np.array_equal(buf[nv + m:].astype(np.uint64), fhits)),
                    "total": int(counts[0]), "n": n, "mine": len(h),
                    "x_range": [float(xy[:, 0].min()), float(xy[:, 0].max())],
                }
        if rank == 0:
            result_q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_slab_allreduce_equals_single(world):
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
    for name, r in res.items():
        assert r["dv"] < 1e-12 and r["dr"] < 1e-12, (name, r)
        assert r["hits_equal"], name
        assert r["total"] == r["n"], name  # the slabs partition the one point set
        assert abs(r["mine"] - r["n"] / world) <= 1, name  # equal counts
    lo, hi = res["cfg5"]["x_range"]
    assert lo >= 0.0 and hi < 1.0 / world  # rank 0 owns the slab x in [0, 1/W)


def test_dyadic_halton_slabs_match_partition_slabs():
    """For the Halton configs the directly generated dyadic slabs are the
    equal-count x-slabs rbg_partition_slabs finds on the whole set."""
    from paper_1806_07884_b200 import configs, distributed
    n = 1 << 14
    xy, _ = configs.points("cfg5", n=n)
    for world in (2, 4, 8):
        bounds, slab = distributed.partition_slabs(xy, world)
        for r in range(world):
            mine, _ = configs.slab_points("cfg5", r, world, n=n)
            ref = xy[slab == r]
            assert abs(len(mine) - len(ref)) <= 1
            common = len(set(map(tuple, mine)) & set(map(tuple, ref)))
            assert common >= min(len(mine), len(ref)) - 1
