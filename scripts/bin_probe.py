"""Would a two-pass binning pay?  Pass B (the fine scatter) = today's binning run on input that is already
partitioned into P spatial stripes (records of a stripe contiguous, random order inside): measure it."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_1806_07884_b200 import api, configs
cfg = configs.CONFIGS["cfg5"]
xy, h = configs.points("cfg5")
refs = configs.centres("cfg5")
k = api.KernelSpec(cfg.kernel, cfg.alpha)
with api.Engine(0) as e:
    e.set_centres(refs, k)
    def run(tag, a, b):
        for _ in range(3):
            e.assemble(a, b); e.synchronize()
        bm, tm = [float(x) for x in bench._asm_times(e)]
        print(f"{tag}: bin_ms {bm:.2f} K3_ms {tm:.2f}", flush=True)
    run("input order (Halton)", xy, h)
    for P in (64, 256, 1024):
        t = time.time()
        stripe = np.minimum((xy[:, 1] * P).astype(np.int32), P - 1)
        order = np.argsort(stripe, kind="stable")
        xs, hs = np.ascontiguousarray(xy[order]), np.ascontiguousarray(h[order])
        print(f"  (host partition into {P} stripes took {time.time() - t:.0f} s)", flush=True)
        run(f"{P} y-stripes", xs, hs)
        del xs, hs, order, stripe
