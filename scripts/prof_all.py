"""One pass through every kernel of the path at cfg5 geometry (for ncu):
centre setup (grid, pattern, layout), assembly of 2e7 cfg5 points, a short
solve, evaluation and error report of 1e6 points, and a small QR re-pass."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1806_07884_b200 import api, configs

cfg = configs.CONFIGS["cfg5"]
refs = configs.centres("cfg5")
xy, h = configs.points("cfg5", n=20_000_000)
k = api.KernelSpec(cfg.kernel, cfg.alpha)
with api.Engine(0) as e:
    e.set_centres(refs, k)
    e.set_tile_divisor(9)
    e.set_super_factor(4)
    e.assemble(xy, h)
    c = np.random.default_rng(1).standard_normal(cfg.m)
    e.evaluate(c, xy[:1_000_000])
    e.error_report(c, xy[:1_000_000], h[:1_000_000])
    try:  # solver kernels last (ncu -c truncates the repeated iterations)
        e.solve(max_iter=12)
    except Exception as ex:  # 40 iterations do not converge: only the kernels matter here
        print("solve:", str(ex)[:80])
with api.Engine(0) as e:
    e.set_centres(configs.grid_refs(9, 9), api.KernelSpec(2, 0.25))
    e.least_squares_repass(xy[:9000], h[:9000])
print("prof_all done")
