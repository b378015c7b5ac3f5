"""Repeated fresh-context fits (the bench's e2e loop) with per-fit wall time; run with RBG_ALLOC_STATS=1 and
2>&1 to see which fits still reach cudaMalloc / cudaFree."""
import sys, time
sys.path.insert(0, ".")
from paper_1806_07884_b200 import api, configs
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 14
cfg = configs.CONFIGS[name]
xy, h = configs.points(name)
refs = configs.centres(name)
k = api.KernelSpec(cfg.kernel, cfg.alpha)
for rep in range(reps):
    t = time.perf_counter()
    model, r = api.fit(xy, h, refs, k, engine=api.Engine(0))
    print(f"fit {rep}: {1e3 * (time.perf_counter() - t):.1f} ms (solve {r.solve_ms:.1f} ms, {r.iterations} its)", file=sys.stderr, flush=True)
