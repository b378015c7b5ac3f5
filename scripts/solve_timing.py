"""Repeated solves of one assembled config (solve_ms per call) -- diagnostics."""
import sys
import time

sys.path.insert(0, ".")
from paper_1806_07884_b200 import api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cfg = configs.CONFIGS[name]
xy, h = configs.points(name)
refs = configs.centres(name)
with api.Engine(0) as eng:
    eng.set_centres(refs, api.KernelSpec(cfg.kernel, cfg.alpha))
    t0 = time.perf_counter()
    eng.assemble(xy, h)
    eng.synchronize()
    print(name, "assemble_s %.3f" % (time.perf_counter() - t0), flush=True)
    for k in range(3):
        t0 = time.perf_counter()
        c, d = eng.solve()
        print(name, "solve wall %.3f" % (time.perf_counter() - t0), "solve_ms %.1f" % d["solve_ms"],
              "its", d["iterations"], flush=True)
