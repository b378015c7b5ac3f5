"""Evaluation / error-report timing at a config's geometry (device time of rbg_evaluate_device is not exposed:
wall time of evaluate on host arrays, which includes the query upload and the result download)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1806_07884_b200 import api, configs
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
nq = int(float(sys.argv[2])) if len(sys.argv) > 2 else 20_000_000
cfg = configs.CONFIGS[name]
xy, h = configs.points(name, n=nq)
refs = configs.centres(name)
c = np.random.default_rng(1).standard_normal(cfg.m)
with api.Engine(0) as e:
    e.set_centres(refs, api.KernelSpec(cfg.kernel, cfg.alpha))
    for rep in range(3):
        t = time.perf_counter(); f = e.evaluate(c, xy); dt = time.perf_counter() - t
        t = time.perf_counter(); r = e.error_report(c, xy, h); dr = time.perf_counter() - t
        print(name, nq, "evaluate_ms %.1f" % (dt * 1e3), "error_report_ms %.1f" % (dr * 1e3), flush=True)
