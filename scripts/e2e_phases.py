"""Wall-clock phases of one public fit (api.fit's calls one by one, synchronised)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1806_07884_b200 import api, configs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cfg = configs.CONFIGS[name]
xy, h = configs.points(name)
refs = configs.centres(name)
k = api.KernelSpec(cfg.kernel, cfg.alpha)
for rep in range(3):
    T = {}
    t = time.perf_counter()
    e = api.Engine(0); e.synchronize(); T["create"] = time.perf_counter() - t
    t = time.perf_counter(); e.set_centres(refs, k); e.synchronize(); T["set_centres"] = time.perf_counter() - t
    t = time.perf_counter(); e.set_poly(False); T["pattern"] = time.perf_counter() - t
    t = time.perf_counter(); e.assemble(xy, h); e.synchronize(); T["assemble"] = time.perf_counter() - t
    lay = e.layout_info()
    b, tl = [float(x) for x in __import__("bench")._asm_times(e)]
    t = time.perf_counter(); hits, dn = e.hits(); T["hits"] = time.perf_counter() - t
    t = time.perf_counter(); c, d = e.solve(); T["solve"] = time.perf_counter() - t
    t = time.perf_counter(); e.close(); T["close"] = time.perf_counter() - t
    print(name, rep, {k2: round(v * 1e3, 1) for k2, v in T.items()}, "total_ms", round(sum(T.values()) * 1e3, 1),
          "layout_build_ms", round(lay["build_ms"], 1), "bin_ms", round(b, 2), "tile_ms", round(tl, 2),
          "solve_dev_ms", round(d["solve_ms"], 1), "its", d["iterations"], flush=True)
