"""cfg4 assembled both ways: with the 5 % uniform floor (configs.py) and as BASELINE's pure
4-Gaussian mixture (empty Halton supports -> the fit would need the ridge / re-pass)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1806_07884_b200 import _native, api, configs

cfg = configs.CONFIGS["cfg4"]
refs = configs.centres("cfg4")
dg = _native.datagen()
for floor in (1, 0):
    xy = np.empty((cfg.n, 2))
    dg.dg_mixture_floor(configs.SEEDS["cfg4"], cfg.n, floor, xy.ctypes.data)
    h = np.empty(cfg.n)
    dg.dg_fbm(configs.SEEDS["cfg4"] * 1000 + 1, xy.ctypes.data, cfg.n, h.ctypes.data)
    with api.Engine(0) as eng:
        eng.set_centres(refs, api.KernelSpec(cfg.kernel, cfg.alpha))
        for rep in range(4):
            eng.assemble(xy, h)
            eng.synchronize()
        import bench
        b, t = [float(x) for x in bench._asm_times(eng)]
        hits, dn = eng.hits()
        lay = eng.layout_info()
        line = (f"cfg4 floor={floor}: bin_ms {b:.3f} K3_ms {t:.3f} design_nnz {dn} empty_supports {int((hits == 0).sum())} "
                f"max_hits {int(hits.max())} layout q={lay['sub_div']} S={lay['super_factor']} n_fallback {lay['n_fallback']}")
        try:
            c, d = eng.solve()
            line += f" | solve_ms {d['solve_ms']:.1f} its {d['iterations']} ridge {d['ridge_lambda']:g}"
        except Exception as e:  # noqa: BLE001
            line += f" | solve: {str(e)[:120]}"
        print(line, flush=True)
