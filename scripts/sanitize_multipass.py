"""Multi-pass sub-tiles (panels, phi scratch, chunks, direct-mode flush with and without a staged
slot map) at small size for compute-sanitizer (memcheck / racecheck / initcheck)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1806_07884_b200 import api, configs

for dim, fam, m, per, n, div in ((2, 1, 400, 55, 30000, 2), (3, 3, 400, 60, 20000, 2), (3, 2, 300, 70, 12000, 2),
                                 (3, 2, 300, 40, 12000, 0)):
    refs = configs.halton(1, m, dim)
    alpha = configs._alpha_for(m, per, dim)
    rng = np.random.default_rng(7 + dim + fam)
    pts = rng.random((n, dim))
    h = rng.standard_normal(n)
    with api.Engine(0) as e:
        e.set_centres(refs, api.KernelSpec(fam, alpha))
        if div:
            e.set_tile_divisor(div)
        e.assemble(pts, h)
        s = e.system()
        lay = e.layout_info()
        print(dim, fam, lay["sub_div"], lay["max_sub_centres"], float(s["values"].sum()), flush=True)
print("sanitize multipass done")
