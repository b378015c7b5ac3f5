"""A small pass through every kernel family for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1806_07884_b200 import api, configs

rng = np.random.default_rng(3)
for dim, fam, m, n in ((2, "wendland-3-1", 400, 12000), (3, "wendland-3-2", 300, 12000)):
    side = int(round(m ** (1.0 / dim)))
    g = (np.stack(np.meshgrid(*[np.arange(side)] * dim, indexing="ij"), -1).reshape(-1, dim) + 0.5) / side
    refs = np.ascontiguousarray(g + (rng.random(g.shape) - 0.5) * 0.3 / side)
    mm = refs.shape[0]
    r = (25.0 / (np.pi * mm)) ** 0.5 if dim == 2 else (30.0 / (mm * 4.0 * np.pi / 3.0)) ** (1.0 / 3.0)
    pts = rng.random((n, dim))
    h = np.sin(3 * pts[:, 0]) + pts[:, 1]
    with api.Engine(0) as e:
        e.set_centres(refs, api.KernelSpec(fam, 1.0 / r))
        e.assemble(pts, h)
        c, d = e.solve()
        c2, d2 = e.solve(precond="jacobi")
        if dim == 2:
            c3, d3 = e.solve(method="band")
        f = e.evaluate(c, pts[:2000])
        rep = e.error_report(c, pts, h)
        e.set_poly(True)
        e.assemble(pts, h)
        c4, d4 = e.solve()
        print(dim, d["iterations"], d2["iterations"], d4["iterations"], rep["mean_absolute_error"], flush=True)
print("sanitize pass done")
