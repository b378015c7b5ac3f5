"""Generates tests/golden/*.npz by running the REFERENCE ITSELF.

Run in a container where /root/reference exists (oracle/_ref/librbfit_ref.so is
compiled from the reference's own kernel/kdtree/coo/data/model sources by
oracle/Makefile).  The fixtures are committed; the GPU box never needs the
reference.  Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as po  # noqa: E402

OUT = Path(__file__).resolve().parent
W30, W31, W33 = 0, 1, 2


def ref_halton(count: int) -> np.ndarray:
    out = np.empty(count * 2)
    po.ref().ref_halton_points(count, 2, out.ctypes.data)
    return out.reshape(-1, 2)


def ref_grid(x0, y0, x1, y1, nx, ny) -> np.ndarray:
    out = np.empty(nx * ny * 2)
    po.ref().ref_uniform_grid_refs(x0, y0, x1, y1, nx, ny, out.ctypes.data)
    return out.reshape(-1, 2)


def kernel_kat():
    rs = np.concatenate([np.linspace(0.0, 1.2, 241), [0.5, 1.0 - 1e-8, np.nextafter(1.0, 0.0)]])
    rows = []
    for fam in (W30, W31, W33):
        for alpha in (0.25, 1.0, 7.5, 10.233267):
            for r in rs:
                rr = r / alpha
                rows.append((fam, alpha, rr, _ref_phi(fam, alpha, rr)))
    arr = np.array(rows, dtype=np.float64)
    np.savez_compressed(OUT / "kernel_kat.npz", table=arr)


def _ref_phi(fam, alpha, r):
    import ctypes as C
    out = C.c_double()
    st = po.ref().ref_kernel_evaluate(fam, alpha, r, C.byref(out))
    assert st == 0
    return out.value


def readme_case():
    # proj/README.md:59-76: 1089 Halton Franke samples, centred by the CLI
    # (rbfit_main.cpp:96), refs = 81-point grid over the centred bbox, phi31 alpha 0.5.
    xy = ref_halton(1089)
    h = np.array([po.ref().ref_franke(x, y) for x, y in xy])
    offset = np.empty(2)
    po.ref().ref_center_cloud(xy.ctypes.data, h.ctypes.data, len(h), offset.ctypes.data)
    lo, hi = xy.min(axis=0), xy.max(axis=0)
    refs = ref_grid(lo[0], lo[1], hi[0], hi[1], 9, 9)
    R = po.ref_build_normal_system(xy, h, refs, W31, 0.5)
    c, _ = po.cholesky_solve(R["b"], R["rhs"])
    f = po.ref_evaluate(refs, c, W31, 0.5, xy)
    er = po.ref_error_report(refs, c, W31, 0.5, xy, h)
    np.savez_compressed(OUT / "readme_case.npz", points=xy, values=h, refs=refs, offset=offset,
                        b=R["b"], rhs=R["rhs"], design_nnz=R["design_nnz"], ref_nnz=R["ref_nnz"],
                        c=c, f=f, mae=er["mean_absolute_error"], deviation=er["deviation_of_error"],
                        rel_pct=er["mean_relative_error_pct"],
                        published_mae=0.002658636306560779,
                        published_deviation=1.0912033239683026e-05, published_design_nnz=88209)


def random_small():
    # Shapes of acceptance C05 (acceptance_main.cpp:138-205): n in [50,500),
    # m in [5,40), refs on data points, phi31 alpha in [0.5, 8); plus phi30/phi33.
    rng = np.random.default_rng(160915)
    data = {}
    for k in range(12):
        n = 50 + int(rng.random() * 450)
        m = 5 + int(rng.random() * 35)
        pts = rng.random((n, 2))
        h = 2.0 * rng.random(n) - 1.0
        refs = pts[[j * n // m for j in range(m)]].copy()
        fam = (W31, W30, W33)[k % 3]
        alpha = 0.5 + 7.5 * rng.random()
        R = po.ref_build_normal_system(pts, h, refs, fam, alpha)
        data.update({f"{k}_points": pts, f"{k}_values": h, f"{k}_refs": refs,
                     f"{k}_family": fam, f"{k}_alpha": alpha, f"{k}_b": R["b"], f"{k}_rhs": R["rhs"],
                     f"{k}_ref_nnz": R["ref_nnz"], f"{k}_design_nnz": R["design_nnz"]})
    data["count"] = 12
    np.savez_compressed(OUT / "random_small.npz", **data)


def cfg1_system():
    # BASELINE config 1 at full size through the reference itself.
    n, m = 100_000, 1_000
    alpha = 1.0 / np.sqrt(30.0 / (np.pi * m))
    xy = ref_halton(n)
    h = np.array([po.ref().ref_franke(x, y) for x, y in xy])
    refs = ref_halton(m)
    R = po.ref_build_normal_system(xy, h, refs, W31, alpha)
    b = R["b"]
    iu, ju = np.nonzero(np.triu(b))
    c, d = po.cholesky_solve(b, R["rhs"])
    f = po.ref_evaluate(refs, c, W31, alpha, xy[:5000])
    er = po.ref_error_report(refs, c, W31, alpha, xy, h)
    np.savez_compressed(OUT / "cfg1_system.npz", alpha=alpha, i=iu.astype(np.uint16),
                        j=ju.astype(np.uint16), v=b[iu, ju], rhs=R["rhs"], ref_nnz=R["ref_nnz"],
                        design_nnz=R["design_nnz"], c=c, f5000=f,
                        mae=er["mean_absolute_error"], deviation=er["deviation_of_error"],
                        points_head=xy[:64], values_head=h[:64])


def poly_cases():
    # The linear-polynomial border (FitOptions::poly; solver.cpp:189-207,
    # 238-262, model.cpp:65-68): README case and random small instances, border
    # blocks from the reference's compiled assemble_submatrix streamed in its
    # own order, c/poly from the restated Cholesky of the bordered system, f
    # from the reference's own evaluate_model with the polynomial.
    g = np.load(OUT / "readme_case.npz")
    xy, h, refs = g["points"], g["values"], g["refs"]
    R = po.ref_build_normal_system(xy, h, refs, W31, 0.5)
    B = po.ref_border(xy, h, refs, W31, 0.5)
    k, rhs = po.bordered_dense(R["b"], R["rhs"], B)
    x, d = po.cholesky_solve(k, rhs)
    m = refs.shape[0]
    c, a = x[:m], x[m:]
    f = po.ref_evaluate_poly(refs, c, a, W31, 0.5, xy)
    mae = float(np.mean(np.abs(f - h)))
    data = {"readme_mae": mae, "readme_points": xy, "readme_values": h, "readme_refs": refs, "readme_atp": B["atp"],
            "readme_ptp": B["ptp"], "readme_pth": B["pth"], "readme_c": c, "readme_a": a, "readme_f": f,
            "readme_ridge": d["ridge_lambda"]}
    rng = np.random.default_rng(20260)
    for t in range(6):
        n = 80 + int(rng.random() * 400)
        mm = 6 + int(rng.random() * 30)
        pts = rng.random((n, 2))
        hv = 2.0 * rng.random(n) - 1.0
        rr = pts[[j * n // mm for j in range(mm)]].copy()
        fam = (W31, W30, W33)[t % 3]
        alpha = 0.75 + 6.0 * rng.random()
        B = po.ref_border(pts, hv, rr, fam, alpha)
        data.update({f"{t}_points": pts, f"{t}_values": hv, f"{t}_refs": rr, f"{t}_family": fam,
                     f"{t}_alpha": alpha, f"{t}_atp": B["atp"], f"{t}_ptp": B["ptp"], f"{t}_pth": B["pth"]})
    data["count"] = 6
    np.savez_compressed(OUT / "poly_cases.npz", **data)


if __name__ == "__main__":
    if "--poly" in sys.argv:
        poly_cases()
    else:
        kernel_kat()
        readme_case()
        random_small()
        cfg1_system()
        poly_cases()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
