"""GPU parity: the CUDA path through the C ABI against the CPU oracle and the
reference's own golden outputs.

Tolerances (north_star): pattern bit-exact; A^T A / A^T h within 1e-10 using
the reference's scale-normalised metric max|d|/max|ref| (acceptance_main.cpp:
118-125), B additionally entry by entry (`entrywise`: scaled by its diagonal
pair, and plain elementwise for every entry above 1e-6 of that scale);
hits / design_nnz exact; evaluation bit-exact for the same c; c within 1e-8.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_1806_07884_b200 import api, configs

pytestmark = pytest.mark.gpu

TOL_SYS = 1e-10
TOL_C = 1e-8


def scaled(a, b):
    s = np.max(np.abs(b)) if b.size else 0.0
    return float(np.max(np.abs(a - b)) / s) if s > 0 else float(np.max(np.abs(a - b), initial=0.0))


def entrywise(a, b, rp, cols):
    """Entry-by-entry metrics of the upper CSR values a against b (the oracle's):
    (max |d_ij| / sqrt(B_ii B_jj), max |d_ij| / |b_ij| over the entries with
    |b_ij| >= 1e-6 sqrt(B_ii B_jj)).  The first is the SPD-natural scaling
    (|B_ij| <= sqrt(B_ii B_jj)), tighter than the reference's global max|ref|;
    the second is plain elementwise agreement wherever an entry is not made of
    near-edge phi values only: the assembly's sqrt is one ulp off the IEEE
    root for ~0.2 % of the distances and its (1 - alpha r) is one FMA, i.e.
    u = 1 - t moves by <= 1e-16, which is a 1e-16 / u relative change of phi
    and only visible in entries below 1e-6 of their diagonal scale."""
    rp = rp.astype(np.int64)
    diag = b[rp[:-1]]
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    sc = np.sqrt(diag[rows] * diag[cols.astype(np.int64)])
    d = np.abs(a - b)
    assert np.all(d[sc == 0] == 0)
    pos = sc > 0
    by_diag = float(np.max(d[pos] / sc[pos], initial=0.0))
    big = pos & (np.abs(b) >= 1e-6 * sc)
    rel = float(np.max(d[big] / np.abs(b[big]), initial=0.0))
    return by_diag, rel


@pytest.fixture(scope="module")
def eng():
    e = api.Engine(0)
    yield e
    e.close()


def run_and_compare(eng, pts, h, refs, family, alpha, accumulate_slabs=1):
    k = api.KernelSpec(family, alpha)
    eng.set_centres(refs, k)
    if accumulate_slabs == 1:
        eng.assemble(pts, h)
    else:
        parts = np.array_split(np.arange(len(h)), accumulate_slabs)
        for i, idx in enumerate(parts):
            eng.assemble(pts[idx], h[idx], accumulate=i > 0)
    rp, cols = eng.pattern()
    orp, ocols = po.pattern(refs, alpha)
    assert np.array_equal(rp, orp), "row_ptr differs"
    assert np.array_equal(cols, ocols), "cols differ"
    s = eng.system()
    ov, orhs, ohits = po.assemble(pts, h, refs, k.family, alpha, orp, ocols)
    assert scaled(s["values"], ov) < TOL_SYS
    assert max(entrywise(s["values"], ov, orp, ocols)) < TOL_SYS
    assert scaled(s["rhs"], orhs) < TOL_SYS
    assert np.array_equal(s["hits"].astype(np.uint64), ohits)
    assert s["design_nnz"] == int(ohits.sum())
    return s, (orp, ocols, ov, orhs, ohits)


# ------------------------------------------------------------- golden pins
def test_readme_case_vs_reference(eng, golden):
    g = golden("readme_case")
    s, (rp, cols, ov, orhs, _) = run_and_compare(eng, g["points"], g["values"], g["refs"], 1, 0.5)
    dense = api.SparseNormalSystem(81, rp, cols, s["values"], s["rhs"], np.array([]), 0).to_dense()
    assert scaled(dense, g["b"]) < TOL_SYS and scaled(s["rhs"], g["rhs"]) < TOL_SYS
    assert s["design_nnz"] == int(g["published_design_nnz"]) == 88209
    f = eng.evaluate(g["c"], g["points"])
    assert np.array_equal(f, g["f"])  # bitwise vs the reference's evaluate_model


def test_small_instances_vs_reference(eng, golden):
    g = golden("random_small")
    for k in range(int(g["count"])):
        s, (rp, cols, *_r) = run_and_compare(eng, g[f"{k}_points"], g[f"{k}_values"], g[f"{k}_refs"],
                                             int(g[f"{k}_family"]), float(g[f"{k}_alpha"]))
        m = len(g[f"{k}_refs"])
        dense = api.SparseNormalSystem(m, rp, cols, s["values"], s["rhs"], np.array([]), 0).to_dense()
        assert scaled(dense, g[f"{k}_b"]) < TOL_SYS
        assert np.array_equal(s["hits"].astype(np.uint32), g[f"{k}_ref_nnz"])


def test_cfg1_full_vs_reference(eng, golden):
    g = golden("cfg1_system")
    xy, h = configs.points("cfg1")
    refs = configs.centres("cfg1")
    s, (rp, cols, ov, orhs, _) = run_and_compare(eng, xy, h, refs, 1, float(g["alpha"]))
    assert len(cols) == 50898 and s["design_nnz"] == int(g["design_nnz"])
    c, diag = eng.solve()
    assert diag["ridge_lambda"] == 0.0 and diag["rel_residual"] < 1e-11
    assert np.max(np.abs(c - g["c"])) / np.max(np.abs(g["c"])) < TOL_C  # vs reference-path Cholesky
    f = eng.evaluate(c, xy[:5000])
    assert np.array_equal(f, po.evaluate(refs, c, 1, float(g["alpha"]), xy[:5000]))
    rep = eng.error_report(c, xy, h)
    assert rep["mean_absolute_error"] == pytest.approx(float(g["mae"]), rel=1e-6)


# ------------------------------------------------------------ configs
@pytest.mark.parametrize("name,n", [("cfg2", 100_000), ("cfg3", 60_000), ("cfg4", 200_000)])
def test_config_subsamples(eng, name, n):
    cfg = configs.CONFIGS[name]
    xy, h = configs.points(name, n=n)
    refs = configs.centres(name)
    if name == "cfg3":
        refs = refs[:6000]  # keeps the oracle's run in seconds; same density class
    run_and_compare(eng, xy, h, refs, api.KERNELS[cfg.kernel], cfg.alpha if name != "cfg3" else cfg.alpha / 2)


@pytest.mark.parametrize("dim,family,m,per_support,n,divisor", [
    (2, 1, 400, 55, 200_000, 2),    # 2-D, 8-block sub-tiles of ~2000 points: panels 4 + 4, shared accumulator
    (3, 3, 400, 60, 100_000, 2),    # 3-D direct mode, ~14-block sub-tiles of ~600 points: panels 5 + 5 + 4
    (3, 2, 300, 70, 40_000, 2),     # 3-D, ~20 blocks: four panels, slot map too large to stage
])
def test_multipass_subtiles_in_chunks(dim, family, m, per_support, n, divisor):
    """Sub-tiles beyond 56 centres are assembled in panels with phi cached in the per-worker
    scratch, and beyond 128 points in chunks of the scratch's capacity (rbg_asm.cuh
    kChunkSteps): dense sub-tiles forced through rbg_set_tile_divisor, every chunk, panel
    shape and flush path against the oracle."""
    refs = configs.halton(1, m, dim)
    alpha = configs._alpha_for(m, per_support, dim)
    rng = np.random.default_rng(100 + dim + family)
    pts = rng.random((n, dim))
    h = rng.standard_normal(n)
    with api.Engine(0) as e:
        e.set_centres(refs, api.KernelSpec(family, alpha))
        e.set_tile_divisor(divisor)
        e.assemble(pts, h)
        lay = e.layout_info()
        per_sub = n * lay["sub_edge"] ** dim  # uniform points in the unit cube
        assert lay["max_sub_centres"] > 56 and per_sub > 128 and lay["n_fallback"] == 0, lay
        rp, cols = e.pattern()
        s = e.system()
    orp, ocols = po.pattern(refs, alpha)
    assert np.array_equal(rp, orp) and np.array_equal(cols, ocols)
    ov, orhs, ohits = po.assemble(pts, h, refs, family, alpha, orp, ocols)
    assert np.array_equal(s["hits"].astype(np.uint64), ohits)
    assert scaled(s["values"], ov) < TOL_SYS and max(entrywise(s["values"], ov, orp, ocols)) < TOL_SYS
    assert scaled(s["rhs"], orhs) < TOL_SYS


def test_slab_accumulation_equals_single(eng):
    xy, h = configs.points("cfg2", n=50_000)
    refs = configs.centres("cfg2")
    run_and_compare(eng, xy, h, refs, 1, configs.CONFIGS["cfg2"].alpha, accumulate_slabs=4)


def test_fallback_tiles_dense_centres(eng):
    # super-tile centre lists above the largest accumulator class take the slow path
    rng = np.random.default_rng(11)
    refs = rng.random((400, 2)) * 0.2
    pts = rng.random((3000, 2)) * 0.3
    h = rng.standard_normal(3000)
    eng.set_centres(refs, api.KernelSpec("wendland-3-1", 8.0))
    run_and_compare(eng, pts, h, refs, 1, 8.0)
    assert eng.layout_info()["n_fallback"] > 0


@pytest.mark.parametrize("family", [0, 1, 2, 3])
def test_all_families_3d_and_2d(eng, family):
    rng = np.random.default_rng(family)
    for dim in (2, 3):
        refs = rng.random((300, dim))
        pts = rng.random((5000, dim))
        h = rng.standard_normal(5000)
        run_and_compare(eng, pts, h, refs, family, 4.0)


# ------------------------------------------------------------- edges
def test_edge_cases(eng):
    k = api.KernelSpec("wendland-3-0", 1.0)
    # one point, one centre: fit degenerates to c = 5 (test_solver.cpp:353-367)
    eng.set_centres(np.array([[0.0, 0.0]]), k)
    eng.assemble(np.array([[0.0, 0.0]]), np.array([5.0]))
    c, _ = eng.solve()
    assert c[0] == pytest.approx(5.0, rel=1e-14)
    assert eng.evaluate(c, np.array([[0.0, 0.0]]))[0] == pytest.approx(5.0, rel=1e-14)
    # empty input, points outside every support, duplicates
    refs = np.array([[0.5, 0.5], [0.6, 0.5]])
    eng.set_centres(refs, api.KernelSpec("wendland-3-1", 5.0))
    eng.assemble(np.zeros((0, 2)), np.zeros(0))
    assert not eng.system()["values"].any()
    far = np.array([[10.0, 10.0], [-5.0, 0.5]])
    pts = np.vstack([far, np.repeat([[0.55, 0.5]], 7, axis=0)])
    h = np.arange(9.0)
    run_and_compare(eng, pts, h, refs, 1, 5.0)
    # strict support boundary: (3,4) at distance 5 with radius 5 is excluded (test_kdtree.cpp:28-38)
    eng.set_centres(np.array([[0.0, 0.0]]), api.KernelSpec("wendland-3-0", 0.2))
    eng.assemble(np.array([[3.0, 4.0], [0.0, 0.0]]), np.array([1.0, 1.0]))
    assert eng.system()["hits"].tolist() == [1.0]


def test_invalid_inputs(eng):
    with pytest.raises(ValueError):
        eng.set_centres(np.array([[0.0, np.nan]]), api.KernelSpec("wendland-3-1", 1.0))
    eng.set_centres(np.array([[0.0, 0.0]]), api.KernelSpec("wendland-3-1", 1.0))
    with pytest.raises(ValueError, match="index 1"):
        eng.assemble(np.array([[0.0, 0.0], [np.inf, 0.0]]), np.zeros(2))


def test_empty_support_ridge_and_pivot_message(eng):
    rng = np.random.default_rng(5)
    pts = rng.random((60, 2))
    h = 2.0 * rng.random(60) - 1.0
    refs = np.array([[0.1, 0.1], [0.9, 0.1], [0.1, 0.9], [0.9, 0.9], [50.0, 50.0]])
    eng.set_centres(refs, api.KernelSpec("wendland-3-0", 1.0))
    eng.assemble(pts, h)
    assert eng.system()["hits"][4] == 0
    c, diag = eng.solve()
    assert diag["ridge_lambda"] > 0.0 and abs(c[4]) < 1e-8
    eng.set_system(np.zeros(eng.pattern_info()["nnz_upper"]), np.ones(5))
    with pytest.raises(RuntimeError, match="pivot"):
        eng.solve()


def test_layout_follows_the_point_count(eng):
    """The assembly tiling is chosen from the point density: a small first call must not pin the
    layout of a later, much larger one (rbg::ensure_layout), and results do not depend on it."""
    cfg = configs.CONFIGS["cfg2"]
    xy, h = configs.points("cfg2", n=400_000)
    refs = configs.centres("cfg2")
    k = api.KernelSpec(cfg.kernel, cfg.alpha)
    with api.Engine(0) as fresh:
        fresh.set_centres(refs, k)
        fresh.assemble(xy, h)
        want = fresh.layout_info()
        ref_sys = fresh.system()
    eng.set_centres(refs, k)
    eng.assemble(xy[:500], h[:500])
    small = eng.layout_info()
    eng.assemble(xy, h)
    got = eng.layout_info()
    assert (got["sub_div"], got["super_factor"]) == (want["sub_div"], want["super_factor"]), (small, got, want)
    s = eng.system()
    assert scaled(s["values"], ref_sys["values"]) < TOL_SYS and np.array_equal(s["hits"], ref_sys["hits"])


def test_solver_methods_and_preconditioners_agree(eng):
    """rbg_solve_options::method / precond: the FSAI-preconditioned CG (default), point-Jacobi CG
    and the banded LLT (the reference's factorisation, solver.cpp:289-330) solve the same assembled
    system to the same c (<= 1e-8), in 2-D and 3-D; FSAI needs an order of magnitude fewer
    iterations than point Jacobi."""
    rng = np.random.default_rng(11)
    for dim, side, n, fam, per_support in ((2, 30, 60_000, "wendland-3-1", 25.0), (3, 9, 60_000, "wendland-3-2", 30.0)):
        # jittered grid centres (random ones cluster: point Jacobi then needs > 20000 iterations)
        g = (np.stack(np.meshgrid(*[np.arange(side)] * dim, indexing="ij"), -1).reshape(-1, dim) + 0.5) / side
        refs = np.ascontiguousarray(g + (rng.random(g.shape) - 0.5) * 0.3 / side)
        m = refs.shape[0]
        r = (per_support / (np.pi * m)) ** 0.5 if dim == 2 else (per_support / (m * 4.0 * np.pi / 3.0)) ** (1.0 / 3.0)
        alpha = 1.0 / r
        pts = rng.random((n, dim))
        h = np.sin(3.0 * pts[:, 0]) + pts[:, 1] ** 2
        eng.set_centres(refs, api.KernelSpec(fam, alpha))
        eng.assemble(pts, h)
        c_f, d_f = eng.solve()
        c_j, d_j = eng.solve(precond="jacobi")
        assert d_f["ridge_lambda"] == 0.0 and d_j["ridge_lambda"] == 0.0
        assert d_f["rel_residual"] < 1e-11 and d_j["rel_residual"] < 1e-11
        assert 0 < d_f["iterations"] * 5 < d_j["iterations"], (d_f["iterations"], d_j["iterations"])
        scale = np.max(np.abs(c_j))
        assert np.max(np.abs(c_f - c_j)) / scale < TOL_C
        if dim == 2:
            c_b, d_b = eng.solve(method="band")
            assert d_b["iterations"] == 0
            assert np.max(np.abs(c_f - c_b)) / scale < TOL_C
        rp, cols = eng.pattern()
        s = eng.system()
        oc, _ = po.cholesky_solve(po.densify(rp, cols, s["values"]), s["rhs"])
        assert np.max(np.abs(c_f - oc)) / np.max(np.abs(oc)) < TOL_C


# ------------------------------------------------- full-size properties
def test_cfg2_full_size_properties(eng):
    """Size-independent checks at BASELINE config 2's full size:
    x^T B x == ||A x||^2 (A x evaluated by the eval kernel), rhs == B c for
    h = A c, and the solve recovers c."""
    cfg = configs.CONFIGS["cfg2"]
    xy, _ = configs.points("cfg2")
    refs = configs.centres("cfg2")
    k = api.KernelSpec(cfg.kernel, cfg.alpha)
    eng.set_centres(refs, k)
    rng = np.random.default_rng(7)
    c_true = rng.standard_normal(cfg.m)
    h = eng.evaluate(c_true, xy)  # h = A c_true exactly representable input
    eng.assemble(xy, h)
    s = eng.system()
    rp, cols = eng.pattern()
    B = api.SparseNormalSystem(cfg.m, rp, cols, s["values"], s["rhs"], np.array([]), 0)
    import scipy.sparse as sp
    rows = np.repeat(np.arange(cfg.m), np.diff(rp.astype(np.int64)))
    U = sp.csr_matrix((s["values"], (rows, cols.astype(np.int64))), shape=(cfg.m, cfg.m))
    Bs = U + sp.triu(U, 1).T
    x = rng.standard_normal(cfg.m)
    ax = eng.evaluate(x, xy)
    assert float(x @ (Bs @ x)) == pytest.approx(float(ax @ ax), rel=1e-10)
    assert scaled(Bs @ c_true, s["rhs"]) < 1e-10
    assert s["design_nnz"] == int(s["hits"].sum())
    c, diag = eng.solve()
    assert np.max(np.abs(c - c_true)) / np.max(np.abs(c_true)) < 1e-7
    del B


@pytest.mark.parametrize("family", [0, 1, 2, 3])
def test_assembly_phi_inclusion_exact_and_value_close(eng, family):
    """phi_k3 (the assembly kernel's phi): inclusion bit-exact against the
    reference rule (kdtree.cpp:64,74 + kernel.hpp:45-46) over distances of
    every magnitude incl. 0, subnormals and the threshold's neighbourhood;
    values bitwise the reference's for wendland-3-0/3-1, within a few ulp
    for 3-3/3-2 (FMA-contracted polynomial, no cancellation)."""
    for alpha in (0.25, 1.0, 10.2333, 280.2496, 1e6):
        r = eng.phi_selftest(family, alpha, 1 << 24, 12345)
        assert r["mismatches"] == 0, (alpha, r)
        if family in (0, 1):
            assert r["max_rel"] == 0.0 and r["max_abs"] == 0.0, (alpha, r)
        else:
            assert r["max_rel"] < 4e-15, (alpha, r)


@pytest.mark.parametrize("family", [0, 1, 2, 3])
def test_assembly_fast_phi_inclusion_exact_and_value_within_ulps(eng, family):
    """phi_k3<FAM, true> (what the assembly's k-loop evaluates): the same bit-exact
    inclusion; values within a few ulp of the reference's away from the support's edge and
    within 4e-15 absolutely everywhere (phi <= 3: a few ulp; measured 2.7e-15, relative 1.3e-14)."""
    for alpha in (0.25, 1.0, 10.2333, 280.2496, 1e6):
        r = eng.phi_selftest(family, alpha, 1 << 24, 54321, fast=True)
        assert r["mismatches"] == 0, (alpha, r)
        assert r["max_abs"] < 4e-15 and r["max_rel"] < 1e-12, (alpha, r)


@pytest.mark.parametrize("div,sup", [(2.0, 1), (3.0, 2), (5.0, 3), (6.0, 4), (8.0, 2), (12.0, 5)])
def test_layout_does_not_change_results(eng, div, sup):
    # sub-tile divisor / super-tile factor are performance knobs only
    cfg = configs.CONFIGS["cfg1"]
    xy, h = configs.points("cfg1", n=30_000)
    refs = configs.centres("cfg1")
    eng.set_tile_divisor(div)
    eng.set_super_factor(sup)
    try:
        run_and_compare(eng, xy, h, refs, 1, cfg.alpha)
        info = eng.layout_info()
        assert info["built"] and info["sub_div"] == int(div) and info["super_factor"] == sup
    finally:
        eng.set_tile_divisor(0)
        eng.set_super_factor(0)


# ------------------------------------------------ linear-polynomial border
def _border_close(b, ref):
    for k in ("atp", "ptp", "pth"):
        assert scaled(b[k], ref[k]) < TOL_SYS, k


def test_border_vs_reference(eng, golden):
    """A^T P, P^T P, P^T h (solver.cpp:189-207, 238-262) on the GPU against the
    reference's own border on the committed instances (A^T P is summed in a
    different order, hence the 1e-10 scaled tolerance)."""
    g = golden("poly_cases")
    try:
        for t in range(int(g["count"])):
            k = api.KernelSpec(int(g[f"{t}_family"]), float(g[f"{t}_alpha"]))
            eng.set_centres(g[f"{t}_refs"], k)
            eng.set_poly(True)
            eng.assemble(g[f"{t}_points"], g[f"{t}_values"])
            _border_close(eng.border(), {kk: g[f"{t}_{kk}"] for kk in ("atp", "ptp", "pth")})
    finally:
        eng.set_poly(False)


def test_bordered_fit_readme_vs_reference(eng, golden):
    """README case with --poly (alpha = 0.5: the bordered system is too ill
    conditioned for a 1e-8 weight comparison with any iterative solver, like
    the plain README case): the border blocks within 1e-10 of the reference's,
    evaluation with the polynomial bitwise equal to the reference's
    evaluate_model for the same weights, and the GPU fit's MAE within 1 % of
    the reference-path (restated Cholesky) fit's."""
    g = golden("poly_cases")
    k = api.KernelSpec(1, 0.5)
    try:
        eng.set_centres(g["readme_refs"], k)
        eng.set_poly(True)
        eng.assemble(g["readme_points"], g["readme_values"])
        _border_close(eng.border(), {kk: g[f"readme_{kk}"] for kk in ("atp", "ptp", "pth")})
        eng.set_model_poly(g["readme_a"])
        f = eng.evaluate(g["readme_c"], g["readme_points"])
        assert np.array_equal(f, g["readme_f"])
        model, rep = api.fit(g["readme_points"], g["readme_values"], g["readme_refs"], k, engine=eng, poly=True)
        er = api.error_report(model, g["readme_points"], g["readme_values"], engine=eng)
        assert er["mean_absolute_error"] == pytest.approx(float(g["readme_mae"]), rel=1e-2)
    finally:
        eng.set_model_poly(None)
        eng.set_poly(False)


def test_bordered_solve_vs_dense_cholesky(eng, golden):
    """c and the polynomial of the bordered solve within 1e-8 of the restated
    dense Cholesky (solver.cpp:289-330 with side = m + 3) on the committed
    well-conditioned instances."""
    g = golden("poly_cases")
    try:
        for t in range(int(g["count"])):
            pts, h, refs = g[f"{t}_points"], g[f"{t}_values"], g[f"{t}_refs"]
            fam, alpha = int(g[f"{t}_family"]), float(g[f"{t}_alpha"])
            k = api.KernelSpec(fam, alpha)
            eng.set_centres(refs, k)
            eng.set_poly(True)
            eng.assemble(pts, h)
            c, diag = eng.solve()
            a = eng.poly_solution()
            rp, cols = po.pattern(refs, alpha)
            v, rhs, _ = po.assemble(pts, h, refs, fam, alpha, rp, cols)
            kd, rd = po.bordered_dense(po.densify(rp, cols, v), rhs,
                                       {kk: g[f"{t}_{kk}"] for kk in ("atp", "ptp", "pth")})
            if np.linalg.cond(kd) > 1e7:
                continue  # 1e-12 residual does not pin 1e-8 weights there
            x, d = po.cholesky_solve(kd, rd)
            if d["ridge_lambda"] != 0.0:
                continue
            got = np.concatenate([c, a])
            assert np.max(np.abs(got - x)) / np.max(np.abs(x)) < TOL_C, t
    finally:
        eng.set_poly(False)


def test_poly_affine_reproduction(eng):
    """acceptance C06 (acceptance_main.cpp:207-225): h = 2x + 3y + 1, 4x4 grid of
    references, phi31 alpha 1, with the border -> MAE < 1e-8 through fit +
    error_report (2-D), and the 3-D analogue with P = [x, y, z, 1]."""
    rng = np.random.default_rng(77)
    pts = rng.random((200, 2))
    h = 2.0 * pts[:, 0] + 3.0 * pts[:, 1] + 1.0
    gx, gy = np.meshgrid(np.linspace(0, 1, 4), np.linspace(0, 1, 4))
    refs = np.stack([gx.ravel(), gy.ravel()], axis=1)
    k = api.KernelSpec(1, 1.0)
    try:
        model, _ = api.fit(pts, h, refs, k, engine=eng, poly=True)
        rep = api.error_report(model, pts, h, engine=eng)
        assert rep["mean_absolute_error"] < 1e-8
        assert np.allclose(model.poly, [2.0, 3.0, 1.0], atol=1e-6)
        p3 = rng.random((600, 3))
        h3 = 1.5 * p3[:, 0] - 0.5 * p3[:, 1] + 2.0 * p3[:, 2] + 0.25
        g3 = np.stack(np.meshgrid(*[np.linspace(0, 1, 3)] * 3), axis=-1).reshape(-1, 3)
        model3, _ = api.fit(p3, h3, g3, api.KernelSpec("wendland-3-2", 1.2), engine=eng, poly=True)
        rep3 = api.error_report(model3, p3, h3, engine=eng)
        assert rep3["mean_absolute_error"] < 1e-8
    finally:
        eng.set_model_poly(None)
        eng.set_poly(False)


def test_border_slab_allreduce_sum(eng):
    """The border is part of the all-reduced system buffer: assembling two
    slabs with accumulate gives the single-pass border."""
    rng = np.random.default_rng(5)
    pts = rng.random((3000, 2))
    h = np.cos(3 * pts[:, 0]) * pts[:, 1]
    refs = rng.random((120, 2))
    k = api.KernelSpec(1, 6.0)
    try:
        eng.set_centres(refs, k)
        eng.set_poly(True)
        eng.assemble(pts, h)
        one = eng.border()
        _, count = eng.system_device()
        assert count == eng.pattern_info()["nnz_upper"] + 2 * 120 + 3 * 120 + 9 + 3
        eng.assemble(pts[:1700], h[:1700])
        eng.assemble(pts[1700:], h[1700:], accumulate=True)
        two = eng.border()
        _border_close(two, one)
        _border_close(one, po.border(pts, h, refs, 1, 6.0))
    finally:
        eng.set_poly(False)


_SUBPROC = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import pyoracle as po
from paper_1806_07884_b200 import api, configs
cfg = configs.CONFIGS["cfg2"]
xy, h = configs.points("cfg2", n=1_200_000)
refs = configs.centres("cfg2")
k = api.KernelSpec(cfg.kernel, cfg.alpha)
with api.Engine(0) as eng:
    eng.set_centres(refs, k)
    pxy, ph = torch.from_numpy(xy).pin_memory(), torch.from_numpy(h).pin_memory()
    eng.assemble_ptr(pxy.data_ptr(), ph.data_ptr(), len(h), validate=True)
    s = eng.system()
    c, d = eng.solve()
rp, cols = po.pattern(refs, cfg.alpha)
ov, orhs, ohits = po.assemble(xy, h, refs, k.family, cfg.alpha, rp, cols)
den = np.max(np.abs(ov))
print("sys", np.max(np.abs(s["values"] - ov)) / den, np.max(np.abs(s["rhs"] - orhs)) / np.max(np.abs(orhs)),
      int(np.array_equal(s["hits"].astype(np.uint64), ohits)))
oc, _ = po.pcg(rp, cols, ov, orhs, tol=1e-12)
print("c", np.max(np.abs(c - oc)) / np.max(np.abs(oc)), d["iterations"])
"""


@pytest.mark.parametrize("env", [{"RBG_H2D_CHUNKS": "3"}, {"RBG_PREC": "jacobi"}, {"RBG_FSAI_RHO": "1.0"},
                                 {"RBG_SOLVER": "band"}])
def test_chunked_upload_and_point_jacobi_paths(env):
    """The chunked pinned-upload path of rbg_assemble (accumulating chunks), the
    point-Jacobi PCG (RBG_PREC=jacobi), the FSAI PCG with a distance-restricted
    pattern and the banded LLT forced from the environment, against the oracle,
    cfg2 geometry at 1.2e6 points (the knobs are read once per process or centre
    set, hence a subprocess)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _SUBPROC.format(root=root)], capture_output=True, text=True,
                       env={**os.environ, **env}, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = dict(l.split(" ", 1) for l in r.stdout.strip().splitlines() if l.startswith(("sys", "c ")))
    eb, er, hits = lines["sys"].split()
    assert float(eb) < TOL_SYS and float(er) < TOL_SYS and hits == "1"
    assert float(lines["c"].split()[0]) < TOL_C
