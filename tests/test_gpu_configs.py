"""GPU parity on every BASELINE config at (or near) full size, against the CPU
oracle (oracle/rbf_oracle.c: the reference's sparse point-ascending sums,
threaded by output rows without changing a bit).

Tolerances, stated per quantity:
* pattern (K2): bit-exact;
* hits / design_nnz: exact;
* A^T A: 1e-10 in the reference's scale-normalised metric max|d|/max|ref|
  (acceptance_main.cpp:118-125) and 1e-10 entry by entry (`entrywise`: every
  entry against sqrt(B_ii B_jj), and elementwise above 1e-6 of that scale);
* A^T h: 1e-10 scale-normalised;
* evaluation: bitwise for the same weights (model.cpp:50-72 order);
* error report: max |e| bitwise, the sums (MAE, deviation, relative %, RMS)
  1e-12 relative (fixed-order device reductions vs the sequential loop);
* c: 1e-8 (max|dc|/max|c|) against the restated dense Cholesky where the
  dense system fits (cfg1, cfg2).  At cfg3-5 no dense or direct CPU solve is
  feasible in a test and cond(A^T A) reaches 1e10 (cfg4, measured with
  scipy eigsh + splu), so no method can pin c forward to
  1e-8 there (forward error ~ cond * eps); c is pinned by its backward error
  on the ORACLE's system: ||B_o c - r_o|| / ||r_o|| <= 1e-9.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_1806_07884_b200 import api, configs

pytestmark = pytest.mark.gpu

TOL_SYS = 1e-10


def scaled(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


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


def sym_matvec(rp, cols, vals, x):
    import scipy.sparse as sp
    m = len(rp) - 1
    rows = np.repeat(np.arange(m), np.diff(rp.astype(np.int64)))
    U = sp.csr_matrix((vals, (rows, cols.astype(np.int64))), shape=(m, m))
    return U @ x + sp.triu(U, 1).T @ x


def check_system(eng, pts, h, refs, family, alpha):
    """GPU pattern + system vs the oracle; returns the oracle's (rp, cols, v, rhs, hits)."""
    eng.set_centres(refs, api.KernelSpec(family, alpha))
    eng.assemble(pts, h)
    rp, cols = eng.pattern()
    orp, ocols = po.pattern(refs, alpha)
    assert np.array_equal(rp, orp) and np.array_equal(cols, ocols), "pattern differs"
    s = eng.system()
    ov, orhs, ohits = po.assemble(pts, h, refs, family, alpha, orp, ocols)
    assert np.array_equal(s["hits"].astype(np.uint64), ohits)
    assert s["design_nnz"] == int(ohits.sum())
    assert scaled(s["values"], ov) < TOL_SYS
    assert max(entrywise(s["values"], ov, orp, ocols)) < TOL_SYS
    assert scaled(s["rhs"], orhs) < TOL_SYS
    return orp, ocols, ov, orhs, ohits


def check_eval_and_report(eng, refs, c, family, alpha, pts, h):
    f = eng.evaluate(c, pts)
    assert np.array_equal(f, po.evaluate(refs, c, family, alpha, pts)), "evaluation not bitwise"
    got = eng.error_report(c, pts, h)
    want = po.error_report(f, h)
    assert got["max_abs_error"] == want["max_abs_error"]
    for k in ("mean_absolute_error", "deviation_of_error", "mean_relative_error_pct", "rms_error"):
        assert got[k] == pytest.approx(want[k], rel=1e-12), k


@pytest.fixture(scope="module")
def eng():
    e = api.Engine(0)
    yield e
    e.close()


def test_cfg2_full_system_c_and_error_report(eng):
    """cfg2 at full size (1e6 points, 1e4 grid centres): system, c against
    the restated dense Cholesky (solver.cpp:289-330; LAPACK dpotrf), the error
    report of the fit."""
    import scipy.linalg as sl
    cfg = configs.CONFIGS["cfg2"]
    xy, h = configs.points("cfg2")
    refs = configs.centres("cfg2")
    rp, cols, ov, orhs, _ = check_system(eng, xy, h, refs, 1, cfg.alpha)
    c, diag = eng.solve()
    assert diag["ridge_lambda"] == 0.0
    B = po.densify(rp, cols, ov)
    oc = sl.cho_solve(sl.cho_factor(B, lower=True), orhs)
    assert np.max(np.abs(c - oc)) / np.max(np.abs(oc)) < 1e-8
    check_eval_and_report(eng, refs, c, 1, cfg.alpha, xy, h)


def test_cfg3_full_size(eng):
    """cfg3 at full size: 4e6 points in [0,1]^3, all 5e4 Halton centres,
    the BASELINE support (~60 centres), wendland-3-2."""
    cfg = configs.CONFIGS["cfg3"]
    xyz, h = configs.points("cfg3")
    refs = configs.centres("cfg3")
    rp, cols, ov, orhs, ohits = check_system(eng, xyz, h, refs, 3, cfg.alpha)
    assert eng.layout_info()["sub_div"] == 2  # first assembly of a centre set: r/2 cubes
    c, diag = eng.solve()
    res = np.linalg.norm(sym_matvec(rp, cols, ov, c) - orhs) / np.linalg.norm(orhs)
    assert res < 1e-9, res
    check_eval_and_report(eng, refs, c, 3, cfg.alpha, xyz[:200_000], h[:200_000])
    # from the third assembly on the same centres the tiling is the density-derived one (r/3
    # here: staged slot maps, two-panel sub-tiles); same system against the same oracle values
    eng.assemble(xyz, h)
    assert eng.layout_info()["sub_div"] == 2
    eng.assemble(xyz, h)
    assert eng.layout_info()["sub_div"] == 3
    s = eng.system()
    assert np.array_equal(s["hits"].astype(np.uint64), ohits)
    assert scaled(s["values"], ov) < TOL_SYS and max(entrywise(s["values"], ov, rp, cols)) < TOL_SYS
    assert scaled(s["rhs"], orhs) < TOL_SYS


def test_cfg4_four_million_points(eng):
    """cfg4 on its first 4e6 points (the mixture's densest regions included),
    all 1e5 Halton centres."""
    cfg = configs.CONFIGS["cfg4"]
    xy, h = configs.points("cfg4", n=4_000_000)
    refs = configs.centres("cfg4")
    rp, cols, ov, orhs, ohits = check_system(eng, xy, h, refs, 1, cfg.alpha)
    assert (ohits == 0).sum() == 0
    c, diag = eng.solve()
    res = np.linalg.norm(sym_matvec(rp, cols, ov, c) - orhs) / np.linalg.norm(orhs)
    assert res < 1e-9, res
    check_eval_and_report(eng, refs, c, 1, cfg.alpha, xy[:200_000], h[:200_000])


def test_cfg5_full_pattern_and_window_system(eng):
    """cfg5: the whole symbolic pattern of the 1e6 grid centres (80.5 M upper
    entries) bit-exact, and the system of the 2.78e6 points of the spatial
    window [0, 1/8) x [0, 1/9) (full cfg5 density, q = 9 / S = 4 layout)
    against all 1e6 centres; evaluation and error report there."""
    cfg = configs.CONFIGS["cfg5"]
    refs = configs.centres("cfg5")
    xy, h = configs.window_points("cfg5", 3, 2)
    assert len(h) >= 2_000_000
    # the layout heuristic sees the window's points spread over the whole centre
    # grid; pin the full-size cfg5 layout (sub-tiles r/9, 4x4 super-tiles)
    eng.set_tile_divisor(9)
    eng.set_super_factor(4)
    try:
        check_system(eng, xy, h, refs, 1, cfg.alpha)
        info = eng.layout_info()
        assert info["sub_div"] == 9 and info["super_factor"] == 4
    finally:
        eng.set_tile_divisor(0)
        eng.set_super_factor(0)
    rng = np.random.default_rng(55)
    c = rng.standard_normal(cfg.m)
    check_eval_and_report(eng, refs, c, 1, cfg.alpha, xy[:500_000], h[:500_000])


def test_banded_llt_is_the_reference_cholesky(eng):
    """The direct solve (rbg_band.cu: LLT of the x-ordered band with the
    reference's ridge ladder, solver.cpp:289-330) against the restated dense
    Cholesky on the same assembled system: cfg1 at full size and a cfg2
    subsample; the empty-support case takes the ridge and the zero system
    names its pivot."""
    import scipy.linalg as sl
    for name, n in (("cfg1", None), ("cfg2", 300_000)):
        cfg = configs.CONFIGS[name]
        xy, h = configs.points(name, n=n)
        refs = configs.centres(name)
        eng.set_centres(refs, api.KernelSpec(cfg.kernel, cfg.alpha))
        eng.assemble(xy, h)
        c, diag = eng.solve(method="band")
        assert diag["iterations"] == 0 and diag["ridge_lambda"] == 0.0, diag  # direct
        assert diag["rel_residual"] < 1e-12, diag
        rp, cols = eng.pattern()
        s = eng.system()
        oc = sl.cho_solve(sl.cho_factor(po.densify(rp, cols, s["values"]), lower=True), s["rhs"])
        assert np.max(np.abs(c - oc)) / np.max(np.abs(oc)) < 1e-9, name
