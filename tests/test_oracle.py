"""The CPU oracle (oracle/rbf_oracle.c) pinned against the reference.

Pins: the reference's own unit-test known answers (cited per test) and the
golden fixtures in tests/golden/ that the compiled reference produced
(tests/golden/make_golden.py).  Runs without a GPU.
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as po

W30, W31, W33, W32 = 0, 1, 2, 3


# ------------------------------------------------------------------ kernel
def test_kernel_half_support_values():  # test_kernel.cpp:12-20
    assert po.phi(W30, 1.0, 0.5) == 0.25
    assert po.phi(W31, 1.0, 0.5) == 0.1875
    assert po.phi(W33, 1.0, 0.5) == 0.0595703125
    assert po.phi(W31, 0.25, 2.0) == 0.1875


@pytest.mark.parametrize("fam", [W30, W31, W33])
@pytest.mark.parametrize("alpha", [0.25, 1.0, 7.5])
def test_kernel_origin_and_edge(fam, alpha):  # test_kernel.cpp:22-35
    edge = 1.0 / alpha
    assert po.phi(fam, alpha, 0.0) == 1.0
    assert po.phi(fam, alpha, edge) == 0.0
    assert po.phi(fam, alpha, edge * 1.5) == 0.0
    assert po.phi(fam, alpha, np.nextafter(edge, 0.0)) > 0.0


def test_kernel_tail_and_domain():  # test_kernel.cpp:53-61, 63-74
    for fam in (W30, W31, W33):
        assert po.phi(fam, 1.0, 1.0 - 1e-8) < 1e-15
    for bad in (-1.0, math.nan, math.inf):
        with pytest.raises(po.OracleError) as e:
            po.phi(W30, 1.0, bad)
        assert e.value.code == 3  # domain_error
    for alpha in (0.0, -2.0, math.nan):
        with pytest.raises(po.OracleError):
            po.phi(W30, alpha, 0.5)


def test_kernel_matches_reference_table(golden):
    t = golden("kernel_kat")["table"]
    for fam, alpha, r, v in t:
        assert po.phi(int(fam), alpha, r) == v


def test_wendland32_extension():
    # BASELINE config 3 formula (1-r)^6 (35 r^2 + 18 r + 3): phi(0) = 3.
    assert po.phi(W32, 1.0, 0.0) == 3.0
    r = 0.3
    assert po.phi(W32, 1.0, r) == pytest.approx((1 - r) ** 6 * (35 * r * r + 18 * r + 3), rel=1e-15)
    assert po.phi(W32, 2.0, 0.5) == 0.0


# ------------------------------------------------------------------- data
def test_franke_and_halton():  # test_data.cpp:61-112
    assert po.orc().orc_franke(0.0, 0.0) == pytest.approx(0.7664205912849231, rel=1e-12)
    ri = po.orc().orc_radical_inverse
    assert [ri(2, i) for i in range(5)] == [0.0, 0.5, 0.25, 0.75, 0.125]
    assert ri(3, 1) == pytest.approx(1 / 3, rel=1e-15)
    assert ri(5, 1) == pytest.approx(0.2, rel=1e-15)


def test_datagen_matches_reference_generators(golden):
    from paper_1806_07884_b200 import configs

    g = golden("cfg1_system")
    xy, h = configs.points("cfg1", n=64)
    assert np.array_equal(xy, g["points_head"])  # halton_2d bit for bit
    assert np.array_equal(h, g["values_head"])  # franke bit for bit


# ----------------------------------------------------------------- pattern
def test_pattern_predicate_brute_force():
    rng = np.random.default_rng(5)
    for dim in (2, 3):
        c = rng.random((300, dim))
        alpha = 6.0
        rp, cols = po.pattern(c, alpha)
        lim = (2.0 * (1.0 / alpha)) ** 2
        for i in range(0, 300, 7):
            d2 = ((c - c[i]) ** 2)[:, 0] + ((c - c[i]) ** 2)[:, 1]
            if dim == 3:
                d2 = d2 + ((c - c[i]) ** 2)[:, 2]
            want = [j for j in range(i, 300) if d2[j] < lim]
            assert cols[rp[i]:rp[i + 1]].tolist() == want


# ---------------------------------------------------------------- assembly
def _check_against_reference_system(pts, h, refs, fam, alpha, b, rhs, ref_nnz):
    rp, cols = po.pattern(refs, alpha)
    vals, r, hits = po.assemble(pts, h, refs, fam, alpha, rp, cols)
    dense = po.densify(rp, cols, vals)
    assert np.array_equal(dense, b)  # bitwise: same summation order as gram_self
    assert np.array_equal(r, rhs)  # bitwise: transpose_matvec order
    assert np.array_equal(hits, ref_nnz.astype(np.uint64))
    # containment: every reference nonzero is inside the 2r pattern
    m = len(refs)
    in_pat = np.zeros((m, m), dtype=bool)
    rows = np.repeat(np.arange(m), np.diff(rp.astype(np.int64)))
    in_pat[rows, cols] = True
    in_pat |= in_pat.T
    assert not np.any((b != 0) & ~in_pat)


def test_small_instances_bitwise_vs_reference(golden):
    g = golden("random_small")
    for k in range(int(g["count"])):
        _check_against_reference_system(g[f"{k}_points"], g[f"{k}_values"], g[f"{k}_refs"],
                                        int(g[f"{k}_family"]), float(g[f"{k}_alpha"]), g[f"{k}_b"],
                                        g[f"{k}_rhs"], g[f"{k}_ref_nnz"])


def test_readme_case_bitwise_and_published(golden):
    g = golden("readme_case")
    _check_against_reference_system(g["points"], g["values"], g["refs"], W31, 0.5, g["b"], g["rhs"],
                                    g["ref_nnz"])
    assert int(g["design_nnz"]) == int(g["published_design_nnz"])  # README.md:68
    c, d = po.cholesky_solve(g["b"], g["rhs"])
    assert d["ridge_lambda"] == 0.0
    f = po.evaluate(g["refs"], c, W31, 0.5, g["points"])
    assert np.array_equal(f, g["f"])  # evaluate_shifted restated bit for bit
    er = po.error_report(f, g["values"])
    # README.md:69-70 (Eigen LLT there; solve rounding differs, system is ill-conditioned)
    assert er["mean_absolute_error"] == pytest.approx(float(g["published_mae"]), rel=1e-8)
    assert er["deviation_of_error"] == pytest.approx(float(g["published_deviation"]), rel=1e-8)
    assert er["mean_absolute_error"] == float(g["mae"])


def test_cfg1_full_bitwise_vs_reference(golden):
    from paper_1806_07884_b200 import configs

    g = golden("cfg1_system")
    xy, h = configs.points("cfg1")
    refs = configs.centres("cfg1")
    alpha = float(g["alpha"])
    assert alpha == configs.CONFIGS["cfg1"].alpha
    rp, cols = po.pattern(refs, alpha)
    vals, rhs, hits = po.assemble(xy, h, refs, W31, alpha, rp, cols)
    dense = po.densify(rp, cols, vals)
    b = np.zeros((1000, 1000))
    b[g["i"], g["j"]] = g["v"]
    b[g["j"], g["i"]] = g["v"]
    assert np.array_equal(dense, b)
    assert np.array_equal(rhs, g["rhs"])
    assert int(hits.sum()) == int(g["design_nnz"]) == 2756742
    assert len(cols) == 50898 and int((g["i"] <= g["j"]).sum()) == 50615  # SURVEY probe numbers


def test_hand_system():  # test_solver.cpp:142-162, test_coo.cpp:183-201
    pts = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]])
    refs = np.array([[1.0, 0.0]])
    rp, cols = po.pattern(refs, 0.5)
    vals, rhs, hits = po.assemble(pts, np.ones(3), refs, W30, 0.5, rp, cols)
    assert vals.tolist() == [1.125] and rhs.tolist() == [1.5] and hits.tolist() == [3]
    c, _ = po.cholesky_solve(np.array([[1.125]]), rhs)
    assert c[0] == pytest.approx(4.0 / 3.0, rel=1e-15)


def test_eval_and_error_kats():  # test_model.cpp:52-65, 80-97
    f = po.evaluate(np.array([[0.0, 0.0]]), np.array([2.0]), W30, 0.5,
                    np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0], [3.0, 0.0]]))
    assert f.tolist() == [2.0, 0.5, 0.0, 0.0]
    er = po.error_report(np.zeros(3), np.array([-1.0, -2.0, -3.0]))
    assert er["mean_absolute_error"] == 2.0
    assert er["deviation_of_error"] == pytest.approx(2.0 / 3.0, rel=1e-15)
    assert er["mean_relative_error_pct"] == pytest.approx(100.0, rel=1e-15)


# ------------------------------------------------------------------- solve
def test_pcg_matches_cholesky_cfg1(golden):
    g = golden("cfg1_system")
    b = np.zeros((1000, 1000))
    b[g["i"], g["j"]] = g["v"]
    b[g["j"], g["i"]] = g["v"]
    c_ref = g["c"]
    iu = np.triu_indices(1000)
    mask = b[iu] != 0
    # upper CSR of the reference's nonzeros
    rows, cols = iu[0][mask], iu[1][mask]
    rp = np.zeros(1001, dtype=np.uint64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    x, d = po.pcg(rp, cols.astype(np.uint32), b[rows, cols], g["rhs"], tol=1e-12)
    assert d["status"] == 0
    assert np.max(np.abs(x - c_ref)) / np.max(np.abs(c_ref)) < 1e-8


def test_zero_matrix_names_pivot():  # test_solver.cpp:314-326
    with pytest.raises(po.OracleError) as e:
        po.cholesky_solve(np.zeros((2, 2)), np.ones(2))
    assert "pivot" in str(e.value) and "0" in str(e.value)


def test_empty_support_takes_ridge():  # test_solver.cpp:264-280
    rng = np.random.default_rng(5)
    pts = rng.random((60, 2))
    h = 2.0 * rng.random(60) - 1.0
    refs = np.vstack([np.array([[x, y] for y in (pts[:, 1].min(), pts[:, 1].max())
                                for x in (pts[:, 0].min(), pts[:, 0].max())]), [[50.0, 50.0]]])
    rp, cols = po.pattern(refs, 1.0)
    vals, rhs, hits = po.assemble(pts, h, refs, W30, 1.0, rp, cols)
    assert hits[4] == 0
    c, d = po.cholesky_solve(po.densify(rp, cols, vals), rhs)
    assert d["ridge_lambda"] > 0.0 and abs(c[4]) < 1e-8


@pytest.mark.skipif(not po.ref_available(), reason="reference not compiled here")
def test_live_reference_random_3d_free_cases():
    # extra seeds straight against the compiled reference (where it exists)
    rng = np.random.default_rng(4242)
    for it in range(6):
        n = 50 + 37 * it
        pts = rng.random((n, 2))
        refs = pts[[j * n // 9 for j in range(9)]].copy()
        alpha = 1.0 + 3.0 * rng.random()
        h = rng.random(n)
        R = po.ref_build_normal_system(pts, h, refs, W31, alpha)
        _check_against_reference_system(pts, h, refs, W31, alpha, R["b"], R["rhs"], R["ref_nnz"])


# ------------------------------------------------ linear-polynomial border
def test_border_oracle_bitwise_vs_reference(golden):
    """orc_border restates solver.cpp:189-207, 238-262: bitwise equal to the
    reference's own triplet-order border on every committed instance."""
    g = golden("poly_cases")
    for t in range(int(g["count"])):
        b = po.border(g[f"{t}_points"], g[f"{t}_values"], g[f"{t}_refs"], int(g[f"{t}_family"]),
                      float(g[f"{t}_alpha"]))
        for k in ("atp", "ptp", "pth"):
            assert np.array_equal(b[k], g[f"{t}_{k}"]), (t, k)
    b = po.border(g["readme_points"], g["readme_values"], g["readme_refs"], 1, 0.5)
    assert all(np.array_equal(b[k], g[f"readme_{k}"]) for k in ("atp", "ptp", "pth"))


def test_poly_eval_oracle_bitwise_vs_reference(golden):
    """model.cpp:65-68 polynomial term, unfused left-to-right: bitwise."""
    g = golden("poly_cases")
    f = po.evaluate_poly(g["readme_refs"], g["readme_c"], g["readme_a"], 1, 0.5, g["readme_points"])
    assert np.array_equal(f, g["readme_f"])


def test_bordered_cholesky_affine_reproduction():
    """acceptance C06 (acceptance_main.cpp:207-225) on the oracle: h = 2x + 3y + 1
    with the border is reproduced to MAE < 1e-8."""
    rng = np.random.default_rng(77)
    pts = rng.random((200, 2))
    h = 2.0 * pts[:, 0] + 3.0 * pts[:, 1] + 1.0
    gx, gy = np.meshgrid(np.linspace(0, 1, 4), np.linspace(0, 1, 4))
    refs = np.stack([gx.ravel(), gy.ravel()], axis=1)
    rp, cols = po.pattern(refs, 1.0)
    v, rhs, _ = po.assemble(pts, h, refs, 1, 1.0, rp, cols)
    k, r = po.bordered_dense(po.densify(rp, cols, v), rhs, po.border(pts, h, refs, 1, 1.0))
    x, _ = po.cholesky_solve(k, r)
    f = po.evaluate_poly(refs, x[:16], x[16:], 1, 1.0, pts)
    assert np.mean(np.abs(f - h)) < 1e-8
