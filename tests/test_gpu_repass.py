"""The orthogonal least-squares re-pass of fit (least_squares_repass,
solver.cpp:345-397, called at solver.cpp:439-464) on the GPU, and the
acceptance cases that depend on it (acceptance_main.cpp:65-101).

The reference's re-pass answer is the least-squares solution of the
augmented design; Eigen (its QR) is absent here, so the stand-in is LAPACK's
QR least squares (numpy.linalg.lstsq) of the dense design built by the
reference's own assemble_submatrix (oracle/_ref)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_1806_07884_b200 import api, configs

pytestmark = pytest.mark.gpu


def franke_cloud(n):  # make_franke_cloud (data.cpp:118-124)
    xy = po.ref_halton_at(np.arange(1, n + 1, dtype=np.uint64), 2)
    return xy, po.ref_franke(xy)


def grid81():  # uniform_grid_refs(Aabb{{0,0},{1,1}}, 81)
    return po.ref_grid_refs(9, 9)


def lstsq_mae(xy, h, refs, family, alpha, poly=False):
    a = po.ref_dense_design(xy, refs, family, alpha)
    if poly:
        a = np.hstack([a, xy, np.ones((len(h), 1))])
    w = np.linalg.lstsq(a, h, rcond=None)[0]
    return float(np.mean(np.abs(a @ w - h))), w


@pytest.fixture(scope="module")
def eng():
    e = api.Engine(0)
    yield e
    e.close()


def fit_mae(eng, xy, h, refs, family, alpha, poly=False):
    model, rep = api.fit(xy, h, refs, api.KernelSpec(family, alpha), engine=eng, poly=poly)
    er = api.error_report(model, xy, h, engine=eng)
    return er["mean_absolute_error"], rep, model


def test_repass_is_the_least_squares_solution(eng):
    """rbg_least_squares_repass against LAPACK least squares on the dense
    augmented design, with and without the polynomial border, several
    4096-row chunks (incremental QR across chunks)."""
    rng = np.random.default_rng(3)
    xy = rng.random((10_000, 2))
    h = np.sin(3 * xy[:, 0]) + xy[:, 1] ** 2 + 0.01 * rng.standard_normal(10_000)
    refs = rng.random((60, 2))
    for poly in (False, True):
        eng.set_centres(refs, api.KernelSpec(1, 3.0))
        eng.set_poly(poly)
        try:
            w = eng.least_squares_repass(xy, h)
        finally:
            eng.set_poly(False)
        _, want = lstsq_mae(xy, h, refs, 1, 3.0, poly)
        assert w is not None
        assert np.max(np.abs(w - want)) / np.max(np.abs(want)) < 1e-9, poly


def test_flat_kernel_fit_escapes_the_ridge_through_the_repass(eng):
    """test_solver.cpp:282-312: 9000 Franke points, 81 grid references,
    wendland-3-3 alpha 0.25: the plain factorisation fails, the fit lands on
    the least-squares solution (MAE within 2 % of a dense QR solve) with
    ridge 0 and says so ("re-pass") in its warnings."""
    xy, h = franke_cloud(9000)
    refs = grid81()
    mae, rep, _ = fit_mae(eng, xy, h, refs, 2, 0.25)
    mae_qr, _ = lstsq_mae(xy, h, refs, 2, 0.25)
    assert rep.ridge_lambda == 0.0
    assert rep.warnings and "re-pass" in rep.warnings[0]
    assert mae == pytest.approx(mae_qr, rel=0.02)
    assert mae < 2.0 * mae_qr


def test_acceptance_c01_c02_c03(eng):
    """acceptance_main.cpp:65-101 on 1089 Franke points and 81 grid refs:
    C01 wendland-3-3 alpha 0.25 MAE in [0.001, 0.004]; C02 MAE(3-0, .707) >
    MAE(3-1, .5) >= MAE(3-3, .25), the roughest in [0.002, 0.008]; C03 the
    polynomial never hurts (MAE with poly <= plain + 1e-4)."""
    xy, h = franke_cloud(1089)
    refs = grid81()
    m30 = fit_mae(eng, xy, h, refs, 0, 0.707)[0]
    m31 = fit_mae(eng, xy, h, refs, 1, 0.5)[0]
    m33 = fit_mae(eng, xy, h, refs, 2, 0.25)[0]
    assert 0.001 <= m33 <= 0.004
    assert m30 > m31 >= m33 and 0.002 <= m30 <= 0.008
    for fam, alpha, plain in ((0, 0.707, m30), (1, 0.5, m31), (2, 0.25, m33)):
        assert fit_mae(eng, xy, h, refs, fam, alpha, poly=True)[0] <= plain + 1e-4, fam
    # each against the least-squares answer the reference's fit reaches
    for fam, alpha, got in ((0, 0.707, m30), (1, 0.5, m31), (2, 0.25, m33)):
        assert got == pytest.approx(lstsq_mae(xy, h, refs, fam, alpha)[0], rel=0.02), fam


def test_repass_limit_and_rank_deficiency(eng):
    """Beyond the device limit the call is rejected; a rank-deficient design
    (an empty-support reference) gives no weights (solver.cpp:392)."""
    import ctypes as C

    from paper_1806_07884_b200 import _native
    assert _native.lib().rbg_repass_max_unknowns() == 4096
    rng = np.random.default_rng(5)
    pts = rng.random((60, 2))
    h = 2.0 * rng.random(60) - 1.0
    refs = np.array([[0.1, 0.1], [0.9, 0.1], [0.1, 0.9], [0.9, 0.9], [50.0, 50.0]])
    eng.set_centres(refs, api.KernelSpec("wendland-3-0", 1.0))
    assert eng.least_squares_repass(pts, h) is None
    big = rng.random((5000, 2))
    eng.set_centres(big, api.KernelSpec(1, 50.0))
    with pytest.raises(ValueError, match="4096"):
        eng.least_squares_repass(pts, h)
