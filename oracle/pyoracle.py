"""ctypes bindings of the CPU checkers (test infrastructure only).

* ``liborc``       -- our C restatement of the reference path (rbf_oracle.c).
* ``librbfit_ref`` -- the reference's own sources compiled from
  /root/reference (only where it exists; the .so travels to the GPU box as a
  built artefact, never as source).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_ORC = HERE / "_build" / "liborc.so"
LIB_REF = HERE / "_ref" / "librbfit_ref.so"

_P = C.c_void_p
_U64 = C.c_uint64
_orc = None
_ref = None


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a, cols=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if cols and a.ndim == 1:
        a = a.reshape(-1, cols)
    return a


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not LIB_ORC.exists():
            subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
        L = C.CDLL(str(LIB_ORC))
        L.orc_phi.argtypes = [C.c_int, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.orc_radical_inverse.argtypes = [C.c_uint, _U64]
        L.orc_radical_inverse.restype = C.c_double
        L.orc_franke.argtypes = [C.c_double, C.c_double]
        L.orc_franke.restype = C.c_double
        L.orc_pattern.argtypes = [C.c_int, _P, _U64, C.c_double, _P, _P]
        L.orc_assemble.argtypes = [C.c_int, _P, _P, _U64, _P, _U64, C.c_int, C.c_double, _P, _P, _P, _P, _P]
        L.orc_evaluate.argtypes = [C.c_int, _P, _U64, _P, C.c_int, C.c_double, _P, _U64, _P]
        L.orc_error_report.argtypes = [_P, _P, _U64] + [C.POINTER(C.c_double)] * 5
        L.orc_cholesky_solve.argtypes = [_U64, _P, _P, _P, C.POINTER(C.c_double), C.POINTER(C.c_int),
                                         C.POINTER(C.c_int64)]
        L.orc_pcg.argtypes = [_U64, _P, _P, _P, _P, C.c_double, C.c_double, C.c_int, _P,
                              C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.orc_border.argtypes = [C.c_int, _P, _P, _U64, _P, _U64, C.c_int, C.c_double, _P, _P, _P]
        L.orc_evaluate_poly.argtypes = [C.c_int, _P, _U64, _P, _P, C.c_int, C.c_double, _P, _U64, _P]
        L.orc_densify.argtypes = [_U64, _P, _P, _P, _P]
        L.orc_densify.restype = None
        _orc = L
    return _orc


def ref_available() -> bool:
    return LIB_REF.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not LIB_REF.exists():
            raise FileNotFoundError(f"{LIB_REF} not built (needs /root/reference at build time)")
        L = C.CDLL(str(LIB_REF))
        L.ref_last_error.restype = C.c_char_p
        L.ref_kernel_evaluate.argtypes = [C.c_int, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.ref_radical_inverse.argtypes = [C.c_uint, _U64]
        L.ref_radical_inverse.restype = C.c_double
        L.ref_halton_points.argtypes = [_U64, C.c_int, _P]
        L.ref_franke.argtypes = [C.c_double, C.c_double]
        L.ref_franke.restype = C.c_double
        L.ref_halton_at.argtypes = [_P, _U64, C.c_int, _P]
        L.ref_franke_many.argtypes = [_P, _U64, _P]
        L.ref_franke_many.restype = None
        L.ref_uniform_grid_refs.argtypes = [C.c_double] * 4 + [_U64, _U64, _P]
        L.ref_center_cloud.argtypes = [_P, _P, _U64, _P]
        L.ref_build_normal_system.argtypes = [_P, _P, _U64, _P, _U64, C.c_int, C.c_double, _P, _P,
                                              C.POINTER(_U64), _P, _P]
        L.ref_assemble_triplets.argtypes = [_P, _U64, _P, _U64, C.c_int, C.c_double, _U64, _P, _P, _P,
                                            C.POINTER(_U64)]
        L.ref_evaluate_model.argtypes = [_P, _P, _U64, C.c_int, C.c_double, _P, _U64, _P]
        L.ref_error_report.argtypes = [_P, _P, _U64, C.c_int, C.c_double, _P, _P, _U64, _P, _P]
        L.ref_bench_step.argtypes = [_P, _P, _U64, _P, _U64, C.c_int, C.c_double, C.POINTER(C.c_double),
                                     C.POINTER(_U64)]
        L.ref_border.argtypes = [_P, _P, _U64, _P, _U64, C.c_int, C.c_double, _P, _P, _P]
        L.ref_evaluate_model_poly.argtypes = [_P, _P, _P, _U64, C.c_int, C.c_double, _P, _U64, _P]
        _ref = L
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(msg or f"oracle status {code}")
        self.code = code


def _ok(st, msg=""):
    if st != 0:
        raise OracleError(st, msg)


# ------------------------------------------------------------- restatement
def phi(family: int, alpha: float, r: float) -> float:
    out = C.c_double()
    _ok(orc().orc_phi(family, alpha, r, C.byref(out)))
    return out.value


def pattern(centres, alpha):
    c = _f64(centres)
    m, dim = c.shape
    rp = np.empty(m + 1, dtype=np.uint64)
    _ok(orc().orc_pattern(dim, _p(c), m, alpha, _p(rp), None))
    cols = np.empty(int(rp[-1]), dtype=np.uint32)
    _ok(orc().orc_pattern(dim, _p(c), m, alpha, _p(rp), _p(cols)))
    return rp, cols


def assemble(points, values, centres, family, alpha, rp, cols):
    p, h, c = _f64(points), _f64(values), _f64(centres)
    n, dim = p.shape
    m = c.shape[0]
    vals = np.empty(len(cols))
    rhs = np.empty(m)
    hits = np.empty(m, dtype=np.uint64)
    _ok(orc().orc_assemble(dim, _p(p), _p(h), n, _p(c), m, family, alpha, _p(rp), _p(cols),
                           _p(vals), _p(rhs), _p(hits)))
    return vals, rhs, hits


def evaluate(centres, w, family, alpha, queries):
    c, ww, q = _f64(centres), _f64(w), _f64(queries)
    f = np.empty(q.shape[0])
    _ok(orc().orc_evaluate(c.shape[1], _p(c), c.shape[0], _p(ww), family, alpha, _p(q), q.shape[0], _p(f)))
    return f


def border(points, values, centres, family, alpha):
    """A^T P (T x m), P^T P, P^T h of the linear-polynomial border."""
    p, h, c = _f64(points), _f64(values), _f64(centres)
    n, dim = p.shape
    m, T = c.shape[0], dim + 1
    atp, ptp, pth = np.empty((T, m)), np.empty((T, T)), np.empty(T)
    _ok(orc().orc_border(dim, _p(p), _p(h), n, _p(c), m, family, alpha, _p(atp), _p(ptp), _p(pth)))
    return {"atp": atp, "ptp": ptp, "pth": pth}


def evaluate_poly(centres, w, a, family, alpha, queries):
    c, ww, aa, q = _f64(centres), _f64(w), _f64(a), _f64(queries)
    f = np.empty(q.shape[0])
    _ok(orc().orc_evaluate_poly(c.shape[1], _p(c), c.shape[0], _p(ww), _p(aa), family, alpha, _p(q),
                                q.shape[0], _p(f)))
    return f


def bordered_dense(b, rhs, border):
    """Dense bordered system [[B, A^T P], [P^T A, P^T P]] and [A^T h; P^T h]."""
    atp, ptp, pth = border["atp"], border["ptp"], border["pth"]
    m, T = b.shape[0], ptp.shape[0]
    k = np.zeros((m + T, m + T))
    k[:m, :m] = b
    k[:m, m:] = atp.T
    k[m:, :m] = atp
    k[m:, m:] = ptp
    return k, np.concatenate([rhs, pth])


def error_report(f, h):
    f, h = _f64(f), _f64(h)
    outs = [C.c_double() for _ in range(5)]
    _ok(orc().orc_error_report(_p(f), _p(h), len(f), *[C.byref(o) for o in outs]))
    keys = ["mean_absolute_error", "deviation_of_error", "mean_relative_error_pct", "rms_error",
            "max_abs_error"]
    return {k: o.value for k, o in zip(keys, outs)}


def cholesky_solve(b_dense, rhs):
    b, r = _f64(b_dense), _f64(rhs)
    side = r.shape[0]
    x = np.empty(side)
    lam, att, piv = C.c_double(), C.c_int(), C.c_int64()
    st = orc().orc_cholesky_solve(side, _p(b), _p(r), _p(x), C.byref(lam), C.byref(att), C.byref(piv))
    if st != 0:
        raise OracleError(st, f"not positive definite; first non-positive pivot at index {piv.value}")
    return x, {"ridge_lambda": lam.value, "attempts": att.value}


def pcg(rp, cols, vals, rhs, shift=0.0, tol=1e-12, max_iter=20000):
    m = len(rhs)
    x = np.empty(m)
    it, rr = C.c_int(), C.c_double()
    st = orc().orc_pcg(m, _p(rp), _p(cols), _p(_f64(vals)), _p(_f64(rhs)), shift, tol, max_iter,
                       _p(x), C.byref(it), C.byref(rr))
    return x, {"status": st, "iterations": it.value, "rel_residual": rr.value}


def densify(rp, cols, vals):
    m = len(rp) - 1
    d = np.empty((m, m))
    orc().orc_densify(m, _p(rp), _p(cols), _p(_f64(vals)), _p(d))
    return d


# ---------------------------------------------------------- the reference
def ref_build_normal_system(points, values, refs, family, alpha, dense=True):
    p, h, r = _f64(points), _f64(values), _f64(refs)
    n, m = p.shape[0], r.shape[0]
    b = np.empty((m, m)) if dense else None
    rhs = np.empty(m)
    dn = _U64()
    ref_nnz = np.empty(m, dtype=np.uint32)
    times = np.empty(3)
    L = ref()
    st = L.ref_build_normal_system(_p(p), _p(h), n, _p(r), m, family, alpha, _p(b), _p(rhs),
                                   C.byref(dn), _p(ref_nnz), _p(times))
    _ok(st, L.ref_last_error().decode())
    return {"b": b, "rhs": rhs, "design_nnz": dn.value, "ref_nnz": ref_nnz,
            "times": {"index": times[0], "assembly": times[1], "gram": times[2]}}


def ref_border(points, values, refs, family, alpha):
    p, h, r = _f64(points), _f64(values), _f64(refs)
    m = r.shape[0]
    atp, ptp, pth = np.empty((3, m)), np.empty((3, 3)), np.empty(3)
    L = ref()
    _ok(L.ref_border(_p(p), _p(h), p.shape[0], _p(r), m, family, alpha, _p(atp), _p(ptp), _p(pth)),
        L.ref_last_error().decode())
    return {"atp": atp, "ptp": ptp, "pth": pth}


def ref_evaluate_poly(refs, w, a, family, alpha, queries):
    r, ww, aa, q = _f64(refs), _f64(w), _f64(a), _f64(queries)
    f = np.empty(q.shape[0])
    L = ref()
    _ok(L.ref_evaluate_model_poly(_p(r), _p(ww), _p(aa), r.shape[0], family, alpha, _p(q), q.shape[0], _p(f)),
        L.ref_last_error().decode())
    return f


def ref_evaluate(refs, w, family, alpha, queries):
    r, ww, q = _f64(refs), _f64(w), _f64(queries)
    f = np.empty(q.shape[0])
    L = ref()
    _ok(L.ref_evaluate_model(_p(r), _p(ww), r.shape[0], family, alpha, _p(q), q.shape[0], _p(f)),
        L.ref_last_error().decode())
    return f


def ref_error_report(refs, w, family, alpha, points, values):
    r, ww, p, h = _f64(refs), _f64(w), _f64(points), _f64(values)
    out = np.empty(3)
    se = np.empty(len(h))
    L = ref()
    _ok(L.ref_error_report(_p(r), _p(ww), r.shape[0], family, alpha, _p(p), _p(h), len(h), _p(out), _p(se)),
        L.ref_last_error().decode())
    return {"mean_absolute_error": out[0], "deviation_of_error": out[1],
            "mean_relative_error_pct": out[2], "signed_errors": se}


def ref_dense_design(points, refs, family, alpha):
    """Dense design matrix A (n x m) from the reference's own assemble_submatrix
    (coo.cpp:166-192): A[p, j] = phi(|p - ref_j|) inside the strict support."""
    p, r = _f64(points), _f64(refs)
    n, m = p.shape[0], r.shape[0]
    cap = n * m
    rows = np.empty(cap, dtype=np.uint32)
    cols = np.empty(cap, dtype=np.uint32)
    vals = np.empty(cap)
    nnz = _U64()
    L = ref()
    _ok(L.ref_assemble_triplets(_p(p), n, _p(r), m, family, alpha, cap, _p(rows), _p(cols), _p(vals),
                                C.byref(nnz)), L.ref_last_error().decode())
    k = nnz.value
    a = np.zeros((n, m))
    a[rows[:k], cols[:k]] = vals[:k]
    return a


def ref_halton_at(indices, dims):
    """Halton points (the reference's radical_inverse) at the given sequence indices."""
    idx = np.ascontiguousarray(indices, dtype=np.uint64)
    out = np.empty((len(idx), dims))
    _ok(ref().ref_halton_at(_p(idx), len(idx), dims, _p(out)))
    return out


def ref_franke(xy):
    p = _f64(xy)
    out = np.empty(p.shape[0])
    ref().ref_franke_many(_p(p), p.shape[0], _p(out))
    return out


def ref_grid_refs(nx, ny, box=(0.0, 0.0, 1.0, 1.0)):
    out = np.empty((nx * ny, 2))
    _ok(ref().ref_uniform_grid_refs(*box, nx, ny, _p(out)))
    return out


def ref_bench_step(points, values, refs, family, alpha):
    p, h, r = _f64(points), _f64(values), _f64(refs)
    sec, dn = C.c_double(), _U64()
    L = ref()
    _ok(L.ref_bench_step(_p(p), _p(h), p.shape[0], _p(r), r.shape[0], family, alpha, C.byref(sec), C.byref(dn)),
        L.ref_last_error().decode())
    return sec.value, dn.value
