"""Python mirror of the reference's (rbfit) hot-path interface over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/rbfit/{kernel,solver,model}.hpp; the
computation is the CUDA engine (librbg.so).  The C++ mirror for native
callers is csrc/rbfit_gpu.hpp.  This module is host plumbing for tests, the
bench and Python users; it never computes anything on the CPU itself.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import KERNELS, check, lib

KERNEL_NAMES = {v: k for k, v in KERNELS.items()}


def _f64(a, cols: int | None = None) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if cols is not None and arr.ndim == 1:
        arr = arr.reshape(-1, cols)
    return arr


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


# ------------------------------------------------------------------ kernel
class KernelSpec:
    """rbfit::KernelSpec (kernel.hpp:32-71): family + shape parameter alpha,
    support radius 1/alpha."""

    def __init__(self, family: str | int, alpha: float):
        if isinstance(family, str):
            if family not in KERNELS:  # kernel.cpp:24-30
                raise ValueError(f"unknown kernel '{family}'; expected one of: " + " ".join(KERNELS))
            family = KERNELS[family]
        if family not in KERNEL_NAMES:
            raise ValueError("unknown kernel family")
        if not (alpha > 0.0) or not np.isfinite(alpha):  # kernel.cpp:35-38
            raise ValueError("kernel shape parameter must be positive and finite")
        self.family = int(family)
        self.alpha = float(alpha)

    @property
    def name(self) -> str:
        return KERNEL_NAMES[self.family]

    def support_radius(self) -> float:
        return 1.0 / self.alpha

    def evaluate(self, r: float) -> float:
        out = C.c_double()
        st = lib().rbg_kernel_value(self.family, self.alpha, float(r), C.byref(out))
        if st == _native.RBG_DOMAIN_ERROR:
            raise _native.DomainError(st, "kernel evaluate: radius must be finite and non-negative")
        check(st)
        return out.value


# ------------------------------------------------------------------ engine
class Engine:
    """One CUDA context (rbg_ctx): centre set, pattern, device system."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._L = lib()
        self._ctx = C.c_void_p()
        st = self._L.rbg_create(device, C.byref(self._ctx))
        if st != 0:
            raise _native._EXC.get(st, _native.RbgError)(st, f"rbg_create(device={device}) failed "
                                                             f"(status {st}); is a CUDA GPU visible?")
        if stream is not None:
            self.set_stream(stream)
        self.dim = 0
        self.m = 0
        self.kernel: KernelSpec | None = None
        self._info: dict | None = None

    def _check(self, st: int) -> None:
        check(st, self._ctx)

    def close(self) -> None:
        if self._ctx:
            self._L.rbg_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_tile_divisor(self, divisor: float) -> None:
        """Assembly sub-tile edge = radius / divisor (0 = automatic; perf knob)."""
        self._check(self._L.rbg_set_tile_divisor(self._ctx, float(divisor)))

    def set_super_factor(self, s: int) -> None:
        """Super-tile = s^dim sub-tiles (0 = automatic; perf knob)."""
        self._check(self._L.rbg_set_super_factor(self._ctx, int(s)))

    def layout_info(self) -> dict:
        """Assembly layout of the current centre set (built at the first assembly)."""
        info = _native.LayoutInfo()
        self._check(self._L.rbg_get_layout_info(self._ctx, C.byref(info)))
        return {k: getattr(info, k) for k, _ in info._fields_}

    def phi_selftest(self, family: int, alpha: float, n: int = 1 << 24, seed: int = 1, fast: bool = False) -> dict:
        """The numeric kernels' phi against the reference arithmetic (rbg_phi_selftest; fast = the
        variant of the assembly's k-loop, rbg_phi_selftest_fast)."""
        bad, rel, ab = C.c_uint64(), C.c_double(), C.c_double()
        fn = self._L.rbg_phi_selftest_fast if fast else self._L.rbg_phi_selftest
        self._check(fn(self._ctx, int(family), float(alpha), n, seed, C.byref(bad), C.byref(rel), C.byref(ab)))
        return {"mismatches": int(bad.value), "max_rel": rel.value, "max_abs": ab.value}

    def set_stream(self, stream: int | None) -> None:
        self._check(self._L.rbg_set_stream(self._ctx, stream))

    def synchronize(self) -> None:
        self._check(self._L.rbg_synchronize(self._ctx))

    @property
    def stream(self) -> int:
        """cudaStream_t the engine issues on (rbg_get_stream)."""
        s = C.c_void_p()
        self._check(self._L.rbg_get_stream(self._ctx, C.byref(s)))
        return int(s.value or 0)

    @property
    def launch_count(self) -> int:
        return int(self._L.rbg_launch_count(self._ctx))

    # --- centres / pattern
    def set_centres(self, centres, kernel: KernelSpec) -> None:
        c = _f64(centres)
        if c.ndim != 2 or c.shape[1] not in (2, 3):
            raise ValueError("centres must be an (m, 2) or (m, 3) array")
        self._check(self._L.rbg_set_centres(self._ctx, c.shape[1], _p(c), c.shape[0],
                                            kernel.family, kernel.alpha))
        self.dim, self.m, self.kernel = c.shape[1], c.shape[0], kernel
        self._info = None
        if getattr(self, "poly", False):  # the border setting survives a new centre set
            self._check(self._L.rbg_set_poly(self._ctx, 1))

    def pattern_info(self) -> dict:
        if self._info is None:
            info = _native.PatternInfo()
            self._check(self._L.rbg_get_pattern_info(self._ctx, C.byref(info)))
            self._info = {k: getattr(info, k) for k, _ in info._fields_}
        return self._info

    def pattern(self) -> tuple[np.ndarray, np.ndarray]:
        info = self.pattern_info()
        rp = np.empty(self.m + 1, dtype=np.uint64)
        cols = np.empty(info["nnz_upper"], dtype=np.uint32)
        self._check(self._L.rbg_get_pattern(self._ctx, _p(rp), _p(cols)))
        return rp, cols

    # --- assembly
    def assemble(self, points, values, accumulate: bool = False, validate: bool = True) -> None:
        pts = _f64(points, self.dim)
        h = _f64(values)
        if pts.shape[0] != h.shape[0]:
            raise ValueError("build_normal_system: value count does not match points")
        self._check(self._L.rbg_assemble(self._ctx, _p(pts), _p(h), h.shape[0],
                                         int(accumulate), int(validate)))

    def assemble_ptr(self, points_ptr: int, values_ptr: int, n: int, accumulate: bool = False,
                     validate: bool = False) -> None:
        """Host-pointer variant (pinned buffers) without numpy conversion."""
        self._check(self._L.rbg_assemble(self._ctx, points_ptr, values_ptr, n, int(accumulate),
                                         int(validate)))

    def assemble_device(self, d_points: int, d_values: int, n: int, accumulate: bool = False) -> None:
        self._check(self._L.rbg_assemble_device(self._ctx, d_points, d_values, n, int(accumulate)))

    def system_device(self) -> tuple[int, int]:
        ptr, cnt = C.c_void_p(), C.c_uint64()
        self._check(self._L.rbg_system_device(self._ctx, C.byref(ptr), C.byref(cnt)))
        return int(ptr.value), int(cnt.value)

    def hits(self) -> tuple[np.ndarray, int]:
        """Per-centre hit counts and design_nnz of the last assembly (no values copied)."""
        hits = np.empty(self.m)
        dn = C.c_uint64()
        self._check(self._L.rbg_get_system(self._ctx, None, None, _p(hits), C.byref(dn)))
        return hits, int(dn.value)

    def system(self) -> dict:
        info = self.pattern_info()
        vals = np.empty(info["nnz_upper"])
        rhs = np.empty(self.m)
        hits = np.empty(self.m)
        dn = C.c_uint64()
        self._check(self._L.rbg_get_system(self._ctx, _p(vals), _p(rhs), _p(hits), C.byref(dn)))
        return {"values": vals, "rhs": rhs, "hits": hits, "design_nnz": int(dn.value)}

    # --- linear-polynomial border (FitOptions::poly)
    def set_poly(self, enable: bool) -> None:
        """Enable the border [x, y, (z), 1] (solver.cpp:189-207, 238-262) for the
        following assemblies / solves of this centre set."""
        self._check(self._L.rbg_set_poly(self._ctx, int(bool(enable))))
        self.poly = bool(enable)

    @property
    def poly_terms(self) -> int:
        return (self.dim + 1) if getattr(self, "poly", False) else 0

    def border(self) -> dict:
        """A^T P (T x m), P^T P (T x T), P^T h (T) of the last assembly."""
        T = self.poly_terms
        atp, ptp, pth = np.empty((T, self.m)), np.empty((T, T)), np.empty(T)
        self._check(self._L.rbg_get_border(self._ctx, _p(atp), _p(ptp), _p(pth)))
        return {"atp": atp, "ptp": ptp, "pth": pth}

    def set_border(self, atp, ptp, pth) -> None:
        a, b, c = _f64(atp), _f64(ptp), _f64(pth)
        self._check(self._L.rbg_set_border(self._ctx, _p(a), _p(b), _p(c)))

    def poly_solution(self) -> np.ndarray:
        a = np.zeros(max(self.poly_terms, 1))
        self._check(self._L.rbg_get_poly_solution(self._ctx, _p(a)))
        return a[: self.poly_terms]

    def set_model_poly(self, a) -> None:
        aa = None if a is None else _f64(a)
        self._check(self._L.rbg_set_model_poly(self._ctx, _p(aa)))

    def set_system(self, values, rhs, hits=None) -> None:
        v, r = _f64(values), _f64(rhs)
        hh = None if hits is None else _f64(hits)
        self._check(self._L.rbg_set_system(self._ctx, _p(v), _p(r), _p(hh)))

    # --- solve / eval
    def solve(self, tol: float = 0.0, max_iter: int = 0, method: str = "auto",
              precond: str = "auto") -> tuple[np.ndarray, dict]:
        """rbg_solve: method "auto" / "pcg" (FSAI-preconditioned CG) or "band" (the
        reference's LLT on the x-ordered band); precond "auto" / "fsai" / "jacobi"."""
        c = np.empty(self.m)
        opts = _native.SolveOptions(tol, max_iter, {"auto": 0, "pcg": 1, "band": 2}[method],
                                    {"auto": 0, "fsai": 1, "jacobi": 2}[precond])
        diag = _native.SolveDiag()
        self._check(self._L.rbg_solve(self._ctx, C.byref(opts), _p(c), C.byref(diag)))
        return c, {k: getattr(diag, k) for k, _ in diag._fields_}

    def least_squares_repass(self, points, values):
        """least_squares_repass (solver.cpp:345-397) on the device: the weights
        (m, then the border terms with poly) or None when they are not finite."""
        pts, h = _f64(points, self.dim), _f64(values)
        w = np.empty(self.m + self.poly_terms)
        ok = C.c_int()
        self._check(self._L.rbg_least_squares_repass(self._ctx, _p(pts), _p(h), h.shape[0], _p(w), C.byref(ok)))
        return w if ok.value else None

    def evaluate(self, c, queries) -> np.ndarray:
        cc = _f64(c)
        q = _f64(queries, self.dim)
        f = np.empty(q.shape[0])
        self._check(self._L.rbg_evaluate(self._ctx, _p(cc), _p(q), q.shape[0], _p(f)))
        return f

    def evaluate_device(self, d_c: int, d_q: int, nq: int, d_f: int) -> None:
        self._check(self._L.rbg_evaluate_device(self._ctx, d_c, d_q, nq, d_f))

    def error_report(self, c, points, values, signed: bool = False) -> dict:
        cc, pts, h = _f64(c), _f64(points, self.dim), _f64(values)
        st = _native.ErrorStats()
        se = np.empty(h.shape[0]) if signed else None
        self._check(self._L.rbg_error_report(self._ctx, _p(cc), _p(pts), _p(h), h.shape[0],
                                             C.byref(st), _p(se)))
        out = {k: getattr(st, k) for k, _ in st._fields_}
        if signed:
            out["signed_errors"] = se
        return out


# ----------------------------------------------- reference-shaped functions
@dataclass
class SparseNormalSystem:
    """NormalSystem (solver.hpp:61-69) in upper-CSR form: b is symmetric with
    b[i, cols[e]] = values[e] for e in row_ptr[i]..row_ptr[i+1] (cols >= i)."""
    side: int
    row_ptr: np.ndarray
    cols: np.ndarray
    values: np.ndarray
    rhs: np.ndarray
    empty_support_refs: np.ndarray
    design_nnz: int
    poly: bool = False

    def to_dense(self) -> np.ndarray:
        b = np.zeros((self.side, self.side))
        rows = np.repeat(np.arange(self.side), np.diff(self.row_ptr.astype(np.int64)))
        b[rows, self.cols] = self.values
        b[self.cols, rows] = self.values
        return b


@dataclass
class Model:
    """rbfit::Model (model.hpp:17-23): weights, optional linear polynomial
    (a_x, a_y, (a_z), a_1), offset."""
    kernel: KernelSpec
    refs: np.ndarray
    weights: np.ndarray
    offset: tuple = (0.0, 0.0)
    poly: np.ndarray | None = None


@dataclass
class FitReport:
    """rbfit::FitReport (solver.hpp:120-131), GPU timings in ms."""
    design_nnz: int = 0
    empty_support_refs: list = field(default_factory=list)
    ridge_lambda: float = 0.0
    ridge_shift: float = 0.0
    iterations: int = 0
    rel_residual: float = 0.0
    setup_ms: float = 0.0
    solve_ms: float = 0.0
    warnings: list = field(default_factory=list)


def _validate_cloud(points, values, refs, who: str):
    pts = _f64(points)
    h = _f64(values)
    if pts.ndim != 2 or pts.shape[0] == 0:
        raise ValueError(f"{who}: empty point cloud")
    if h.shape[0] != pts.shape[0]:
        raise ValueError(f"{who}: cloud value count mismatch")
    r = _f64(refs)
    if r.ndim != 2 or r.shape[0] == 0:
        raise ValueError(f"{who}: no reference points")
    return pts, h, r


def build_normal_system(points, values, refs, kernel: KernelSpec, engine: Engine | None = None,
                        poly: bool = False) -> SparseNormalSystem:
    """build_normal_system (solver.hpp:86-94) on the GPU; single plan (the
    whole pattern is resident).  With poly the border blocks are attached as
    ``border`` (A^T P, P^T P, P^T h)."""
    pts, h, r = _validate_cloud(points, values, refs, "build_normal_system")
    eng = engine or Engine()
    eng.set_centres(r, kernel)
    eng.set_poly(poly)
    eng.assemble(pts, h)
    sysd = eng.system()
    rp, cols = eng.pattern()
    empty = np.flatnonzero(sysd["hits"] == 0).astype(np.uint32)
    s = SparseNormalSystem(r.shape[0], rp, cols, sysd["values"], sysd["rhs"], empty,
                           sysd["design_nnz"], poly)
    if poly:
        s.border = eng.border()
    return s


def fit(points, values, refs, kernel: KernelSpec, tol: float = 0.0, max_iter: int = 0,
        engine: Engine | None = None, poly: bool = False) -> tuple[Model, FitReport]:
    """fit (solver.cpp:401-478): assemble on the GPU, solve, package
    (poly = FitOptions::poly, the linear-polynomial border)."""
    pts, h, r = _validate_cloud(points, values, refs, "fit")
    rep = FitReport()
    if pts.shape[0] < r.shape[0]:  # solver.cpp:409-412
        rep.warnings.append("fewer data points than reference points; the least-squares system is "
                            "underdetermined")
    eng = engine or Engine()
    eng.set_centres(r, kernel)
    eng.set_poly(poly)
    eng.assemble(pts, h)
    hits, design_nnz = eng.hits()
    rep.design_nnz = design_nnz
    rep.empty_support_refs = np.flatnonzero(hits == 0).tolist()
    rep.setup_ms = eng.pattern_info()["setup_ms"]
    m, T = r.shape[0], eng.poly_terms
    try:
        c, diag = eng.solve(tol, max_iter)
        a = eng.poly_solution() if poly else None
    except _native.RuntimeFailure:
        # solver.cpp:439-451: even the deepest ridge rung failed; the re-pass is
        # the last resort and a rank-deficient design rethrows
        if m + T > _native.lib().rbg_repass_max_unknowns():
            raise
        w = eng.least_squares_repass(pts, h)
        if w is None:
            raise
        c, a = w[:m], (w[m:] if poly else None)
        diag = {"ridge_lambda": 0.0, "ridge_shift": 0.0, "iterations": 0, "rel_residual": 0.0, "solve_ms": 0.0}
        rep.warnings.append("normal equations unsolvable; weights recovered by an orthogonal re-pass "
                            "over the data")
    rep.ridge_lambda = diag["ridge_lambda"]
    rep.ridge_shift = diag["ridge_shift"]
    rep.iterations = diag["iterations"]
    rep.rel_residual = diag["rel_residual"]
    rep.solve_ms = diag["solve_ms"]
    if rep.ridge_lambda > 0.0:  # solver.cpp:452-464
        if m + T > _native.lib().rbg_repass_max_unknowns():
            raise _native.RuntimeFailure(
                _native.RBG_RUNTIME_ERROR,
                f"normal equations numerically singular (ridge lambda {rep.ridge_lambda:g}); the orthogonal "
                f"re-pass (solver.cpp:345-397) is limited to {_native.lib().rbg_repass_max_unknowns()} "
                f"unknowns on the GPU path")
        w = eng.least_squares_repass(pts, h)
        if w is not None:
            c, a = w[:m], (w[m:] if poly else None)
            rep.ridge_lambda = rep.ridge_shift = 0.0
            rep.warnings.append("normal equations numerically singular; weights recovered by an orthogonal "
                                "re-pass over the data")
    return Model(kernel, r, c, poly=a), rep


def evaluate_model(model: Model, queries, engine: Engine | None = None) -> np.ndarray:
    """evaluate_model (model.cpp:192-194); raw queries are shifted by -offset."""
    q = _f64(queries, model.refs.shape[1])
    if any(model.offset):
        q = q - np.asarray(model.offset[: q.shape[1]])
    eng = engine or Engine()
    eng.set_centres(model.refs, model.kernel)  # no device work when the engine already holds this set
    eng.set_model_poly(model.poly)
    return eng.evaluate(model.weights, q)


def error_report(model: Model, points, values, design_nnz: int | None = None,
                 engine: Engine | None = None) -> dict:
    """error_report (model.cpp:196-232) + rms / max."""
    pts = _f64(points, model.refs.shape[1])
    h = _f64(values)
    if h.shape[0] == 0:
        raise ValueError("error_report: empty cloud")
    if h.shape[0] != pts.shape[0]:
        raise ValueError("error_report: cloud value count mismatch")
    eng = engine or Engine()
    eng.set_centres(model.refs, model.kernel)  # no device work when the engine already holds this set
    eng.set_model_poly(model.poly)
    rep = eng.error_report(model.weights, pts, h, signed=True)
    if design_nnz is not None:
        rep["density_pct"] = 100.0 * design_nnz / (h.shape[0] * float(model.refs.shape[0]))
    return rep
