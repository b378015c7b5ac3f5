"""ctypes binding of the native libraries (the C ABI in include/rbg.h).

The CUDA library must be built in-tree (``python -m paper_1806_07884_b200.build``
or ``__graft_entry__.build()``); there is deliberately no CPU fallback: a
missing library raises immediately.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_RBG = PKG / "librbg.so"
LIB_DATAGEN = PKG / "librbg_datagen.so"

RBG_OK, RBG_INVALID_ARGUMENT, RBG_RUNTIME_ERROR, RBG_DOMAIN_ERROR, RBG_CUDA_ERROR, RBG_NOT_READY = range(6)

KERNELS = {"wendland-3-0": 0, "wendland-3-1": 1, "wendland-3-3": 2, "wendland-3-2": 3}


class RbgError(RuntimeError):
    """Base class; ``code`` is the rbg_status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(RbgError, ValueError):
    """std::invalid_argument in the reference."""


class RuntimeFailure(RbgError):
    """std::runtime_error in the reference (e.g. unsolvable system)."""


class DomainError(RbgError, ValueError):
    """std::domain_error in the reference."""


class CudaError(RbgError):
    """Device failure (no reference analogue)."""


class NotReady(RbgError):
    """Call-order violation."""


_EXC = {RBG_INVALID_ARGUMENT: InvalidArgument, RBG_RUNTIME_ERROR: RuntimeFailure,
        RBG_DOMAIN_ERROR: DomainError, RBG_CUDA_ERROR: CudaError, RBG_NOT_READY: NotReady}


class PatternInfo(C.Structure):
    _fields_ = [("m", C.c_uint64), ("nnz_upper", C.c_uint64), ("nnz_full", C.c_uint64),
                ("n_tiles", C.c_uint64), ("n_fallback", C.c_uint64),
                ("max_tile_centres", C.c_uint32), ("tile_edge", C.c_double),
                ("setup_ms", C.c_double)]


class LayoutInfo(C.Structure):
    _fields_ = [("built", C.c_int), ("sub_div", C.c_int), ("super_factor", C.c_int), ("n_buckets", C.c_int),
                ("n_super", C.c_uint64), ("n_fallback", C.c_uint64),
                ("max_super_centres", C.c_uint32), ("max_sub_centres", C.c_uint32),
                ("mean_super_centres", C.c_double), ("mean_sub_centres", C.c_double),
                ("sub_edge", C.c_double), ("build_ms", C.c_double)]


class SolveOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("method", C.c_int), ("precond", C.c_int)]


class SolveDiag(C.Structure):
    _fields_ = [("ridge_lambda", C.c_double), ("ridge_shift", C.c_double), ("attempts", C.c_int),
                ("iterations", C.c_int), ("rel_residual", C.c_double), ("solve_ms", C.c_double)]


class ErrorStats(C.Structure):
    _fields_ = [("mean_absolute_error", C.c_double), ("deviation_of_error", C.c_double),
                ("mean_relative_error_pct", C.c_double), ("rms_error", C.c_double),
                ("max_abs_error", C.c_double)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_U64 = C.c_uint64
_SIGS = {
    "rbg_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "rbg_destroy": (C.c_int, [_P]),
    "rbg_last_error": (C.c_char_p, [_P]),
    "rbg_set_stream": (C.c_int, [_P, _P]),
    "rbg_synchronize": (C.c_int, [_P]),
    "rbg_get_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "rbg_launch_count": (_U64, [_P]),
    "rbg_set_centres": (C.c_int, [_P, C.c_int, _P, _U64, C.c_int, C.c_double]),
    "rbg_get_pattern_info": (C.c_int, [_P, C.POINTER(PatternInfo)]),
    "rbg_get_pattern": (C.c_int, [_P, _P, _P]),
    "rbg_assemble": (C.c_int, [_P, _P, _P, _U64, C.c_int, C.c_int]),
    "rbg_assemble_device": (C.c_int, [_P, _P, _P, _U64, C.c_int]),
    "rbg_system_device": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_U64)]),
    "rbg_get_system": (C.c_int, [_P, _P, _P, _P, C.POINTER(_U64)]),
    "rbg_set_system": (C.c_int, [_P, _P, _P, _P]),
    "rbg_solve": (C.c_int, [_P, C.POINTER(SolveOptions), _P, C.POINTER(SolveDiag)]),
    "rbg_evaluate": (C.c_int, [_P, _P, _P, _U64, _P]),
    "rbg_least_squares_repass": (C.c_int, [_P, _P, _P, _U64, _P, C.POINTER(C.c_int)]),
    "rbg_repass_max_unknowns": (_U64, []),
    "rbg_evaluate_device": (C.c_int, [_P, _P, _P, _U64, _P]),
    "rbg_error_report": (C.c_int, [_P, _P, _P, _P, _U64, C.POINTER(ErrorStats), _P]),
    "rbg_partition_slabs": (C.c_int, [C.c_int, _P, _U64, C.c_int, C.c_int, _P, _P]),
    "rbg_kernel_value": (C.c_int, [C.c_int, C.c_double, C.c_double, _D]),
    "rbg_support_counts": (C.c_int, [_P, _P, _U64, C.POINTER(_U64), C.POINTER(_U64)]),
    "rbg_fp64_peak": (C.c_int, [_P, _D]),
    "rbg_assembly_times": (C.c_int, [_P, _D, _D]),
    "rbg_phi_selftest": (C.c_int, [_P, C.c_int, C.c_double, _U64, _U64, C.POINTER(_U64),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "rbg_phi_selftest_fast": (C.c_int, [_P, C.c_int, C.c_double, _U64, _U64, C.POINTER(_U64),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "rbg_set_tile_divisor": (C.c_int, [_P, C.c_double]),
    "rbg_set_super_factor": (C.c_int, [_P, C.c_int]),
    "rbg_get_layout_info": (C.c_int, [_P, C.POINTER(LayoutInfo)]),
    "rbg_set_poly": (C.c_int, [_P, C.c_int]),
    "rbg_get_border": (C.c_int, [_P, _P, _P, _P]),
    "rbg_set_border": (C.c_int, [_P, _P, _P, _P]),
    "rbg_get_poly_solution": (C.c_int, [_P, _P]),
    "rbg_set_model_poly": (C.c_int, [_P, _P]),
}

_lib = None
_datagen = None


def lib() -> C.CDLL:
    """The CUDA engine; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_RBG.exists():
            raise ImportError(f"{LIB_RBG} is missing: build it with "
                              "`python -m paper_1806_07884_b200.build` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_RBG))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(status: int, ctx=None) -> None:
    if status == RBG_OK:
        return
    msg = lib().rbg_last_error(ctx).decode() if ctx else f"rbg status {status}"
    raise _EXC.get(status, RbgError)(status, msg)


def datagen() -> C.CDLL:
    global _datagen
    if _datagen is None:
        if not LIB_DATAGEN.exists():
            raise ImportError(f"{LIB_DATAGEN} is missing: run the package build")
        L = C.CDLL(str(LIB_DATAGEN))
        L.dg_halton.argtypes = [_U64, _U64, C.c_int, _P]
        L.dg_grid_refs.argtypes = [C.c_double] * 4 + [_U64, _U64, _P]
        L.dg_halton_strided.argtypes = [_U64, _U64, _U64, C.c_int, _P]
        L.dg_add_noise_strided.argtypes = [_U64, _U64, _U64, _U64, C.c_double, _P]
        L.dg_franke.argtypes = [_P, _U64, _P]
        L.dg_uniform.argtypes = [_U64, _U64, C.c_int, _P]
        L.dg_add_noise.argtypes = [_U64, _U64, C.c_double, _P]
        L.dg_sincos.argtypes = [_P, _U64, _P]
        L.dg_bump3.argtypes = [_P, _U64, _P]
        L.dg_mixture.argtypes = [_U64, _U64, _P]
        L.dg_mixture_floor.argtypes = [_U64, _U64, C.c_int, _P]
        L.dg_fbm.argtypes = [_U64, _P, _U64, _P]
        for f in ("dg_halton", "dg_halton_strided", "dg_add_noise_strided", "dg_grid_refs", "dg_franke", "dg_uniform", "dg_add_noise",
                  "dg_sincos", "dg_bump3", "dg_mixture", "dg_fbm"):
            getattr(L, f).restype = None
        _datagen = L
    return _datagen
