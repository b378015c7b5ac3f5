"""On-disk formats of the reference, Python mirror.

Thin ctypes binding of the C++ implementation in ``csrc/rbfit_io.cpp``
(``librbfit_b200.so``), so files written here are byte-identical to the
reference's own (``save_model`` model.cpp:76-115, ``save_xyz`` data.cpp:143-157,
``write_signed_errors`` model.cpp:234-256) and the readers accept exactly what
the reference accepts (``load_model`` model.cpp:117-190, ``load_xyz`` /
``load_eval_points`` / ``load_ref_points`` data.cpp:126-196).  Error classes:
``ValueError`` for the reference's ``std::invalid_argument``, ``RuntimeError``
for its ``std::runtime_error`` (I/O and format errors), messages verbatim.
These are host-only functions: no GPU is needed.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .api import KernelSpec, Model

_LIB = Path(__file__).resolve().parent / "librbfit_b200.so"
_lib = None

_d = C.POINTER(C.c_double)


def _L():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            raise RuntimeError(f"{_LIB} is not built (python -m paper_1806_07884_b200.build)")
        lib = C.CDLL(str(_LIB))
        lib.rbfit_io_last_error.restype = C.c_char_p
        lib.rbfit_io_save_model.argtypes = [C.c_char_p, C.c_int, C.c_double, _d, _d, C.c_uint64, _d, _d]
        lib.rbfit_io_load_model.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.POINTER(C.c_uint64), _d]
        lib.rbfit_io_take_model.argtypes = [_d, _d]
        lib.rbfit_io_save_xyz.argtypes = [C.c_char_p, _d, _d, C.c_uint64]
        lib.rbfit_io_load_records.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        lib.rbfit_io_take_records.argtypes = [_d]
        lib.rbfit_io_write_signed_errors.argtypes = [C.c_char_p, _d, _d, C.c_uint64, _d, _d]
        lib.rbfit_io_center_cloud.argtypes = [_d, C.c_uint64, _d]
        _lib = lib
    return _lib


def _check(st: int) -> None:
    if st == 0:
        return
    msg = _L().rbfit_io_last_error().decode()
    raise (ValueError if st == 1 else RuntimeError)(msg)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_d)


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def _xy(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 2:
        raise ValueError("expected an (n, 2) array of 2-D points (the reference formats are 2-D)")
    return a


def save_model(model: Model, path) -> None:
    """save_model (model.cpp:76-115): "rbfit model 1" text file."""
    refs = _xy(model.refs)
    w = np.ascontiguousarray(model.weights, dtype=np.float64)
    off = np.ascontiguousarray(model.offset, dtype=np.float64)
    poly = None if model.poly is None else np.ascontiguousarray(model.poly, dtype=np.float64)
    if poly is not None and poly.shape != (3,):
        raise ValueError("the model file holds a 2-D linear polynomial (3 coefficients)")
    if len(refs) and len(w) != len(refs):
        raise ValueError("model weight count does not match reference count")
    _check(_L().rbfit_io_save_model(_path(path), model.kernel.family, model.kernel.alpha, _p(refs), _p(w),
                                    len(refs), _p(off), _p(poly)))


def load_model(path) -> Model:
    """load_model (model.cpp:117-190)."""
    fam, has_poly, m = C.c_int(), C.c_int(), C.c_uint64()
    scal = np.zeros(6)
    _check(_L().rbfit_io_load_model(_path(path), C.byref(fam), C.byref(has_poly), C.byref(m), _p(scal)))
    refs = np.empty((m.value, 2))
    w = np.empty(m.value)
    _check(_L().rbfit_io_take_model(_p(refs), _p(w)))
    return Model(KernelSpec(fam.value, float(scal[0])), refs, w, (float(scal[1]), float(scal[2])),
                 scal[3:6].copy() if has_poly.value else None)


def _records(path, kind: int) -> np.ndarray:
    n, ar = C.c_uint64(), C.c_int()
    _check(_L().rbfit_io_load_records(_path(path), kind, C.byref(n), C.byref(ar)))
    out = np.empty((n.value, ar.value))
    _check(_L().rbfit_io_take_records(_p(out)))
    return out


def load_xyz(path) -> tuple[np.ndarray, np.ndarray]:
    """load_xyz (data.cpp:126-141): (points (n, 2), values (n,))."""
    r = _records(path, 0)
    return np.ascontiguousarray(r[:, :2]), r[:, 2].copy()


def save_xyz(points, values, path) -> None:
    """save_xyz (data.cpp:143-157): "x y h" lines, shortest round-trip digits."""
    xy = _xy(points)
    h = np.ascontiguousarray(values, dtype=np.float64)
    if len(h) != len(xy):
        raise ValueError("save_xyz: value count mismatch")
    _check(_L().rbfit_io_save_xyz(_path(path), _p(xy), _p(h), len(h)))


def load_eval_points(path) -> tuple[np.ndarray, np.ndarray | None]:
    """load_eval_points (data.cpp:159-180): points and, for 3-field files, values."""
    r = _records(path, 1)
    return np.ascontiguousarray(r[:, :2]), (r[:, 2].copy() if r.shape[1] == 3 else None)


def load_ref_points(path) -> np.ndarray:
    """load_ref_points (data.cpp:182-196)."""
    return _records(path, 2)


def write_signed_errors(points, values, predictions, path, offset=(0.0, 0.0)) -> None:
    """write_signed_errors (model.cpp:234-256): "x y h f f-h" in the original frame."""
    xy = _xy(points)
    h = np.ascontiguousarray(values, dtype=np.float64)
    f = np.ascontiguousarray(predictions, dtype=np.float64)
    if len(h) != len(xy):
        raise ValueError("write_signed_errors: cloud value count mismatch")
    if len(f) != len(xy):
        raise ValueError("write_signed_errors: prediction count mismatch")
    off = np.ascontiguousarray(offset, dtype=np.float64)
    _check(_L().rbfit_io_write_signed_errors(_path(path), _p(xy), _p(h), len(h), _p(off), _p(f)))


def center_cloud(points, offset=(0.0, 0.0)) -> tuple[np.ndarray, tuple]:
    """center_cloud (data.cpp:198-223): subtract the compensated mean; returns
    (centred points, new offset)."""
    xy = _xy(points).copy()
    off = np.ascontiguousarray(offset, dtype=np.float64).copy()
    _check(_L().rbfit_io_center_cloud(_p(xy), len(xy), _p(off)))
    return xy, (float(off[0]), float(off[1]))
