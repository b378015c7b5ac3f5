"""Generates tests/golden/io_cases.npz by running the REFERENCE'S OWN file
writers and readers (model.cpp save_model/load_model/write_signed_errors,
data.cpp save_xyz/load_xyz/load_eval_points/load_ref_points/center_cloud,
compiled from /root/reference by oracle/Makefile into oracle/_ref).

The fixture holds the exact bytes the reference writes for tricky doubles, the
records its loaders parse from awkward text (comments, commas, tabs, '+',
CR, blank lines) and its error messages (file path replaced by <PATH>).
Usage (in a container with /root/reference):  python tests/golden/make_io_golden.py
"""
from __future__ import annotations

import ctypes as C
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as po  # noqa: E402

OUT = Path(__file__).resolve().parent
_P, _U64 = C.c_void_p, C.c_uint64

# doubles whose shortest round-trip text differs between printf styles
TRICKY = np.array([0.1, 1e-5, 1e16, 123456.789, -0.0, 5e-324, 1.7976931348623157e308, 0.0001, 100.0,
                   1e21, 1e22, 2.0 ** 53, 1.0 / 3.0, -2.5e-8, 0.5, 7.0, 1e-7, 12345678901234567890.0,
                   0.30000000000000004, 2.2250738585072014e-308])

LOADER_TEXT = (b"# header comment\n"
               b"0.25 0.5 1.0\n"
               b"\n"
               b"  +1e-3,\t2.5e+2 , -0.0   # trailing comment\r\n"
               b"3 4 5\n"
               b"\t\n"
               b"1.7976931348623157e308 5e-324 0.1\n")
LOADER_TEXT2 = b"0.1 0.2\n# c\n0.3,0.4\n"

BAD_RECORDS = [  # (text, kind)
    (b"1 2\n", 0), (b"1 2 3 4 5\n", 0), (b"1 x 3\n", 0), (b"1 2 inf\n", 0), (b"# only\n\n", 0),
    (b"1 2\n1 2 3\n", 1), (b"1\n", 1), (b"1 2 3 4\n", 2), (b"nan 1\n", 2), (b"1 2 3e\n", 1),
]
BAD_MODELS = [
    b"",
    b"rbfit modle 1\n",
    b"rbfit model 2\n",
    b"rbfit model\n",
    b"rbfit model 1\nkernel wendland-9-9\n",
    b"rbfit model 1\nkernel wendland-3-1\nalpha x\n",
    b"rbfit model 1\nkernel wendland-3-1\nalpha 2\noffset 0 0\npoly 2\n",
    b"rbfit model 1\nkernel wendland-3-1\nalpha 2\noffset 0 0\npoly 0\nrefs 0\n",
    b"rbfit model 1\nkernel wendland-3-1\nalpha 2\noffset 0 0\npoly 0\nrefs 2\n0 0 1\n",
    b"rbfit model 1\nkernel wendland-3-1\nalpha 2\noffset 0 0\npoly 1\nrefs 1\n0 0 1\n",
    b"rbfit model 1\nkernel wendland-3-1\nalpha 2\noffset 0\n",
]


def lib():
    L = po.ref()
    L.ref_save_model.argtypes = [C.c_char_p, C.c_int, C.c_double, _P, _P, _U64, C.c_double, C.c_double, _P]
    L.ref_load_model.argtypes = [C.c_char_p, _P, _P, _P, _P, _P, _P, _U64]
    L.ref_save_xyz.argtypes = [C.c_char_p, _P, _P, _U64]
    L.ref_load_records.argtypes = [C.c_char_p, C.c_int, _P, _P, _P, _U64]
    L.ref_write_signed_errors.argtypes = [C.c_char_p, _P, _P, _U64, C.c_double, C.c_double, _P]
    return L


def main():
    L = lib()
    tmp = Path(tempfile.mkdtemp())
    path = tmp / "f.txt"
    bpath = str(path).encode()
    data = {}
    rng = np.random.default_rng(77)
    m = len(TRICKY)
    refs = np.stack([TRICKY, rng.random(m)], axis=1).copy()
    w = (rng.standard_normal(m) * 10.0 ** rng.integers(-12, 12, m)).copy()
    poly = np.array([1e-300, -3.25, 0.1])
    for tag, pp in (("poly", poly), ("nopoly", None)):
        st = L.ref_save_model(bpath, 1, 10.2333, refs.ctypes.data, w.ctypes.data, m, 0.5, -1e-9,
                              None if pp is None else pp.ctypes.data)
        assert st == 0, L.ref_last_error()
        data[f"model_{tag}_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()
    data.update(model_refs=refs, model_w=w, model_poly=poly, model_alpha=10.2333, model_family=1,
                model_offset=np.array([0.5, -1e-9]))

    xy = np.stack([TRICKY, TRICKY[::-1]], axis=1).copy()
    h = (TRICKY * 0.5).copy()
    assert L.ref_save_xyz(bpath, xy.ctypes.data, h.ctypes.data, len(h)) == 0
    data["xyz_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()
    data["xyz_points"], data["xyz_values"] = xy, h
    pred = h + rng.standard_normal(len(h))
    assert L.ref_write_signed_errors(bpath, xy.ctypes.data, h.ctypes.data, len(h), 0.25, -3.0,
                                     pred.ctypes.data) == 0
    data["err_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()
    data["err_pred"] = pred

    def load(text: bytes, kind: int):
        path.write_bytes(text)
        n, ar = C.c_uint64(), C.c_int()
        out = np.zeros(4096)
        st = L.ref_load_records(bpath, kind, C.byref(n), C.byref(ar), out.ctypes.data, len(out))
        if st:
            return st, L.ref_last_error().decode().replace(str(path), "<PATH>"), None
        return 0, "", out[: n.value * ar.value].reshape(n.value, ar.value).copy()

    for kind in (0, 1, 2):
        st, msg, rows = load(LOADER_TEXT, kind)
        assert st == 0, msg
        data[f"load_text_k{kind}"] = rows
    for kind in (1, 2):
        st, msg, rows = load(LOADER_TEXT2, kind)
        assert st == 0, msg
        data[f"load_text2_k{kind}"] = rows
    data["loader_text"] = np.frombuffer(LOADER_TEXT, dtype=np.uint8).copy()
    data["loader_text2"] = np.frombuffer(LOADER_TEXT2, dtype=np.uint8).copy()
    msgs, codes = [], []
    for text, kind in BAD_RECORDS:
        st, msg, _ = load(text, kind)
        assert st != 0, text
        msgs.append(msg)
        codes.append(st)
    data["bad_record_texts"] = np.array([t for t, _ in BAD_RECORDS], dtype=object).astype("S")
    data["bad_record_kinds"] = np.array([k for _, k in BAD_RECORDS])
    data["bad_record_msgs"] = np.array(msgs)
    data["bad_record_codes"] = np.array(codes)
    mmsgs, mcodes = [], []
    for text in BAD_MODELS:
        path.write_bytes(text)
        fam, hp, mm = C.c_int(), C.c_int(), C.c_uint64()
        scal = np.zeros(6)
        r = np.zeros(64)
        ww = np.zeros(32)
        st = L.ref_load_model(bpath, C.byref(fam), C.byref(hp), C.byref(mm), scal.ctypes.data, r.ctypes.data,
                              ww.ctypes.data, 32)
        assert st != 0, text
        mmsgs.append(L.ref_last_error().decode().replace(str(path), "<PATH>"))
        mcodes.append(st)
    data["bad_model_texts"] = np.array(BAD_MODELS, dtype=object).astype("S")
    data["bad_model_msgs"] = np.array(mmsgs)
    data["bad_model_codes"] = np.array(mcodes)

    cxy = (rng.random((1000, 2)) * 1e3 + 5e5).copy()
    vals = np.zeros(1000)
    off = np.zeros(2)  # the reference helper starts from a fresh (zero-offset) cloud
    out = cxy.copy()
    assert L.ref_center_cloud(out.ctypes.data, vals.ctypes.data, 1000, off.ctypes.data) == 0
    data.update(center_in=cxy, center_out=out, center_offset=off)
    # `rbfit gen-synthetic -n 1089` (rbfit_main.cpp:120-125): make_franke_cloud + save_xyz
    n = 1089
    hal = np.empty(2 * n)
    L.ref_halton_points(n, 2, hal.ctypes.data)
    fr = np.array([L.ref_franke(hal[2 * i], hal[2 * i + 1]) for i in range(n)])
    assert L.ref_save_xyz(bpath, hal.ctypes.data, fr.ctypes.data, n) == 0
    data["gen1089_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()
    np.savez_compressed(OUT / "io_cases.npz", **data)
    print("io_cases.npz", (OUT / "io_cases.npz").stat().st_size)


if __name__ == "__main__":
    main()
