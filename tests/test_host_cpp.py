"""The C++ host layer (rbfit_b200::fit & co.) driven from a C++ caller."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1806_07884_b200"


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = tmp_path_factory.mktemp("cpp") / "host_api_check"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{PKG / 'csrc'}", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "host_api_check.cpp"), "-o", str(out),
                    f"-L{PKG}", "-lrbfit_b200", "-lrbg", f"-Wl,-rpath,{PKG}"], check=True)
    return out


def test_host_layer_validation_without_gpu(exe):
    r = subprocess.run([str(exe), "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_host_layer_fit_matches_reference_golden(exe, tmp_path, golden):
    g = golden("readme_case")
    xy, h, refs = g["points"], g["values"], g["refs"]
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        np.array([len(h), len(refs)], dtype=np.uint64).tofile(f)
        np.array([0.5]).tofile(f)
        xy.astype(np.float64).tofile(f)
        h.astype(np.float64).tofile(f)
        refs.astype(np.float64).tofile(f)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), "gpu", str(inp), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    raw = np.fromfile(out, dtype=np.uint8)
    hdr = raw[:24].view(np.uint64)
    dbl = raw[24:].view(np.float64)
    m, n = len(refs), len(h)
    mae, dev = dbl[0], dbl[1]
    c = dbl[2:2 + m]
    f = dbl[2 + m:2 + m + n]
    rhs = dbl[2 + m + n:2 + 2 * m + n]
    diag = dbl[2 + 2 * m + n:]
    assert int(hdr[0]) == 88209 and int(hdr[1]) == 0
    assert np.max(np.abs(rhs - g["rhs"])) / np.max(np.abs(g["rhs"])) < 1e-10
    assert np.max(np.abs(diag - np.diag(g["b"]))) / np.max(np.diag(g["b"])) < 1e-10
    # README.md:69 mae of this fit (ill-conditioned, alpha = 0.5: loose by design)
    assert mae == pytest.approx(float(g["published_mae"]), rel=1e-4)
    assert np.all(np.isfinite(f)) and np.all(np.isfinite(c))


@pytest.mark.gpu
def test_host_layer_poly_affine_reproduction(exe, tmp_path):
    """FitOptions::poly through rbfit_b200::fit (acceptance C06,
    acceptance_main.cpp:207-225): h = 2x + 3y + 1 -> MAE < 1e-8."""
    rng = np.random.default_rng(77)
    xy = rng.random((200, 2))
    h = 2.0 * xy[:, 0] + 3.0 * xy[:, 1] + 1.0
    gx, gy = np.meshgrid(np.linspace(0, 1, 4), np.linspace(0, 1, 4))
    refs = np.stack([gx.ravel(), gy.ravel()], axis=1)
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        np.array([len(h), len(refs)], dtype=np.uint64).tofile(f)
        np.array([1.0]).tofile(f)
        xy.tofile(f)
        h.tofile(f)
        refs.tofile(f)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), "poly", str(inp), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    d = np.fromfile(out, dtype=np.float64)
    assert d[0] < 1e-8
    assert np.allclose(d[1:4], [2.0, 3.0, 1.0], atol=1e-6)
    assert np.allclose(d[-3:], d[1:4], rtol=1e-8, atol=1e-10)


@pytest.mark.gpu
def test_allreduce_hook_runs_on_the_context_stream(tmp_path):
    """rbfit_b200::AllReduce gets the context's stream (rbg_get_stream): a hook
    that only enqueues an add of a second context's partial system on that
    stream reproduces the single-pass assembly (rbfit_gpu.hpp; the NCCL
    all-reduce of SURVEY 8(e) plugs in the same way)."""
    from paper_1806_07884_b200 import configs
    exe = tmp_path / "hook_check"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++20", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                    f"-I{PKG / 'csrc'}", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "hook_check.cu"),
                    "-o", str(exe), f"-L{PKG}", "-lrbfit_b200", "-lrbg", f"-Xlinker=-rpath,{PKG}"], check=True)
    cfg = configs.CONFIGS["cfg2"]
    xy, h = configs.points("cfg2", n=400_000)
    refs = configs.centres("cfg2")
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        np.array([len(h), len(refs)], dtype=np.uint64).tofile(f)
        np.array([cfg.alpha]).tofile(f)
        xy.tofile(f)
        h.tofile(f)
        refs.tofile(f)
    r = subprocess.run([str(exe), str(inp)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_host_layer_flat_kernel_fit_takes_the_repass(exe, tmp_path):
    """rbfit_b200::fit on test_solver.cpp:282-312's flat-kernel case: the
    warnings name the re-pass, ridge is 0 and the MAE is the least-squares
    one (within 2 %, LAPACK lstsq on the reference's dense design)."""
    from oracle import pyoracle as po
    xy = po.ref_halton_at(np.arange(1, 9001, dtype=np.uint64), 2)
    h = po.ref_franke(xy)
    refs = po.ref_grid_refs(9, 9)
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        np.array([len(h), len(refs)], dtype=np.uint64).tofile(f)
        np.array([0.25]).tofile(f)
        xy.tofile(f)
        h.tofile(f)
        refs.tofile(f)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), "flat", str(inp), str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    mae, ridge = np.fromfile(out, dtype=np.float64)
    a = po.ref_dense_design(xy, refs, 2, 0.25)
    w = np.linalg.lstsq(a, h, rcond=None)[0]
    assert ridge == 0.0
    assert mae == pytest.approx(float(np.mean(np.abs(a @ w - h))), rel=0.02)
