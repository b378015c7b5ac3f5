"""Native libraries without a GPU: load, exports, host-side logic."""
import math
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_1806_07884_b200 import _native, api, configs, distributed

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "rbg.h").read_text()
    return sorted(set(re.findall(r"\b(rbg_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    L = _native.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_native.exported_symbols())


def test_io_header_symbols_are_exported():
    import ctypes

    L = ctypes.CDLL(str(ROOT / "paper_1806_07884_b200" / "librbfit_b200.so"))
    syms = sorted(set(re.findall(r"\b(rbfit_io_[a-z0-9_]+)\s*\(", (ROOT / "include" / "rbfit_io.h").read_text())))
    assert len(syms) == 9
    for s in syms:
        assert hasattr(L, s), s


def test_host_layer_library_exports_reference_api():
    import subprocess
    out = subprocess.run(["nm", "-DC", str(ROOT / "paper_1806_07884_b200" / "librbfit_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    for name in ("rbfit_b200::fit(", "rbfit_b200::build_normal_system(", "rbfit_b200::solve_weights(",
                 "rbfit_b200::evaluate_model(", "rbfit_b200::error_report(", "rbfit_b200::KernelSpec::evaluate",
                 "rbfit_b200::save_model(", "rbfit_b200::load_model(", "rbfit_b200::load_xyz(",
                 "rbfit_b200::save_xyz(", "rbfit_b200::write_signed_errors(", "rbfit_b200::center_cloud(",
                 "rbfit_b200::bench_block_sizes(", "rbfit_b200::PointIndex::PointIndex("):
        assert name in out, name


def test_kernel_value_matches_oracle_bitwise():
    for fam in (0, 1, 2, 3):
        k = api.KernelSpec(fam, 3.7)
        for r in np.linspace(0.0, 0.3, 301):
            assert k.evaluate(r) == po.phi(fam, 3.7, r)
    with pytest.raises(_native.DomainError):
        api.KernelSpec(1, 1.0).evaluate(-1.0)


def test_kernel_spec_validation_and_names():
    for bad in (0.0, -2.0, math.nan, math.inf):
        with pytest.raises(ValueError):
            api.KernelSpec("wendland-3-1", bad)
    with pytest.raises(ValueError):
        api.KernelSpec("gaussian", 1.0)
    assert api.KernelSpec("wendland-3-1", 2.0).name == "wendland-3-1"
    assert api.KernelSpec("wendland-3-1", 4.0).support_radius() == 0.25


@pytest.mark.parametrize("n,k", [(1000, 2), (1001, 4), (10, 8), (0, 3)])
def test_partition_slabs(n, k):
    rng = np.random.default_rng(n + k)
    pts = rng.random((n, 2))
    bounds, slab = distributed.partition_slabs(pts, k)
    assert bounds[0] == -math.inf and bounds[-1] == math.inf
    assert np.all(bounds[1:] >= bounds[:-1])
    counts = np.bincount(slab, minlength=k)
    assert counts.sum() == n
    if n >= 100:
        assert counts.max() - counts.min() <= 1
    for s in range(k):
        x = pts[slab == s, 0]
        assert np.all(x >= bounds[s]) and np.all(x < bounds[s + 1])


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.RbgError):
        api.Engine(0)


def test_config_generators_deterministic_and_windowed():
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        a, ha = configs.points(name, n=300)
        b, hb = configs.points(name, n=100, start=200)
        assert np.array_equal(a[200:], b) and np.array_equal(ha[200:], hb)
        assert np.all(np.isfinite(a)) and np.all(np.isfinite(ha))
        assert a.shape[1] == configs.CONFIGS[name].dim
        assert a.min() >= 0.0 and a.max() <= 1.0
    assert configs.centres("cfg5").shape == (1_000_000, 2)
    g = configs.centres("cfg2")
    assert g[0].tolist() == [0.0, 0.0] and g[-1].tolist() == [1.0, 1.0] and g[1, 0] == 1.0 / 99.0


def test_config_support_sizes():
    # the pinned radii give the per-support populations BASELINE asks for
    for name, want in (("cfg1", 30), ("cfg2", 50), ("cfg4", 40), ("cfg5", 40)):
        c = configs.CONFIGS[name]
        assert math.pi * c.radius ** 2 * c.m == pytest.approx(want, rel=1e-12)
    c = configs.CONFIGS["cfg3"]
    assert 4.0 / 3.0 * math.pi * c.radius ** 3 * c.m == pytest.approx(60, rel=1e-12)
