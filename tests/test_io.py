"""On-disk formats against the reference's own writers and
readers (tests/golden/io_cases.npz, made by tests/golden/make_io_golden.py from
the compiled reference): byte-identical files, identical parsed records and
error messages.  Host-only: runs without a GPU."""
from pathlib import Path

import numpy as np
import pytest

from paper_1806_07884_b200 import api, rbfit_io as io


@pytest.fixture(scope="module")
def g(golden):
    return golden("io_cases")


def _model(g, poly: bool) -> api.Model:
    return api.Model(api.KernelSpec(int(g["model_family"]), float(g["model_alpha"])), g["model_refs"],
                     g["model_w"], tuple(g["model_offset"]), g["model_poly"] if poly else None)


@pytest.mark.parametrize("poly", [True, False])
def test_save_model_bytes_equal_reference(g, tmp_path, poly):
    p = tmp_path / "m.txt"
    io.save_model(_model(g, poly), p)
    assert p.read_bytes() == bytes(g["model_poly_bytes" if poly else "model_nopoly_bytes"])


@pytest.mark.parametrize("poly", [True, False])
def test_load_reference_model_file(g, tmp_path, poly):
    p = tmp_path / "m.txt"
    p.write_bytes(bytes(g["model_poly_bytes" if poly else "model_nopoly_bytes"]))
    m = io.load_model(p)
    assert m.kernel.family == int(g["model_family"]) and m.kernel.alpha == float(g["model_alpha"])
    assert np.array_equal(m.refs.view(np.uint64), g["model_refs"].view(np.uint64))  # -0.0 and subnormals too
    assert np.array_equal(m.weights, g["model_w"])
    assert m.offset == tuple(g["model_offset"])
    if poly:
        assert np.array_equal(m.poly, g["model_poly"])
    else:
        assert m.poly is None
    # a save/load/save cycle is the identity on the bytes
    q = tmp_path / "m2.txt"
    io.save_model(m, q)
    assert q.read_bytes() == p.read_bytes()


def test_save_xyz_and_signed_errors_bytes(g, tmp_path):
    p = tmp_path / "x.txt"
    io.save_xyz(g["xyz_points"], g["xyz_values"], p)
    assert p.read_bytes() == bytes(g["xyz_bytes"])
    io.write_signed_errors(g["xyz_points"], g["xyz_values"], g["err_pred"], p, offset=(0.25, -3.0))
    assert p.read_bytes() == bytes(g["err_bytes"])


def test_loaders_parse_like_reference(g, tmp_path):
    p = tmp_path / "r.txt"
    p.write_bytes(bytes(g["loader_text"]))
    xy, h = io.load_xyz(p)
    k0 = g["load_text_k0"]
    assert np.array_equal(np.column_stack([xy, h]).view(np.uint64), k0.view(np.uint64))
    exy, eh = io.load_eval_points(p)
    assert np.array_equal(np.column_stack([exy, eh]), g["load_text_k1"])
    assert np.array_equal(io.load_ref_points(p), g["load_text_k2"])
    p.write_bytes(bytes(g["loader_text2"]))
    exy, eh = io.load_eval_points(p)
    assert eh is None and np.array_equal(exy, g["load_text2_k1"])
    assert np.array_equal(io.load_ref_points(p), g["load_text2_k2"])


def test_loader_errors_match_reference(g, tmp_path):
    p = tmp_path / "bad.txt"
    for text, kind, msg, code in zip(g["bad_record_texts"], g["bad_record_kinds"], g["bad_record_msgs"],
                                     g["bad_record_codes"]):
        p.write_bytes(bytes(text))
        fn = (io.load_xyz, io.load_eval_points, io.load_ref_points)[kind]
        exc = ValueError if int(code) == 1 else RuntimeError
        with pytest.raises(exc) as ei:
            fn(p)
        assert str(ei.value) == str(msg).replace("<PATH>", str(p))


def test_model_errors_match_reference(g, tmp_path):
    p = tmp_path / "bad_model.txt"
    for text, msg, code in zip(g["bad_model_texts"], g["bad_model_msgs"], g["bad_model_codes"]):
        p.write_bytes(bytes(text))
        with pytest.raises(ValueError if int(code) == 1 else RuntimeError) as ei:
            io.load_model(p)
        want = str(msg).replace("<PATH>", str(p))
        if "unknown kernel" in want:  # we also accept wendland-3-2 (3-D configs): the list is longer
            assert str(ei.value).startswith(want.split(";")[0])
        else:
            assert str(ei.value) == want
    with pytest.raises(RuntimeError, match="cannot open"):
        io.load_model(tmp_path / "missing.txt")


def test_save_model_validation(g, tmp_path):
    m = _model(g, False)
    with pytest.raises(ValueError, match="weight count"):
        io.save_model(api.Model(m.kernel, m.refs, m.weights[:-1]), tmp_path / "a")
    with pytest.raises(ValueError, match="no reference points"):
        io.save_model(api.Model(m.kernel, np.zeros((0, 2)), np.zeros(0)), tmp_path / "a")
    with pytest.raises(RuntimeError, match="cannot open"):
        io.save_model(m, tmp_path / "no_such_dir" / "m.txt")


def test_center_cloud_bitwise(g):
    xy, off = io.center_cloud(g["center_in"])
    assert np.array_equal(xy, g["center_out"])
    assert off == tuple(g["center_offset"]) or np.array_equal(np.array(off), g["center_offset"])


# ---------------------------------------------------------------- CLI (§8(f) row 4)
CLI = Path(__file__).resolve().parents[1] / "paper_1806_07884_b200" / "rbfit-b200"


def _cli(*args):
    import subprocess

    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True)


def test_cli_gen_synthetic_bytes_equal_reference(g, tmp_path):
    out = tmp_path / "franke.xyz"
    r = _cli("gen-synthetic", "-n", 1089, "--out", out)
    assert r.returncode == 0, r.stderr
    assert r.stdout == "points 1089\n"
    assert out.read_bytes() == bytes(g["gen1089_bytes"])


def test_cli_usage_errors(tmp_path):
    assert _cli().returncode == 106
    assert _cli("frobnicate").returncode == 109
    assert _cli("gen-synthetic", "-n", 5).returncode == 106  # --out required
    assert _cli("gen-synthetic", "-n", "x", "--out", tmp_path / "a").returncode == 104
    assert _cli("fit", "--in", "a", "--alpha", 1, "--model", "m").returncode == 1  # missing refs: error line
    r = _cli("fit", "--in", tmp_path / "missing.xyz", "--alpha", 1, "--refs-grid", 4, "--model", tmp_path / "m")
    assert r.returncode == 1 and r.stderr.startswith("error: cannot open")
    r = _cli("fit", "--in", "a", "--alpha", 1, "--refs-grid", 4, "--refs-file", "b", "--model", "m")
    assert r.returncode == 108
    assert _cli("--help").returncode == 0


@pytest.mark.gpu
def test_cli_fit_and_eval_readme_case(golden, tmp_path):
    """The README walk-through (proj/README.md:62-76) through the CLI: gen-synthetic,
    fit on an 81-point grid with alpha 0.5, eval with values; the model file
    loads back and the error lines agree between fit and eval."""
    xyz, model = tmp_path / "franke.xyz", tmp_path / "model.txt"
    assert _cli("gen-synthetic", "-n", 1089, "--out", xyz).returncode == 0
    r = _cli("fit", "--in", xyz, "--kernel", "wendland-3-1", "--alpha", 0.5, "--refs-grid", 81, "--model", model)
    assert r.returncode == 0, r.stderr
    kv = dict(line.split(" ", 1) for line in r.stdout.strip().splitlines())
    assert kv["points"] == "1089" and kv["refs"] == "81" and kv["design-nnz"] == "88209"
    assert kv["n-blocks"] == "1" and kv["empty-support-refs"] == "0"
    assert float(kv["mae"]) == pytest.approx(float(golden("readme_case")["published_mae"]), rel=1e-4)
    assert "assembly:" in r.stderr
    m = io.load_model(model)
    assert len(m.refs) == 81 and m.kernel.alpha == 0.5
    errs = tmp_path / "errors.txt"
    r2 = _cli("eval", "--model", model, "--in", xyz, "--out", errs)
    assert r2.returncode == 0, r2.stderr
    kv2 = dict(line.split(" ", 1) for line in r2.stdout.strip().splitlines())
    assert float(kv2["mae"]) == pytest.approx(float(kv["mae"]), rel=1e-12)
    rows = np.loadtxt(errs)
    assert rows.shape == (1089, 5)
    np.testing.assert_allclose(rows[:, 4], rows[:, 3] - rows[:, 2], rtol=0, atol=1e-15)
