"""bench.py's contract on CPU: the reference arm's JSON line, its
independence from this package's libraries, and the pinned config table."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_config_table_matches_package():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1806_07884_b200 import configs
    for name, c in bench.CFG.items():
        p = configs.CONFIGS[name]
        assert (p.n, p.m, p.dim, p.kernel) == (c["n"], c["m"], c["dim"], c["kernel"])
        assert p.alpha == bench.alpha_of(name)
    assert bench.DEFAULT_CONFIG == "cfg5"


def test_reference_window_inputs_equal_the_config_points():
    """The reference arm's window sample (built from the reference's own
    radical_inverse / franke and the restated noise) is the config's own
    points at those sequence positions."""
    sys.path.insert(0, str(ROOT))
    import numpy as np

    import bench
    from paper_1806_07884_b200 import configs
    xy, h, refs, _ = bench.reference_window("cfg5")
    for k in (0, 1, 777, len(h) - 1):
        pxy, ph = configs.points("cfg5", n=1, start=432 * (k + 1) - 1)
        assert np.array_equal(xy[k], pxy[0])
        assert abs(h[k] - ph[0]) <= 1e-18
    r = 1.0 / bench.alpha_of("cfg5")
    assert refs[:, 0].min() > -r and refs[:, 0].max() < 1 / 16 + r


def test_reference_arm_line_and_no_package_library():
    code = (
        "import sys, json, io, contextlib; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'cfg1',"
        " '--steps', '1', '--warmup', '0']; sys.path.insert(0, %r); import bench; bench.main();"
        "maps = open('/proc/self/maps').read();"
        "assert 'paper_1806_07884_b200' not in maps, 'package library loaded';"
        "assert not any(m.startswith('paper_1806_07884_b200') for m in sys.modules)" % str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    sys.path.insert(0, str(ROOT))
    import bench
    assert line["config"] == json.loads(json.dumps(bench.workload("cfg1")))
