"""One line per bench JSON log: tile/bin ms, frac, value, layout."""
import json
import sys

for f in sys.argv[1:]:
    line = None
    for ln in open(f):
        if ln.startswith("{"):
            line = json.loads(ln)
    if not line:
        print(f, "NO JSON")
        continue
    r = line.get("roofline") or {}
    lay = line["config"].get("layout", {})
    print(f"{f}: tile={r.get('tile_ms', 0):.4f}ms bin={r.get('bin_ms', 0):.4f}ms frac={r.get('frac', 0):.3f} "
          f"val={line['value']:.3g} e2e={line['e2e']['value']:.3g} q={lay.get('sub_div')} S={lay.get('super_factor')} "
          f"Ls={lay.get('mean_super_centres')}/{lay.get('max_super_centres')} "
          f"Lsub={lay.get('mean_sub_centres')}/{lay.get('max_sub_centres')} nb={lay.get('n_buckets')} fb={lay.get('n_fallback')}")
