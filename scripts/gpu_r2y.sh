TAG=${1:-r2y}
( timeout 1800 python -m pytest tests -q -x -m gpu -k "configs or readme or small or chunked or repass or families or edge or host" ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg5 cfg4 cfg2 cfg3; do
    echo "== $c" >> gpurun_out/${TAG}_solve.log
    timeout 600 python scripts/solve_timing.py $c 2>&1 | tail -1 >> gpurun_out/${TAG}_solve.log
done
cat > /tmp/one_solve.py <<'PY'
import sys
sys.path.insert(0, ".")
from paper_1806_07884_b200 import api, configs
name = sys.argv[1]
cfg = configs.CONFIGS[name]
xy, h = configs.points(name, n=int(float(sys.argv[2])))
refs = configs.centres(name)
with api.Engine(0) as eng:
    eng.set_centres(refs, api.KernelSpec(cfg.kernel, cfg.alpha))
    eng.assemble(xy, h)
    c, d = eng.solve()
    print(d)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python /tmp/one_solve.py cfg5 4e7 > gpurun_out/${TAG}_l.log 2>&1
python scripts/summarize_launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1
rm -f gpurun_out/${TAG}_launches.csv
echo done > gpurun_out/${TAG}_done.txt
