TAG=${1:-r2q}
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
RBG_FSAI_RHO=2.0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsai_setup -c 1 -o /tmp/${TAG}_fs python /tmp/one_solve.py cfg5 4e7 > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/${TAG}_fs.ncu-rep --page raw --csv > gpurun_out/${TAG}_fs_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_fs.ncu-rep --page source --csv --print-source sass,cuda > /tmp/${TAG}_fs_src.csv 2>/dev/null
python scripts/src_hot.py /tmp/${TAG}_fs_src.csv 50 > gpurun_out/${TAG}_fs_hot.txt 2>&1
echo done > gpurun_out/${TAG}_done.txt
