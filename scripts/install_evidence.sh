# usage: bash scripts/install_evidence.sh TAG -- copy the outputs of `scripts/gpu_round2.sh TAG`
# (gpurun_out/TAG_*) into profiles/r02_* (the tracked evidence) and rebuild profiles/traffic.json
TAG=$1
G=gpurun_out
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do grep '^{' $G/${TAG}_bench_$c.log | tail -1 > profiles/r02_bench_$c.json; done
grep '^{' $G/${TAG}_ref_cfg5.log | tail -1 > profiles/r02_ref_cfg5.json
grep '^cfg4' $G/${TAG}_cfg4_both.log > profiles/r02_cfg4_both_ways.txt
cp $G/${TAG}_launches_cfg5.txt profiles/r02_launches_cfg5_bench.txt
{ head -2 profiles/r02_ncu_all_kernels.md | sed "s/run r[0-9a-z]* = final code/run ${TAG} = final code/"; cat $G/${TAG}_all_table.md; } > /tmp/_all.md && mv /tmp/_all.md profiles/r02_ncu_all_kernels.md
for c in cfg2 cfg3 cfg4 cfg5; do cp $G/${TAG}_asm_${c}_summary.txt profiles/r02_ncu_asm_$c.txt; done
cp $G/${TAG}_scatter_cfg5_summary.txt profiles/r02_ncu_bin_scatter_cfg5.txt
python scripts/make_traffic.py $TAG
# the bench lines read profiles/traffic.json at run time (the previous capture): stamp the capture of this run
python - <<'PY'
import json
t = json.load(open("profiles/traffic.json"))
for c, v in t.items():
    p = f"profiles/r02_bench_{c}.json"
    d = json.loads(open(p).read())
    d["roofline"]["traffic"] = v
    open(p, "w").write(json.dumps(d) + "\n")
PY
