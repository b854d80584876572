#!/bin/bash
# verifier SpMV lanes per row / column (SFDG_VG_LANES) and the two-blocks-per-SM B' stream:
# warm per-kernel durations (ncu, one lane) and the c4 step (20 flushes)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "verif" 2>&1 | tail -1
for G in 16 8 32; do
  SFDG_VG_LANES=$G SFDG_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"vg_" --csv \
    --log-file gpurun_out/vg_warm_$G.csv python bench.py --config c4 --rows 150000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > /dev/null 2>&1
  python - <<PY
import csv,collections
rows=list(csv.reader(open("gpurun_out/vg_warm_$G.csv")))
h=[r for r in rows if r and r[0]=="ID"][0]; ii={x:i for i,x in enumerate(h)}
agg=collections.defaultdict(list)
for r in rows:
    if len(r)==len(h) and r[0]!="ID" and r[ii["Metric Name"]]=="gpu__time_duration.sum":
        agg[r[ii["Kernel Name"]][:36]].append(float(r[ii["Metric Value"]].replace(",","")))
print("G=$G", "  ".join("%s %d %.1fus"%(k.split('::')[-1][:18],len(v),sum(v)/len(v)/1e3) for k,v in agg.items() if len(v)>20))
PY
  SFDG_VG_LANES=$G timeout 600 python bench.py --config c4 --rows 1000000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/vg_ab.json 2>/dev/null
  echo "G=$G c4 20 flushes: $(python -c "import json;d=json.load(open('gpurun_out/vg_ab.json'));print(round(d['ms_per_step'],1))")"
done
