#!/bin/bash
# c3 full-size parity + the c4 verifier's warm kernel durations against its traced wall time
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_verify_spectral.py -q -p no:cacheprovider -x -k "verif" 2>&1 | tail -3
SFDG_LANES=1 SFDG_TRACE=gpurun_out/tr_vg.jsonl timeout 600 python bench.py --config c4 --rows 300000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/vg_l1.json 2>&1
python tools/trace_report.py gpurun_out/tr_vg.jsonl
SFDG_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"vg_" --csv --log-file gpurun_out/vg_warm.csv python bench.py --config c4 --rows 150000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/vg_ncu.log 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open("gpurun_out/vg_warm.csv")))
h=[r for r in rows if r and r[0]=="ID"][0]; ii={x:i for i,x in enumerate(h)}
agg=collections.defaultdict(list)
for r in rows:
    if len(r)==len(h) and r[0]!="ID" and r[ii["Metric Name"]]=="gpu__time_duration.sum":
        agg[r[ii["Kernel Name"]][:40]].append(float(r[ii["Metric Value"]].replace(",","")))
for k,v in agg.items(): print(k, len(v), "mean %.1f us"%(sum(v)/len(v)/1e3), "max %.1f"%(max(v)/1e3))
PY
