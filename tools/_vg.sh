cd $GRAFT_REPO_ROOT
SFDG_LANES=1 SFDG_TRACE=gpurun_out/tr7_L1.jsonl python bench.py --config c4 --rows 1000000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/lanes7_L1.json 2>&1; python tools/trace_report.py gpurun_out/tr7_L1.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"vg_" --csv --log-file gpurun_out/vg_launches_warm.csv python bench.py --config c4 --rows 100000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/vg_ncu.log 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open("gpurun_out/vg_launches_warm.csv")))
h=[r for r in rows if r and r[0]=="ID"][0]; ii={x:i for i,x in enumerate(h)}
agg=collections.defaultdict(list)
for r in rows:
    if len(r)==len(h) and r[0]!="ID" and r[ii["Metric Name"]]=="gpu__time_duration.sum":
        agg[r[ii["Kernel Name"]][:40]].append(float(r[ii["Metric Value"]].replace(",","")))
for k,v in agg.items(): print(k, len(v), "mean %.1f us"%(sum(v)/len(v)/1e3), "max %.1f"%(max(v)/1e3))
PY
