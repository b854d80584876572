#!/bin/bash
# Launch list (durations, DRAM bytes) of the verifier kernels of one c5 flush, one lane.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SFDG_LANES=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"vg_|verify|vcost|vstate|vdec" --csv --log-file gpurun_out/c5_verify_launches.csv \
  python bench.py --config c5 --rows 1000000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/c5_verify.log 2>&1
echo "rc $?"
python - <<'PY'
import csv, collections
rows=list(csv.reader(open("gpurun_out/c5_verify_launches.csv")))
h=[r for r in rows if r and r[0]=="ID"][0]; ii={x:i for i,x in enumerate(h)}
acc=collections.defaultdict(lambda: collections.defaultdict(float)); cnt=collections.Counter()
for r in rows:
    if len(r)==len(h) and r[0]!="ID":
        k=r[ii["Kernel Name"]].split("(")[0][-48:]
        m=r[ii["Metric Name"]]; v=float(r[ii["Metric Value"]].replace(",",""))
        acc[k][m]+=v
        if m.startswith("gpu__time"): cnt[k]+=1
for k,v in sorted(acc.items(), key=lambda kv:-kv[1]["gpu__time_duration.sum"]):
    n=cnt[k]; t=v["gpu__time_duration.sum"]
    print(f"{k:50s} n={n:5d} total {t/1e6:8.2f} ms  mean {t/n/1e3:8.1f} us  dram rd {v['dram__bytes_read.sum']/n/1e6:9.1f} MB wr {v['dram__bytes_write.sum']/n/1e6:8.1f} MB per launch")
PY
