#!/bin/bash
# c5 SpMM DRAM traffic per launch on the current build (one flush of d = 1e6, ell = 256)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SFDG_LANES=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:"spmm_kernel" -s 8 -c 6 --csv --log-file gpurun_out/c5_spmm_dram.csv \
  python bench.py --config c5 --rows 1000000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/c5_spmm_dram.log 2>&1
echo "rc $?"
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/c5_spmm_dram.csv")))
h=[r for r in rows if r and r[0]=="ID"][0]; ii={x:i for i,x in enumerate(h)}
cur={}
for r in rows:
    if len(r)==len(h) and r[0]!="ID":
        cur.setdefault(r[0],{})[r[ii["Metric Name"]]]=(r[ii["Metric Value"]],r[ii["Metric Unit"]])
for k,v in cur.items(): print(k, v)
PY
