#!/bin/bash
# SpMM windowed pieces (default for panels > L2) vs plain pieces (SFDG_PIECE_ORDER=0)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spmm_paths.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "window or piece or family or wide or c5" 2>&1 | tail -2
for P in 1 0; do
  SFDG_PIECE_ORDER=$P SFDG_LANES=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"spmm_kernel" -s 8 -c 2 --csv --log-file gpurun_out/po_c5_$P.csv \
    python bench.py --config c5 --rows 1000000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/po_c5_$P.csv")))
h=[r for r in rows if r and r[0]=="ID"][0]; ii={x:i for i,x in enumerate(h)}
cur={}
for r in rows:
    if len(r)==len(h) and r[0]!="ID":
        cur.setdefault(r[0],{})[r[ii["Metric Name"]].split('.')[0]]=r[ii["Metric Value"]]
for k,v in cur.items(): print("c5 porder=$P", k, v)
PY
done
for P in 1 0; do
  SFDG_PIECE_ORDER=$P timeout 900 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/po.json 2>/dev/null
  echo "c5 shard porder=$P: $(python -c "import json;d=json.load(open('gpurun_out/po.json'));print(round(d['ms_per_step'],1))")"
  SFDG_PIECE_ORDER=$P timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/po3.json 2>/dev/null
  echo "c3 porder=$P: $(python -c "import json;d=json.load(open('gpurun_out/po3.json'));print(round(d['ms_per_step'],1))")"
done
