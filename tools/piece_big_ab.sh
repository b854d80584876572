#!/bin/bash
# Piece length / grid size of the SpMM for gathered panels larger than L2 (c5, c3): ncu DRAM bytes
# and duration of one CSR and one CSC launch, then whole-step times.
# (the fourth field, var, drove an experiment whose code was removed: leave it 0)
# Usage: piece_big_ab.sh "<piece:blocks:dyn> ..." [c3]   (piece 0 = default length; dyn 1 = pieces by ticket)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
OUT=gpurun_out/piece_big_ab.txt
: > $OUT
for V in ${1:-0:16:0 128:16:1 64:16:1}; do
  IFS=: read P B D VAR <<< "$V"; export SFDG_PIECE_VAR=${VAR:-0}; if [ "$D" = x ]; then unset SFDG_SPMM_DYN; else export SFDG_SPMM_DYN=$D; fi
  SFDG_PIECE_BIG=$P SFDG_SPMM_BLOCKS=$B SFDG_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"spmm_kernel" -s 8 -c 2 --csv --log-file gpurun_out/pb_c5_${P}_${B}_${D}_${VAR:-0}.csv \
    python bench.py --config c5 --rows 1000000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > /dev/null 2>&1
  python - <<PY >> $OUT
import csv
rows=list(csv.reader(open("gpurun_out/pb_c5_${P}_${B}_${D}_${VAR:-0}.csv")))
h=[r for r in rows if r and r[0]=="ID"][0]; ii={x:i for i,x in enumerate(h)}
cur={}
for r in rows:
    if len(r)==len(h) and r[0]!="ID":
        cur.setdefault(r[0],{})[r[ii["Metric Name"]].split('.')[0]]=r[ii["Metric Value"]]
for k,v in cur.items(): print("c5 piece=$P blocks=$B dyn=$D var=${VAR:-0} launch", k, v)
PY
  SFDG_PIECE_BIG=$P SFDG_SPMM_BLOCKS=$B timeout 900 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/pb.json 2>/dev/null
  echo "c5 shard piece=$P blocks=$B dyn=$D var=${VAR:-0}: $(python -c "import json;d=json.load(open('gpurun_out/pb.json'));print(round(d['ms_per_step'],1), 'ms; spmm', round(d['kernels']['spmm']['ms'],1), 'ms over', d['kernels']['spmm']['launches'])")" >> $OUT
  [ "$2" = c3 ] && SFDG_PIECE_BIG=$P SFDG_SPMM_BLOCKS=$B timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/pb3.json 2>/dev/null
  [ "$2" = c3 ] && echo "c3 piece=$P blocks=$B dyn=$D var=${VAR:-0}: $(python -c "import json;d=json.load(open('gpurun_out/pb3.json'));print(round(d['ms_per_step'],1), 'ms; spmm', round(d['kernels']['spmm']['ms'],1), 'ms over', d['kernels']['spmm']['launches'])")" >> $OUT
done
cat $OUT
