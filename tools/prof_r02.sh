#!/bin/bash
# Round-2 measurement recipe (run under gpurun from the repo root):
#  1. c4 (1M rows = 20 flushes) with SFDG_TRACE at 4 and 1 lanes -> per-phase busy fractions
#  2. ncu launch list of a short c4 bench (per-kernel launch counts and cold serialised times)
#  3. ncu --set full of the c4 SpMM (both directions) and the Gram / TRSM kernels
set -x
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for L in 4 1; do
  SFDG_LANES=$L SFDG_TRACE=gpurun_out/tr_c4_L$L.jsonl timeout 600 python bench.py --config c4 --rows 1000000 --steps 1 --warmup 1 \
     --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/lanes_c4_L$L.json 2>&1
  python tools/trace_report.py gpurun_out/tr_c4_L$L.jsonl > gpurun_out/trace_c4_L$L.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --config c4 --rows 200000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated \
  > gpurun_out/launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_kernel|gram_tn|tsmm|trinv" -s 200 -c 8 \
  -o gpurun_out/r02b_c4_full -f python bench.py --config c4 --rows 200000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  --no-accuracy --no-isolated > gpurun_out/ncu_full_c4.log 2>&1
echo done
