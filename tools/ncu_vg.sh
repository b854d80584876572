#!/bin/bash
# ncu --set full of the kernel-sequence verifier's kernels on c4 (one lane)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SFDG_LANES=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"vg_rows|vg_colsum|vg_cols_kernel" -s 30 -c 6 \
  -o gpurun_out/r02e_vg_c4_full -f python bench.py --config c4 --rows 100000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  --no-accuracy --no-isolated > gpurun_out/ncu_vg.log 2>&1
echo "rc $?"; tail -3 gpurun_out/ncu_vg.log
