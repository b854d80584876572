#!/bin/bash
# c5 shard with an L2 persisting window over the CSR gather's first MB of W (SFDG_L2_WINDOW)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for W in 0 32 64 96; do
  SFDG_L2_WINDOW=$W timeout 900 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/l2w.json 2>gpurun_out/l2w.err
  echo "window $W MB: $(python -c "import json;d=json.load(open('gpurun_out/l2w.json'));print(round(d['ms_per_step'],1), round(d['kernels']['spmm']['ms']), d['kernels']['spmm']['launches'])" 2>&1 | tail -1)"
done
bash tools/torchrun_dry.sh
