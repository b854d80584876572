#!/bin/bash
# c5 shard under kappa targets and lane counts; the probe's measured per-sweep growth
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
run() {
  env "$@" timeout 900 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/c5k.json 2>gpurun_out/c5k.err
  echo "$* : $(python -c "import json;d=json.load(open('gpurun_out/c5k.json'));print(round(d['ms_per_step'],1), d['kernels']['gram']['launches'], d['attempts_per_step_rank0'])" 2>&1 | tail -1)"
  grep "sfdg probe" gpurun_out/c5k.err | sort | uniq -c | head -12
}
run SFDG_DEBUG_KAPPA=1
run SFDG_DEBUG_KAPPA=1 SFDG_KAPPA_TARGET=1e5
run SFDG_LANES=2
run SFDG_LANES=4
timeout 300 tools/kbench 1000000 256 20 10 2>&1 | grep -E "gram|trsm|gemm|spmm"
timeout 300 tools/kbench 50000 128 50 100 2>&1 | grep -E "gram|trsm|gemm|spmm"
