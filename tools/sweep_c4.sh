#!/bin/bash
# c4 (1M rows = 20 flushes) under the scheduling / schedule switches: ms per step
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
run() {
  env "$@" timeout 600 python bench.py --config c4 --rows 1000000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/sw.json 2>gpurun_out/sw.err
  echo "$* : $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['ms_per_step'],1), d['kernels']['gram']['launches'], d['attempts_per_step_rank0'])" 2>&1 | tail -1)"
}
run X=0
run SFDG_VERIFY_PRIO=0
run SFDG_CHAIN_PRIORITY=1
run SFDG_KAPPA_TARGET=1e5
run SFDG_KAPPA_TARGET=1e6
run SFDG_PDL=0
run SFDG_LANES=3 SFDG_VERIFY_PRIO=0
run SFDG_HOT=1
