#!/bin/bash
# kappa target 1e5 (SFDG_KAPPA_TARGET): full-size parity against the reference, the fuzz, and the
# benches of c5 / c4 / c2 under it
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
export SFDG_KAPPA_TARGET=1e5
timeout 1500 python -m pytest tests/test_fullsize_parity.py tests/test_gpu_parity.py tests/test_wide_ell.py -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python tools/fuzz_parity.py --cases 300 --seed 71 > gpurun_out/fuzz_k5.txt 2>&1; tail -2 gpurun_out/fuzz_k5.txt
timeout 900 python tools/fuzz_parity.py --cases 30 --seed 72 --big --max-d 1200 > gpurun_out/fuzz_k5_big.txt 2>&1; tail -2 gpurun_out/fuzz_k5_big.txt
for c in c5 c4 c2; do
  R=""; if [ $c = c5 ]; then R="--rows 6250000 --steps 1 --warmup 1"; else R="--steps 2 --warmup 3"; fi
  timeout 900 python bench.py --config $c $R --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/bench_k5_$c.json 2> gpurun_out/bench_k5_$c.err
  python -c "
import json;d=json.load(open('gpurun_out/bench_k5_$c.json'));print('$c', round(d['ms_per_step'],1), '%.3g'%d['value'], d.get('e2e',{}).get('value'), d['attempts_per_step_rank0'], d['kernels']['gram']['launches'])" || tail -3 gpurun_out/bench_k5_$c.err
done
