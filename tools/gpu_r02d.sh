#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spmm_paths.py tests/test_wide_ell.py -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 1200 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/bench_c5_shard.json 2> gpurun_out/bench_c5.err
for m in default graph; do
  if [ $m = graph ]; then export SFDG_VERIFY_MODE=graph; fi
  timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-accuracy --no-e2e --no-isolated > gpurun_out/bench_c2_$m.json 2> gpurun_out/bench_c2_$m.err
done
unset SFDG_VERIFY_MODE
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for f in bench_c5_shard bench_c2_default bench_c2_graph bench_c4; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['ms_per_step'],1), '%.3g'%d['value'], d.get('e2e',{}).get('value'), d['flushes_per_step_rank0'], d['attempts_per_step_rank0'], {k:(round(v['ms']),v['launches']) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/$f.err; done
