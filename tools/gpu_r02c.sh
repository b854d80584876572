#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc $?"
tail -25 gpurun_out/gpu_tests.log
timeout 1200 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/bench_c5_shard.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for f in bench_c5_shard bench_c4 bench_c2; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['ms_per_step'], '%.3g'%d['value'], d.get('e2e',{}).get('value'), d['flushes_per_step_rank0'], d['attempts_per_step_rank0'], {k:(round(v['ms']),v['launches']) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/$f.err; done
