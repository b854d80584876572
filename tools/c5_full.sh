#!/bin/bash
# BASELINE configs[4] (5e7 rows, d = 1e6, ell = 256, ~1.05e9 nnz) sketched whole on ONE B200
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
free -g | head -2; nproc
SECONDS=0; timeout 2400 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/bench_c5_full.json 2> gpurun_out/bench_c5_full.err
echo "rc $? wall ${SECONDS}s"
python -c "
import json;d=json.load(open('gpurun_out/bench_c5_full.json'));print('c5 full', round(d['ms_per_step'],1), '%.3g'%d['value'], d['flushes_per_step_rank0'], d['attempts_per_step_rank0'], d['nnz_per_step'], {k:(round(v['ms']),v['launches']) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/bench_c5_full.err
