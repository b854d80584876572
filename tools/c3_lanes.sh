#!/bin/bash
# c3 lane count (panels 160 MB > L2) and the whole c3 stream
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for L in 2 3 4; do
  SFDG_LANES=$L timeout 900 python bench.py --config c3 --rows 600000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/c3L.json 2>/dev/null
  echo "c3 600k rows lanes $L: $(python -c "import json;d=json.load(open('gpurun_out/c3L.json'));print(round(d['ms_per_step'],1), d['flushes_per_step_rank0'])")"
done
timeout 1500 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c3_full.json 2> gpurun_out/bench_c3_full.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c3_full.json'));print('c3 full', round(d['ms_per_step'],1), '%.3g'%d['value'], d['e2e']['value'], d['flushes_per_step_rank0'], d['attempts_per_step_rank0'], d['roofline']['frac'], d['roofline'].get('l2_gather',{}).get('frac'), d['roofline'].get('isolated',{}).get('spmm',{}))" || tail -3 gpurun_out/bench_c3_full.err
