#!/bin/bash
# SFDG_TRACE of a full c4 stream: warm-up step, timed step, profiled step (100 flushes each);
# the report covers the timed step only (chain steps 100..199)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SFDG_TRACE=gpurun_out/tr_c4_full.jsonl timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/tr_c4_full.json 2>&1
python -c "import json;print('ms/step', json.load(open('gpurun_out/tr_c4_full.json'))['ms_per_step'])"
python tools/trace_report.py gpurun_out/tr_c4_full.jsonl 100 100
