#!/bin/bash
# Round-2 final evidence: GPU tests, smoke, the default bench (c4), c2, the c4 launch list and a
# full ncu capture of the c4 SpMM, all on the final build.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/final_gpu_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/final_smoke.log
timeout 1200 python bench.py > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err; echo "bench rc $?"
timeout 900 python bench.py --config c2 > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err; echo "bench c2 rc $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c4.csv \
  python bench.py --config c4 --rows 200000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/final_launches.log 2>&1
echo "launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_kernel" -s 200 -c 4 \
  -o gpurun_out/r02_final_c4_spmm -f python bench.py --config c4 --rows 200000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  --no-accuracy --no-isolated > gpurun_out/final_ncu_full.log 2>&1
echo "ncu full rc $?"
for f in final_bench_c4 final_bench_c2; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));r=d['roofline']
print('$f', round(d['ms_per_step'],1), '%.4g'%d['value'], '%.4g'%d['e2e']['value'], r['frac'], r.get('traffic'), r.get('l2_gather',{}).get('frac'), r.get('isolated',{}).get('spmm',{}).get('frac'), d.get('clocks'), d.get('cpu_baseline',{}).get('value'), d.get('accuracy',{}).get('cov_err'))"; done
