#!/bin/bash
# Round 2, session 5: the big-panel configurations on the final SpMM (pieces by ticket, L2-window
# piece length, two-level sums): c5 shard and c3 bench lines, configs[4] whole on one B200, and a
# full ncu capture of one CSR and one CSC launch at c5.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/r02f_bench_c5_shard.json 2> gpurun_out/r02f_bench_c5_shard.err; echo "c5 shard rc $?"
timeout 1500 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy > gpurun_out/r02f_bench_c3_full.json 2> gpurun_out/r02f_bench_c3_full.err; echo "c3 rc $?"
SECONDS=0; timeout 2400 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/r02f_bench_c5_full_1gpu.json 2> gpurun_out/r02f_bench_c5_full.err
echo "c5 full rc $? wall ${SECONDS}s"
SFDG_LANES=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"spmm_kernel" -s 8 -c 2 \
  -o gpurun_out/r02f_c5_spmm -f python bench.py --config c5 --rows 1000000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  --no-accuracy --no-isolated > gpurun_out/r02f_ncu_c5.log 2>&1
echo "ncu rc $?"
for f in r02f_bench_c5_shard r02f_bench_c3_full r02f_bench_c5_full_1gpu; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));r=d['roofline']
print('$f', round(d['ms_per_step'],1), '%.4g'%d['value'], (d.get('e2e') or {}).get('value'), d['flushes_per_step_rank0'], d['attempts_per_step_rank0'], r['frac'], r.get('isolated',{}).get('spmm',{}).get('frac'), {k:(round(v['ms']),v['launches']) for k,v in d['kernels'].items() if v['ms']>100})"; done
