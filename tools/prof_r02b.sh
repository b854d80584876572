#!/bin/bash
# Round-2 state of the other configurations and the c4 lane count.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for L in 2 3 6; do
  SFDG_LANES=$L timeout 600 python bench.py --config c4 --rows 1000000 --steps 1 --warmup 1 \
     --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/lanes_c4_L$L.json 2>&1
  echo "c4 lanes $L: $(python -c "import json;print(json.load(open('gpurun_out/lanes_c4_L$L.json'))['ms_per_step'])")"
done
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c3 --rows 400000 --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy > gpurun_out/bench_c3_400k.json 2> gpurun_out/bench_c3.err
timeout 1200 python bench.py --config c5 --rows 6250000 --steps 1 --warmup 1 --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/bench_c5_shard.json 2> gpurun_out/bench_c5.err
for f in bench_c2 bench_c3_400k bench_c5_shard; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['ms_per_step'], '%.3g'%d['value'], d.get('e2e',{}).get('value'), d['roofline'].get('frac'), d['roofline'].get('gram',{}).get('frac'), {k:(round(v['ms']),v['launches']) for k,v in d['kernels'].items()})"; done
