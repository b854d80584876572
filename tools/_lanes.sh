cd $GRAFT_REPO_ROOT
for L in 1 2 4 6; do
  SFDG_LANES=$L SFDG_TRACE=gpurun_out/tr_L$L.jsonl timeout 600 python bench.py --config c4 --rows 1000000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-accuracy --no-isolated > gpurun_out/lanes_L$L.json 2>&1
  echo "L=$L"; python -c "
import json;d=json.load(open('gpurun_out/lanes_L$L.json'));print(d['ms_per_step'], {k:(round(v['ms']),v['launches']) for k,v in d['kernels'].items()})"
  python tools/trace_report.py gpurun_out/tr_L$L.jsonl
done
