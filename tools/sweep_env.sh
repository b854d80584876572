#!/bin/bash
# Runs bench.py (c2, device-resident arm only) under a list of SFDG_* environment variants and
# prints one "variant value ms_per_step" line each. Usage: tools/sweep_env.sh "VAR=1 VAR2=2" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  out=$(env $v timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-accuracy 2>/dev/null | tail -1)
  python - "$v" "$out" <<'PY'
import json, sys
v, out = sys.argv[1], sys.argv[2]
try:
    d = json.loads(out); print(f"{v:60s} {d['value']:.4e} nnz/s {d['ms_per_step']:.1f} ms")
except Exception:
    print(f"{v:60s} FAILED {out[-200:]}")
PY
done
