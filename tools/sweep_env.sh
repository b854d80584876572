#!/bin/bash
# Runs bench.py (device-resident arm only) under a list of SFDG_* environment variants and
# prints one "variant value ms_per_step verify_ms spmm_ms" line each.
# Usage: CONFIG=c4 ROWS=1000000 tools/sweep_env.sh "VAR=1 VAR2=2" ...
cd "$(dirname "$0")/.."
CONFIG=${CONFIG:-c2}
ROWS=${ROWS:-0}
for v in "$@"; do
  out=$(env $v timeout 600 python bench.py --config $CONFIG --rows $ROWS --steps ${STEPS:-3} --warmup ${WARMUP:-3} \
        --no-e2e --no-cpu-baseline --no-accuracy 2>/dev/null | tail -1)
  python - "$v" "$out" <<'PY'
import json, sys
v, out = sys.argv[1], sys.argv[2]
try:
    d = json.loads(out)
    k = d.get("kernels", {})
    ex = " ".join(f"{n}={k[n]['ms']:.0f}ms/{k[n]['launches']}" for n in ("verify", "spmm", "gram", "trsm") if n in k)
    print(f"{v:50s} {d['value']:.4e} nnz/s {d['ms_per_step']:.1f} ms  {ex}")
except Exception:
    print(f"{v:50s} FAILED {out[-200:]}")
PY
done
