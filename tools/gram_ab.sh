#!/bin/bash
# Gram A/B: TMA bulk-copy stages against per-thread cp.async (SFDG_GRAM=cp), split-K waves
cd ${GRAFT_REPO_ROOT:-.}
for shape in "10000 100 10 200" "50000 128 50 100" "1000000 256 20 10"; do
  for G in tma cp; do for W in 2 3 4 6; do
    echo "== kbench $shape SFDG_GRAM=$G waves=$W: $(SFDG_GRAM_WAVES=$W SFDG_GRAM=$G timeout 600 tools/kbench $shape 2>&1 | grep -E "gram" | tr -s ' ' | tr '\n' ' ')"
  done; done
done
