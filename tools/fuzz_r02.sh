#!/bin/bash
# Round-2 randomized parity sweep on the final build (tools/fuzz_parity.py against the oracle)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python tools/fuzz_parity.py --cases 1200 --seed 101 > gpurun_out/fuzz_sfd.txt 2>&1; tail -1 gpurun_out/fuzz_sfd.txt
timeout 1200 python tools/fuzz_parity.py --cases 60 --seed 102 --big --max-d 1200 > gpurun_out/fuzz_big.txt 2>&1; tail -1 gpurun_out/fuzz_big.txt
timeout 600 python tools/fuzz_parity.py --cases 300 --seed 103 --mode fd > gpurun_out/fuzz_fd.txt 2>&1; tail -1 gpurun_out/fuzz_fd.txt
timeout 600 python tools/fuzz_parity.py --cases 200 --seed 104 --mode merge > gpurun_out/fuzz_merge.txt 2>&1; tail -1 gpurun_out/fuzz_merge.txt
