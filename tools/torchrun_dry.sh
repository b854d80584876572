#!/bin/bash
# Functional dry run of bench.py's multi-rank path on ONE GPU (two ranks, gloo transport for the
# tree): both ranks sketch their shard, the tree merges rank 1 into rank 0, rank 0 prints the
# line. Not a scaling measurement (two ranks share one GPU).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SFDG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --config c4 --rows 100000 --steps 1 --warmup 1 > gpurun_out/dry2.json 2> gpurun_out/dry2.err
echo "rc $?"; tail -c 600 gpurun_out/dry2.json; echo; tail -5 gpurun_out/dry2.err
SFDG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --impl reference --gpus 2 --config c4 --steps 1 --warmup 1 > gpurun_out/dry2_ref.json 2> gpurun_out/dry2_ref.err
echo "ref rc $?"; tail -c 400 gpurun_out/dry2_ref.json
