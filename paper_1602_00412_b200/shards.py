"""Row-sharded sketching and the log2 merge-shrink tree.

FD sketches are mergeable (PAPER.md; reference merge = dense_shrink(vstack(b1, b2)),
core/src/sketch.cpp:80-83; "shard the stream across workers, sketch
independently (distinct seeds), merge pairwise"). Each rank sketches a contiguous shard
with seed + rank; sketches then meet in a binary tree: at level L (step = 2^L) rank r
with r % 2^(L+1) == 2^L sends its B to r - 2^L, which merges (lower rank stacked first).
The tree order is fixed, so for a given world size the result is deterministic and the
CPU oracle can replay it exactly (tests/test_shards.py).

Transport is pluggable: NCCL send/recv of device tensors in bench.py (B^T, d x ell FP64,
merged on device by sfdg_merge_device), gloo on CPU tensors in the tests.
"""
from __future__ import annotations

from typing import Callable, List, Tuple


def tree_plan(rank: int, world: int) -> List[Tuple[int, str, int]]:
    """[(step, 'recv'|'send', peer), ...] for this rank, in execution order."""
    plan = []
    step = 1
    while step < world:
        if rank % (2 * step) == step:
            plan.append((step, "send", rank - step))
            break
        if rank % (2 * step) == 0 and rank + step < world:
            plan.append((step, "recv", rank + step))
        step *= 2
    return plan


def merge_tree(local, rank: int, world: int, send: Callable, recv: Callable, merge: Callable):
    """Runs this rank's part of the tree. Returns the merged sketch on rank 0, else None."""
    cur = local
    for _step, role, peer in tree_plan(rank, world):
        if role == "send":
            send(cur, peer)
            return None
        other = recv(peer)
        cur = merge(cur, other)
    return cur


def replay_tree(sketches: list, merge: Callable):
    """Single-process replay of the same tree over per-shard sketches (oracle side)."""
    world = len(sketches)
    cur = list(sketches)
    step = 1
    while step < world:
        for r in range(0, world, 2 * step):
            if r + step < world:
                cur[r] = merge(cur[r], cur[r + step])
        step *= 2
    return cur[0]
