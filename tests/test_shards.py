"""Multi-rank host logic of the sharded sketch + log2 merge tree, on CPU with gloo.

The GPU run uses the same tree code with NCCL and the device merge (bench.py); here the
transport is gloo and each shard is sketched by the CPU oracle, so the merged result
must equal the single-process replay of the same tree bit for bit.
"""
import os
import socket

import numpy as np
import pytest

from paper_1602_00412_b200 import shards

D, ELL, N = 60, 8, 480


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(world, rank):
    from oracle.oracle import Oracle
    from paper_1602_00412_b200 import synthetic as S
    O = Oracle()
    g = O.rng(4242)
    rp, cs, vs = S.random_sparse(g, N, D, 0.15)
    r0, r1 = S.shard_rows(N, world, rank)
    srp = rp[r0:r1 + 1] - rp[r0]
    b, _ = O.sketch(srp, cs[rp[r0]:rp[r1]], vs[rp[r0]:rp[r1]], D, ELL, seed=100 + rank)
    return b


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    local = torch.from_numpy(_shard(world, rank))

    def send(t, peer):
        dist.send(t.contiguous(), dst=peer)

    def recv(peer):
        t = torch.empty((ELL, D), dtype=torch.float64)
        dist.recv(t, src=peer)
        return t

    def merge(a, b):
        return torch.from_numpy(O.merge(a.numpy(), b.numpy(), ELL))

    out = shards.merge_tree(local, rank, world, send, recv, merge)
    if rank == 0:
        np.save(os.path.join(outdir, f"merged_{world}.npy"), out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_tree_plan_is_a_tree(world):
    sends = {}
    recvs = []
    for r in range(world):
        plan = shards.tree_plan(r, world)
        s = [p for p in plan if p[1] == "send"]
        assert len(s) == (0 if r == 0 else 1)
        if s:
            sends[r] = s[0][2]
        recvs += [(p[2], r) for p in plan if p[1] == "recv"]
    assert sorted(recvs) == sorted(sends.items())


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_merge_tree_matches_replay(tmp_path, world):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    from oracle.oracle import Oracle
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / f"merged_{world}.npy")
    O = Oracle()
    want = shards.replay_tree([_shard(world, r) for r in range(world)], lambda a, b: O.merge(a, b, ELL))
    assert np.array_equal(got, want)
    # the merged sketch still satisfies the covariance bound (tests/acceptance.cpp:420-445)
    from paper_1602_00412_b200 import synthetic as S
    g = O.rng(4242)
    rp, cs, vs = S.random_sparse(g, N, D, 0.15)
    a = np.zeros((N, D))
    for i in range(N):
        a[i, cs[rp[i]:rp[i + 1]]] = vs[rp[i]:rp[i + 1]]
    assert np.linalg.norm(a.T @ a - got.T @ got, 2) <= (a ** 2).sum() / ((6 / 41) * ELL)
