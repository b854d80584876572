"""Seeded synthetic row streams for the five BASELINE.json configurations.

The reference ships no generator for these families; they are defined
here from BASELINE.json's prose, deterministically from the config seed. Rows are produced
in fixed chunks of CHUNK rows, chunk c drawing from numpy.random.default_rng([seed, c]),
so any row range (a shard, or the first few flushes of a large stream) can be generated
without producing the rows before it. Output is CSR: row_ptr int64 (n+1), cols uint32
(strictly increasing per row), vals float64 -- the SparseBuffer layout (sparse.hpp:52-57).

Configs (BASELINE.json "configs"):
  c1  n=1e4  d=1e3  ell=50   rank-10 (sigma_i = 10*0.8^i) + 0.1 N, Bernoulli 1%,   seed 0
  c2  n=1e6  d=1e4  ell=100  rank-20 (sigma_i = 10*0.9^i) + 0.1 N, Bernoulli 0.1%, seed 1
  c3  n=2e6  d=1e5  ell=200  lognormal lengths, Zipf(1.1) columns, log(1+c) values, seed 2
  c4  n=5e6  d=5e4  ell=128  Geometric(mean 50) lengths, power-law(0.9) items, centred ratings, seed 3
  c5  n=5e7  d=1e6  ell=256  Poisson(20)+1 lengths, Zipf(1.05), N(0,1) + planted rank-32, seed 4
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CHUNK = 1 << 14


@dataclass(frozen=True)
class StreamConfig:
    name: str
    n: int
    d: int
    ell: int
    seed: int


CONFIGS = {
    "c1": StreamConfig("c1", 10_000, 1_000, 50, 0),
    "c2": StreamConfig("c2", 1_000_000, 10_000, 100, 1),
    "c3": StreamConfig("c3", 2_000_000, 100_000, 200, 2),
    "c4": StreamConfig("c4", 5_000_000, 50_000, 128, 3),
    "c5": StreamConfig("c5", 50_000_000, 1_000_000, 256, 4),
}


def _global_rng(cfg: StreamConfig) -> np.random.Generator:
    return np.random.default_rng([cfg.seed, 0x5FD])


def _orthonormal(rng: np.random.Generator, d: int, r: int) -> np.ndarray:
    q, _ = np.linalg.qr(rng.standard_normal((d, r)))
    return q


def _unique_rows(rng, lengths: np.ndarray, draw) -> tuple[np.ndarray, np.ndarray]:
    """Per row, `lengths[i]` distinct columns drawn by `draw(rng, k)` (rejecting repeats).
    Returns (row_ptr, sorted cols)."""
    n = lengths.size
    need = lengths.astype(np.int64).copy()
    rows_out: list[np.ndarray] = []
    cols_out: list[np.ndarray] = []
    have_rows = np.zeros(0, np.int64)
    have_cols = np.zeros(0, np.int64)
    pending = np.nonzero(need > 0)[0]
    first = True
    while pending.size:
        cnt = need[pending]
        rr = np.repeat(pending, cnt)
        cc = draw(rng, rr.size)
        allr = np.concatenate([have_rows, rr])
        allc = np.concatenate([have_cols, cc])
        key = allr * (1 << 32) + allc
        uk, first_idx = np.unique(key, return_index=True)
        have_rows = (uk >> 32).astype(np.int64)
        have_cols = (uk & 0xFFFFFFFF).astype(np.int64)
        got = np.bincount(have_rows, minlength=n)
        need = lengths - got
        pending = np.nonzero(need > 0)[0]
        first = False
    del rows_out, cols_out, first
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(have_rows, minlength=n), out=row_ptr[1:])
    return row_ptr, have_cols.astype(np.uint32)


def _bernoulli_lowrank(cfg: StreamConfig, rank: int, decay: float, p: float, r0: int, r1: int):
    g0 = _global_rng(cfg)
    V = _orthonormal(g0, cfg.d, rank)
    sig = 10.0 * decay ** np.arange(rank)
    SV = V * sig  # d x rank
    rps, css, vss = [np.zeros(1, np.int64)], [], []
    base = 0
    for c in range(r0 // CHUNK, (r1 + CHUNK - 1) // CHUNK):
        rng = np.random.default_rng([cfg.seed, c])
        lo, hi = c * CHUNK, min(cfg.n, (c + 1) * CHUNK)
        rows = hi - lo
        lengths = rng.binomial(cfg.d, p, size=rows)
        rp, cols = _unique_rows(rng, lengths, lambda r, k: r.integers(0, cfg.d, size=k))
        G = rng.standard_normal((rows, rank))
        ridx = np.repeat(np.arange(rows), np.diff(rp))
        vals = np.einsum("ij,ij->i", G[ridx], SV[cols]) + 0.1 * rng.standard_normal(cols.size)
        a, b = max(lo, r0) - lo, min(hi, r1) - lo
        rps.append(rp[a + 1:b + 1] - rp[a] + base)
        css.append(cols[rp[a]:rp[b]])
        vss.append(vals[rp[a]:rp[b]])
        base += rp[b] - rp[a]
    return np.concatenate(rps), np.concatenate(css).astype(np.uint32), np.concatenate(vss)


def _zipf_cdf(d: int, s: float) -> np.ndarray:
    w = np.arange(1, d + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    return c / c[-1]


def _draw_cdf(cdf: np.ndarray):
    def draw(rng, k):
        return np.minimum(np.searchsorted(cdf, rng.random(k), side="right"), cdf.size - 1)
    return draw


def _heavy(cfg: StreamConfig, r0: int, r1: int):
    rps, css, vss = [np.zeros(1, np.int64)], [], []
    base = 0
    if cfg.name == "c3":
        cdf = _zipf_cdf(cfg.d, 1.1)
    elif cfg.name == "c4":
        cdf = _zipf_cdf(cfg.d, 0.9)
    else:
        cdf = _zipf_cdf(cfg.d, 1.05)
    g0 = _global_rng(cfg)
    if cfg.name == "c5":
        top, rank = 5000, 32
        V = _orthonormal(g0, top, rank) * (10.0 * 0.9 ** np.arange(rank))
    for c in range(r0 // CHUNK, (r1 + CHUNK - 1) // CHUNK):
        rng = np.random.default_rng([cfg.seed, c])
        lo, hi = c * CHUNK, min(cfg.n, (c + 1) * CHUNK)
        rows = hi - lo
        if cfg.name == "c3":
            lengths = np.minimum(np.maximum(np.round(rng.lognormal(np.log(80.0), 0.8, rows)), 1), 2000).astype(np.int64)
        elif cfg.name == "c4":
            lengths = rng.geometric(1.0 / 50.0, rows).astype(np.int64)
        else:
            lengths = (rng.poisson(20.0, rows) + 1).astype(np.int64)
        lengths = np.minimum(lengths, cfg.d)
        rp, cols = _unique_rows(rng, lengths, _draw_cdf(cdf))
        nnz = cols.size
        if cfg.name == "c3":
            cnt = rng.geometric(0.5, nnz) + 1
            vals = np.log1p(cnt.astype(np.float64))
        elif cfg.name == "c4":
            ratings = rng.choice(np.arange(1, 6), size=nnz, p=[0.05, 0.1, 0.25, 0.35, 0.25]).astype(np.float64)
            ridx = np.repeat(np.arange(rows), np.diff(rp))
            means = np.bincount(ridx, weights=ratings, minlength=rows) / np.maximum(np.diff(rp), 1)
            vals = ratings - means[ridx]
        else:
            vals = rng.standard_normal(nnz)
            ridx = np.repeat(np.arange(rows), np.diff(rp))
            U = rng.standard_normal((rows, 32))
            sel = cols < 5000
            vals[sel] += np.einsum("ij,ij->i", U[ridx[sel]], V[cols[sel]])
        a, b = max(lo, r0) - lo, min(hi, r1) - lo
        rps.append(rp[a + 1:b + 1] - rp[a] + base)
        css.append(cols[rp[a]:rp[b]])
        vss.append(vals[rp[a]:rp[b]])
        base += rp[b] - rp[a]
    return np.concatenate(rps), np.concatenate(css).astype(np.uint32), np.concatenate(vss)


def generate(name: str | StreamConfig, rows: tuple[int, int] | None = None):
    """CSR of rows [r0, r1) of config `name` (default: the whole stream). A StreamConfig
    selects the family by its name with its own seed (e.g. per-shard seeds)."""
    cfg = name if isinstance(name, StreamConfig) else CONFIGS[name]
    r0, r1 = rows if rows is not None else (0, cfg.n)
    r1 = min(r1, cfg.n)
    if cfg.name == "c1":
        return _bernoulli_lowrank(cfg, 10, 0.8, 0.01, r0, r1)
    if cfg.name == "c2":
        return _bernoulli_lowrank(cfg, 20, 0.9, 0.001, r0, r1)
    return _heavy(cfg, r0, r1)


def _gen_job(args):
    cfg, r0, r1 = args
    return generate(cfg, (r0, r1))


def generate_parallel(name: str | StreamConfig, rows: tuple[int, int] | None = None, procs: int | None = None):
    """generate() over chunk-aligned row ranges in parallel processes; identical output
    (every CHUNK-row chunk draws from its own seeded generator)."""
    import os
    import multiprocessing as mp

    cfg = name if isinstance(name, StreamConfig) else CONFIGS[name]
    r0, r1 = rows if rows is not None else (0, cfg.n)
    r1 = min(r1, cfg.n)
    procs = procs or min(32, os.cpu_count() or 1)
    nchunks = (r1 - r0 + CHUNK - 1) // CHUNK
    if procs <= 1 or nchunks < 4:
        return generate(cfg, (r0, r1))
    per = max(1, (nchunks + 4 * procs - 1) // (4 * procs)) * CHUNK
    cuts = [r0] + list(range((r0 // CHUNK + 1) * CHUNK, r1, CHUNK))  # chunk boundaries inside (r0, r1)
    bounds = [r0]
    for c in cuts[1:]:
        if c - bounds[-1] >= per:
            bounds.append(c)
    bounds.append(r1)
    jobs = [(cfg, a, b) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    with mp.get_context("spawn").Pool(min(procs, len(jobs))) as pool:  # the caller may hold CUDA / threads
        parts = pool.map(_gen_job, jobs)
    rps, base = [np.zeros(1, np.int64)], 0
    for rp, _, _ in parts:
        rps.append(rp[1:] + base)
        base += int(rp[-1])
    return (np.concatenate(rps), np.concatenate([p[1] for p in parts]).astype(np.uint32),
            np.concatenate([p[2] for p in parts]))


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard of rank `rank`."""
    per = (n + world - 1) // world
    return min(n, rank * per), min(n, (rank + 1) * per)


def random_sparse(rng, m: int, d: int, fill: float):
    """tests/oracles.hpp:111-124 (random_sparse) over any object with uniform()/normal()."""
    rp, cs, vs = [0], [], []
    for _ in range(m):
        for j in range(d):
            if rng.uniform() < fill:
                cs.append(j)
                vs.append(rng.normal())
        rp.append(len(cs))
    return np.array(rp, np.int64), np.array(cs, np.uint32), np.array(vs, np.float64)
