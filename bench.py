#!/usr/bin/env python
"""bench.py -- nnz sketched/s (and rows/s) of the SFD sketch path on B200.

Workload (default): BASELINE.json configs[3] ("c4"), the largest configuration that runs on
one GPU -- n = 5e6 rows, d = 5e4, ell = 128, FP64, Geometric(mean 50) row lengths, power-law
(s = 0.9) items, mean-centred 1-5 ratings (~2.5e8 nnz), seed 3 -- as seeded synthetic data of
that recipe (paper_1602_00412_b200/synthetic.py; the reference ships no data set). One step =
sketching the whole stream (100 flushes: SparseShrink + verify + DenseShrink each) with
SfdSketcher and finalize(). `--config c2` (configs[1]) and the others select the other families.

  value : inputs already resident in HBM (append_csr_device), B left on device
  e2e   : the public host API (append_csr from pinned host CSR, finalize() to host),
          host->device copies inside the timed region

Multi-GPU (torchrun, one rank per GPU): one stream cut into contiguous row
shards, rank r sketching its shard with seed + r, then the log2 merge tree (NCCL send/recv of
B^T + device merge-shrink, lower rank stacked first); time = max over ranks.
  c1-c4: weak scaling -- the family's stream has world x n rows, n per rank;
  c5   : configs[4] itself (5e7 rows, the 8-GPU sharded stream), split over the ranks (strong).

--impl reference: the unmodified reference C++ (oracle/_ref, built from /root/reference) on
every host core, same config dict and metric. One c4 flush takes ~25 min on a core, so each
step times one power sweep of simultaneous_iteration (randsvd.cpp:39-48, the reference's own
rmatvec / matvec / orthonormalize on a flush buffer) per process and extrapolates a flush as
q+1 sweeps (the projection / svd_top / dense_shrink tail, ~3% of a reference flush, is not
counted, which favours the reference).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "nnz sketched/sec (and rows/s) at ell, 1/2/4/8 B200; SpMM HBM GB/s vs peak"
UNIT = "nnz/s"
CONFIG_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4}
DEFAULT_CONFIG = "c4"  # the largest single-GPU configuration in BASELINE.json
FP64_PEAK_TFLOPS = 36.9  # DMMA (mma.sync m8n8k4 f64) measured on this pool: profiles/r01_fp64_peak.txt
REF_BUDGET_S = 200.0  # reference arm: wall-clock budget of all timed samples together
# sustained L2 -> SM gather bandwidth of the SpMM access pattern (ell-wide FP64 panel rows at random
# row ids), measured on this pool: tools/probe_l2 16, profiles/r01c_l2_gather_sustained.txt
L2_GATHER_GBS = 19567.3


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="sfdg", choices=["sfdg", "reference"])
    p.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIG_INDEX))
    p.add_argument("--rows", type=int, default=0, help="limit rows per shard (debug only)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-accuracy", action="store_true", help="skip the whole-stream cov_err check")
    p.add_argument("--no-isolated", action="store_true", help="skip the one-lane profiled step")
    return p.parse_args()


def workload(name: str, world: int, rows_limit: int):
    """(stream, scaling, config dict) -- identical for both arms (same_config)."""
    from paper_1602_00412_b200 import synthetic as S
    base = S.CONFIGS[name]
    if name == "c5":
        n, scaling = base.n, "strong"
        shard = "configs[4]'s 5e7-row stream split into contiguous row shards"
    else:
        n, scaling = base.n * world, "weak"
        shard = f"one {world} x {base.n}-row stream of the family, a contiguous {base.n}-row shard per rank"
    if rows_limit:
        n = min(n, rows_limit * world)
    stream = S.StreamConfig(name, n, base.d, base.ell, base.seed)
    cfg = {"workload": f"{name} = BASELINE.json configs[{CONFIG_INDEX[name]}]: n={n} d={base.d} ell={base.ell} "
                       f"FP64, data seed {base.seed}; step = full-stream SfdSketcher.append + finalize"
                       + (" + log2 merge tree" if world > 1 else ""),
           "config_index": CONFIG_INDEX[name], "n": n, "d": base.d, "ell": base.ell, "seed": base.seed,
           "shards": world, "parallelism": f"row shards x{world} ({shard}), sketch seed {base.seed}+rank"
                                           + (", log2 NCCL merge-shrink tree" if world > 1 else ""),
           "l2_flush": "256 MB device write between timed steps (inputs 3 GB > 126 MB L2)"}
    return stream, scaling, cfg


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference (CPU) samples
def power_q(m: int) -> int:
    """power_iteration_count (randsvd.cpp:10-16) with the default epsilon 1/4, c_q = 1."""
    return max(1, math.ceil(math.log(max(m, 1) / 0.25) / 0.25))


_REF_CACHE = {}


def _sweep_job(args):
    """One reference power sweep over the first `rows` rows of flush `f` of config `name`,
    from a seeded Gaussian Y. Returns (seconds, nnz, rows)."""
    name, f, rows = args
    from oracle.oracle import Reference
    from paper_1602_00412_b200 import synthetic as S
    cfg = S.CONFIGS[name]
    key = (name, f, rows)
    if key not in _REF_CACHE:
        _REF_CACHE.clear()
        r0 = (f * cfg.d) % max(1, cfg.n - cfg.d + 1)
        _REF_CACHE[key] = S.generate(name, (r0, r0 + rows))
    rp, cs, vs = _REF_CACHE[key]
    y = np.random.default_rng(f).standard_normal((rows, cfg.ell))
    _, secs = Reference().power_sweep(rp, cs, vs, cfg.d, y)
    return secs, int(rp[-1]), rows


def reference_sweeps(name: str, procs: int, flush0: int, rows: int, pool=None):
    """Sweeps on `procs` processes in parallel (flushes flush0 .. flush0 + procs - 1).
    Returns (wall seconds, per-process results)."""
    jobs = [(name, flush0 + p, rows) for p in range(procs)]
    t = time.perf_counter()
    res = pool.map(_sweep_job, jobs) if pool is not None else [_sweep_job(j) for j in jobs]
    return time.perf_counter() - t, res


def sweep_rate(name: str, res) -> tuple[float, float]:
    """Extrapolated reference throughput of the processes in `res` running side by side: each
    sketches a flush in (q + 1) sweeps over its nonzeros, so its rate is nnz / ((q+1) t)."""
    from paper_1602_00412_b200 import synthetic as S
    q = power_q(S.CONFIGS[name].d)  # every flush of the five configs has m = d rows
    nnz_s = sum(r[1] / ((q + 1) * r[0]) for r in res)
    rows_s = sum(r[2] / ((q + 1) * r[0]) for r in res)
    return nnz_s, rows_s


def sample_rows(name: str, budget_s: int | float, procs: int, pool=None) -> tuple[int, float]:
    """Rows per sweep sample so that one sample takes about budget_s: a 1/16-flush calibration
    sweep, scaled linearly (MGS and the SpMV pair are linear in the rows) with a 2x margin
    for the cache effects that make small samples faster per row."""
    from paper_1602_00412_b200 import synthetic as S
    m = S.CONFIGS[name].d
    cal = max(64, m // 16)
    _, res = reference_sweeps(name, procs, 10_000, cal, pool)
    t_full = 2.0 * max(r[0] for r in res) * m / cal
    return (m if t_full <= budget_s else max(cal, int(m * budget_s / t_full))), t_full


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    import multiprocessing as mp
    from paper_1602_00412_b200 import synthetic as S
    name = a.config
    cfg = S.CONFIGS[name]
    _, scaling, config = workload(name, world, a.rows)
    procs = os.cpu_count() or 1
    q = power_q(cfg.d)
    with mp.get_context("fork").Pool(procs) as pool:
        for w in range(a.warmup):  # warm the processes (library load, page cache) on tiny sweeps
            reference_sweeps(name, procs, 20_000 + w * procs, 256, pool)
        rows, t_full = sample_rows(name, REF_BUDGET_S / max(1, a.steps), procs, pool)
        vals, rvals, walls = [], [], []
        for k in range(a.steps):
            wall, res = reference_sweeps(name, procs, k * procs, rows, pool)
            v, rv = sweep_rate(name, res)
            vals.append(v)
            rvals.append(rv)
            walls.append(wall)
    v = float(np.mean(vals))
    sample = (f"{a.steps} steps x {procs} processes x one power sweep (randsvd.cpp:39-48 through the unmodified "
              f"reference's SparseBuffer::rmatvec/matvec and orthonormalize, oracle/_ref) over {rows} of the {cfg.d} "
              f"rows of a {name} flush buffer; a flush extrapolated as q+1 = {q + 1} sweeps (EXTRAPOLATED; the "
              f"flush tail and the row-sampling's cache effects both favour the reference); est. full sweep "
              f"{t_full:.1f} s/core")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * float(np.mean(walls)), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "rows_per_sec": float(np.mean(rvals)), "config": config, "extrapolated": True,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def merge_tree(torch, dist, s, d, ell, device, rank, world):
    """log2 tree (paper_1602_00412_b200/shards.py): at level L, rank r with
    r % 2^(L+1) == 2^L sends its B^T (d x ell, FP64) to r - 2^L, which merge-shrinks it into
    its own sketch (sketch.cpp:80-83, sfdg_sketcher_merge_device: no allocation on the timed
    path), lower rank stacked first. Rank 0 ends with the merged sketch."""
    from paper_1602_00412_b200 import shards
    host = dist.get_backend() == "gloo"  # gloo (CI / single-GPU dry runs) moves host tensors
    for _step, role, peer in shards.tree_plan(rank, world):
        if role == "send":
            bt = torch.empty((d, ell), dtype=torch.float64, device=f"cuda:{device}")
            s.sketch_device_t(bt.data_ptr(), ell)
            dist.send(bt.cpu() if host else bt, dst=peer)
            return
        o = torch.empty((d, ell), dtype=torch.float64, device="cpu" if host else f"cuda:{device}")
        dist.recv(o, src=peer)
        if host:
            o = o.to(f"cuda:{device}")
        torch.cuda.synchronize(device)
        s.merge_device(o.data_ptr(), ell)


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import paper_1602_00412_b200 as P
    from paper_1602_00412_b200 import synthetic as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        local = local % max(1, torch.cuda.device_count())  # dry runs may put several ranks on one GPU
        torch.cuda.set_device(local)
        backend = os.environ.get("SFDG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    device = local
    torch.cuda.set_device(device)

    stream, scaling, config = workload(a.config, world, a.rows)
    d, ell = stream.d, stream.ell
    r0, r1 = S.shard_rows(stream.n, world, rank)
    seed = stream.seed + rank
    rp, cs, vs = S.generate_parallel(stream, (r0, r1))
    n = r1 - r0
    nnz = int(rp[-1])

    # device-resident copy (value) and pinned host copy (e2e)
    d_cols = torch.from_numpy(cs.view(np.int32)).to(f"cuda:{device}")
    d_vals = torch.from_numpy(vs).to(f"cuda:{device}")
    if not a.no_e2e:  # pinned host copies only for the e2e leg (c5 full stream: 12.6 GB)
        h_cols = torch.from_numpy(cs.view(np.int32)).pin_memory()
        h_vals = torch.from_numpy(vs).pin_memory()
        h_cs = h_cols.numpy().view(np.uint32)
        h_vs = h_vals.numpy()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")  # > 126 MB L2

    sk = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=seed), device=device)

    def step_device(s=sk, merge=True):
        s.append_csr_device(rp, d_cols.data_ptr(), d_vals.data_ptr())
        s.finalize_device()
        if world > 1 and merge:  # every rank takes part in the tree, or none does
            merge_tree(torch, dist, s, d, ell, device, rank, world)

    def step_host():
        sk.append_csr(rp, h_cs, h_vs)
        b = sk.finalize()  # B to host (the public API result)
        if world > 1:
            merge_tree(torch, dist, sk, d, ell, device, rank, world)
        return b

    def barrier():
        if world > 1:
            if dist.get_backend() == "nccl":
                dist.barrier(device_ids=[device])
            else:
                dist.barrier()

    prange = os.environ.get("SFDG_PROFILE_RANGE") == "1"  # ncu --replay-mode app-range around step 1

    def timed(fn, k):
        total = 0.0
        for it in range(k):
            sk.reset(seed)
            flush_buf.random_(0, 255)  # evict L2 between timed steps (outside the timed region)
            torch.cuda.synchronize(device)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(device)
            if prange and it == 0:
                torch.cuda.profiler.start()
            e0.record()
            fn()
            torch.cuda.synchronize(device)
            e1.record()
            if prange and it == 0:
                torch.cuda.profiler.stop()
            e1.synchronize()
            barrier()
            total += e0.elapsed_time(e1)
        t = torch.tensor([total], dtype=torch.float64,
                         device=f"cuda:{device}" if world == 1 or dist.get_backend() == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / 1e3

    for _ in range(a.warmup):
        sk.reset(seed)
        step_device()
    torch.cuda.synchronize(device)
    stats = sk.stats()

    clocks = ClockSampler(device)
    clocks.start()
    l0 = P.launch_count()
    t_dev = timed(step_device, a.steps)
    launches = (P.launch_count() - l0) // a.steps
    clk = clocks.stop()
    t_e2e = None
    if not a.no_e2e:
        sk.reset(seed)
        step_host()  # warm the host path
        t_e2e = timed(step_host, a.steps)

    # one profiled step: per-kernel-class device time with CUDA events on the library's streams
    sk.reset(seed)
    torch.cuda.synchronize(device)
    P.profile_begin()
    step_device()
    prof = P.profile_end()
    iso = None
    if rank == 0 and not a.no_isolated:
        # the same step with one flush in flight: each launch runs without the other lanes'
        # kernels beside it (its standalone duration; the pipelined step overlaps four flushes)
        os.environ["SFDG_LANES"] = "1"
        s1 = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=seed), device=device)
        del os.environ["SFDG_LANES"]
        torch.cuda.synchronize(device)
        P.profile_begin()
        step_device(s1, merge=False)  # rank 0 alone: its shard's sketch, no tree
        iso = P.profile_end()
        s1.close()
    accuracy = None
    if rank == 0 and world == 1 and not a.no_accuracy:
        # the paper's guarantee checked on the whole stream, on the device (SURVEY 8(d) accuracy
        # gate; cov_err = bench.cpp:171-183 with its default 1000 power steps, untimed)
        sk.reset(seed)
        step_device()
        b = sk.sketch()
        t0 = time.time()
        ce, _ = P.cov_err((rp, cs, vs), d, b, P.RngState(4242), iterations=1000, device=device)
        alpha = 6.0 / 41.0
        fsq = float(np.dot(vs, vs))
        # the north_star bound |A^T A - B^T B|_2 <= |A - A_k|_F^2 / (ell - k) at k = the planted
        # rank (c1, c2, c5), with |A - A_k|_F^2 from exact_tail (bench.cpp:68-137) on the device;
        # the rating / text families have no planted rank: k = 0
        kp = {"c1": 10, "c2": 20, "c5": 32}.get(a.config, 0)
        tail = P.exact_tail((rp, cs, vs), d, kp, P.RngState(4243), device=device)[0] if kp else fsq
        accuracy = {"cov_err": ce, "definition": "|A^T A - B^T B|_2 / |A|_F^2 over the whole stream (1000 "
                                                 "power steps on the device, bench.cpp:171-183)",
                    "alpha_bound_k0": 1.0 / (alpha * ell), "within_alpha_bound": bool(ce <= 1.0 / (alpha * ell)),
                    "fd_bound_k0": 1.0 / ell, "within_fd_bound": bool(ce <= 1.0 / ell),
                    "k": kp, "tail_k_over_fsq": tail / fsq,
                    "north_star_bound_k": tail / fsq / (ell - kp),
                    "within_north_star_bound": bool(ce <= tail / fsq / (ell - kp)),
                    "seconds": round(time.time() - t0, 3)}

    value = nnz_total(torch, dist, nnz, world) * a.steps / t_dev
    rows_total = stream.n if world > 1 else n
    ms_step = 1e3 * t_dev / a.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "rows_per_sec": rows_total * a.steps / t_dev, "config": config,
            "nnz_per_step": int(value * t_dev / a.steps), "flushes_per_step_rank0": stats["flushes"],
            "attempts_per_step_rank0": stats["attempts"], "gpu_launches": int(launches), "clocks": clk}
    if t_e2e is not None:
        line["e2e"] = {"value": line["nnz_per_step"] * a.steps / t_e2e, "unit": UNIT,
                       "h2d_bytes_per_step": int(nnz * 12 + (n + stats["flushes"]) * 4),
                       "d2h_bytes_per_step": int(ell * d * 8),
                       "note": "bytes of rank 0's shard (every rank copies its own)"}
    gather = 8.0 * ((ell + 7) // 8 * 8) * nnz / max(1, stats["flushes"])  # panel bytes one SpMM launch gathers
    line.update(roofline_from_profile(prof, a.config, ms_step, gather))
    if iso:
        line["roofline"]["isolated"] = isolated_roofline(iso, gather)
    if accuracy is not None:
        line["accuracy"] = accuracy
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            rows_s, t_full = sample_rows(a.config, 15.0, 1)
            wall, res = reference_sweeps(a.config, 1, 0, rows_s)
            v, _ = sweep_rate(a.config, res)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"one power sweep of the unmodified reference (oracle/_ref) over {rows_s} "
                                              f"rows of the first {a.config} flush buffer, 1 thread, {res[0][0]:.1f} s; "
                                              f"a flush extrapolated as q+1 = {power_q(d) + 1} sweeps (EXTRAPOLATED)"}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def nnz_total(torch, dist, nnz, world):
    """Stored entries over all ranks' shards (each rank sketches its own)."""
    if world == 1:
        return nnz
    t = torch.tensor([float(nnz)], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t)
    return int(t.item())


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "B200_PROFILING.md fallback 6.65 TB/s (MEASURED_PEAKS.json absent)"


def _traffic(config: str):
    """ncu dram bytes per SpMM launch for this configuration (profiles/ncu_summary.json), or None."""
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return ncu.get("spmm_dram_bytes_per_launch", {}).get(config)
    except Exception:
        return None


def l2_gather_roofline(ms: float, cnt: int, gather: float) -> dict:
    """The SpMM's own bound: every stored entry pulls one ell-wide FP64 panel row (lp * 8 bytes)
    from L2 (the panels of c1-c4 are L2-resident; L1 hits make > 1 possible), against the
    measured sustained L2 -> SM gather rate."""
    ach = gather / (ms * 1e-3 / cnt) / 1e9
    return {"bound": "l2 gather", "achieved": round(ach, 1), "peak": L2_GATHER_GBS, "unit": "GB/s",
            "frac": round(ach / L2_GATHER_GBS, 4), "gather_bytes_per_launch": gather,
            "peak_source": "tools/probe_l2 16 (profiles/r01c_l2_gather_sustained.txt)"}


def roofline_from_profile(prof: dict, config: str, ms_step: float, gather: float = 0.0) -> dict:
    """Roofline of the metric's kernel (the SpMM, HBM-bound) and the Gram (FP64 tensor) from
    the profiled step: achieved = the algorithmic bytes / flops the library declared for
    those launches (SURVEY 8(d) formulas) / their summed CUDA-event durations."""
    peaks, src = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    kern = {}
    total_ms = sum(v[0] for k, v in prof.items() if k != "rng_gen")
    for k, (ms, cnt, fl, by) in prof.items():
        kern[k] = {"ms": round(ms, 4), "launches": cnt, "share": round(ms / total_ms, 4) if total_ms else None}
        if cnt and by:
            kern[k]["alg_bytes_per_launch"] = by / cnt
            kern[k]["achieved_gbs"] = round(by / (ms * 1e-3) / 1e9, 1)
        if cnt and fl:
            kern[k]["alg_flops_per_launch"] = fl / cnt
            kern[k]["achieved_tflops"] = round(fl / (ms * 1e-3) / 1e12, 3)
    out = {"kernels": kern}
    sp = kern.get("spmm", {})
    ach = sp.get("achieved_gbs")
    out["roofline"] = {"bound": "hbm", "kernel": "spmm (CSR / CSC gather, ell-wide FP64 panels)",
                       "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4) if ach else None,
                       "traffic": _traffic(config), "peak_source": src,
                       "alg_bytes_per_launch": sp.get("alg_bytes_per_launch"),
                       "frac_of_nominal_8tbs": round(ach / 8000.0, 4) if ach else None,
                       "note": "achieved = SURVEY 8(d) bytes 12 nnz + 8 (m+1) + 8 ell (m + d) per launch / average "
                               "launch duration (CUDA events on the lane stream, four flushes in flight); traffic = "
                               "ncu dram__bytes per launch for this config (profiles/ncu_summary.json)"}
    if gather and sp.get("launches"):
        out["roofline"]["l2_gather"] = l2_gather_roofline(sp["ms"], sp["launches"], gather)
    g = kern.get("gram", {})
    if g.get("achieved_tflops"):
        out["roofline"]["gram"] = {"bound": "tensor (FP64 DMMA)", "achieved": g["achieved_tflops"],
                                   "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                                   "frac": round(g["achieved_tflops"] / FP64_PEAK_TFLOPS, 4),
                                   "flops": "n k (k+1) per Gram (distinct dot products), declared per launch",
                                   "peak_source": "profiles/r01_fp64_peak.txt (mma.sync m8n8k4 f64 probe)"}
    dom = max((k for k in prof if k != "rng_gen"), key=lambda k: prof[k][0]) if prof else None
    out["dominant_kernel"] = {"class": dom, "share_of_step": kern[dom]["share"] if dom else None}
    return out


def isolated_roofline(prof: dict, gather: float = 0.0) -> dict:
    peaks, _ = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    res = {"what": "the same profiled step with one flush in flight (SFDG_LANES=1): standalone launch durations"}
    for k, peak, unit in (("spmm", hbm, "GB/s"), ("gram", FP64_PEAK_TFLOPS, "TFLOP/s")):
        if k not in prof or not prof[k][1]:
            continue
        ms, cnt, fl, by = prof[k]
        ach = by / (ms * 1e-3) / 1e9 if unit == "GB/s" else fl / (ms * 1e-3) / 1e12
        res[k] = {"achieved": round(ach, 2), "peak": peak, "unit": unit, "frac": round(ach / peak, 4),
                  "us_per_launch": round(1e3 * ms / cnt, 2), "launches": cnt}
        if k == "spmm" and gather:
            res[k]["l2_gather"] = l2_gather_roofline(ms, cnt, gather)
    return res


if __name__ == "__main__":
    sys.exit(main())
