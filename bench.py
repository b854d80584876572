#!/usr/bin/env python
"""bench.py -- nnz sketched/s (and rows/s) of the SFD sketch path on B200.

Workload (BASELINE.json configs[1], "c2"): n = 1e6 rows, d = 1e4, ell = 100, FP64,
rank-20 + noise, Bernoulli 0.1% (~1e7 nnz), seed 1 -- seeded synthetic data of that
recipe (paper_1602_00412_b200/synthetic.py). One step = sketching the whole stream
(100 flushes: SparseShrink + verify + DenseShrink each) with SfdSketcher and finalize().

  value : inputs already resident in HBM (append_csr_device), B left on device
  e2e   : the public host API (append_csr from pinned host CSR, finalize() to host),
          host->device copies inside the timed region
Multi-GPU (torchrun, one rank per GPU): weak scaling -- every rank sketches its own
c2-sized stream (seed 1 + rank), then the ranks' sketches are merged in a log2 tree
(NCCL send/recv + device merge-shrink). Time = max over ranks.

--impl reference: the reference C++ implementation (oracle/_ref, built from the
unmodified /root/reference sources) on all host cores (one process per core, each
sketching one flush worth of c2 rows), same metric and units.
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="sfdg", choices=["sfdg", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--rows", type=int, default=0, help="limit rows per stream (debug only)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-accuracy", action="store_true", help="skip the whole-stream cov_err check")
    return p.parse_args()


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


# ------------------------------------------------------------------ reference arm
def _ref_worker(args):
    name, r0, r1, ell, seed = args
    from oracle.oracle import Reference
    from paper_1602_00412_b200 import synthetic as S
    rp, cs, vs = S.generate(name, (r0, r1))
    R = Reference()
    t = time.perf_counter()
    R.sketch(rp, cs, vs, S.CONFIGS[name].d, ell, seed=seed)
    return time.perf_counter() - t, int(rp[-1]), r1 - r0


def reference_sample(name: str, procs: int, rows_per_proc: int):
    """Run the unmodified reference on `procs` host cores in parallel; returns (seconds, nnz, rows)."""
    import multiprocessing as mp
    from paper_1602_00412_b200 import synthetic as S
    cfg = S.CONFIGS[name]
    span = max(1, cfg.n - rows_per_proc + 1)  # wrap so every job is a full in-range sample
    jobs = [(name, (p * rows_per_proc) % span, (p * rows_per_proc) % span + rows_per_proc, cfg.ell, cfg.seed)
            for p in range(procs)]
    t = time.perf_counter()
    if procs == 1:
        res = [_ref_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_ref_worker, jobs)
    wall = time.perf_counter() - t
    return wall, sum(r[1] for r in res), sum(r[2] for r in res)


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1602_00412_b200 import synthetic as S
    cfg = S.CONFIGS[a.config]
    procs = os.cpu_count() or 1
    flush_rows = cfg.d  # every flush of this config fires on rows == d
    for _ in range(a.warmup):
        reference_sample("c1", procs, 1000)  # warm the processes/caches on a tiny sample
    total_t, total_nnz, total_rows = 0.0, 0, 0
    for _ in range(a.steps):
        t, nnz, rows = reference_sample(a.config, procs, flush_rows)
        total_t += t
        total_nnz += nnz
        total_rows += rows
    v = total_nnz / total_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * total_t / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "rows_per_sec": total_rows / total_t,
            "config": {"workload": f"{a.config}: n={cfg.n} d={cfg.d} ell={cfg.ell} seed={cfg.seed} (BASELINE.json "
                                   f"configs[1]); reference sample per step = one flush ({flush_rows} rows) on each "
                                   f"of {procs} host processes", "l2_flush": "n/a (CPU)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": "reference",
                             "sample": f"{a.steps} steps x {procs} processes x 1 flush ({flush_rows} rows of "
                                       f"{a.config}), oracle/_ref = unmodified reference core/src, -O3"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def merge_tree(P, torch, dist, s, d, ell, device, rank, world):
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

    cfg = S.CONFIGS[a.config]
    n = min(cfg.n, a.rows) if a.rows else cfg.n
    seed = cfg.seed + rank
    rp, cs, vs = S.generate(S.StreamConfig(cfg.name, cfg.n, cfg.d, cfg.ell, seed), (0, n))
    nnz = int(rp[-1])
    d, ell = cfg.d, cfg.ell

    # device-resident copy (value) and pinned host copy (e2e)
    d_cols = torch.from_numpy(cs.view(np.int32)).to(f"cuda:{device}")
    d_vals = torch.from_numpy(vs).to(f"cuda:{device}")
    h_cols = torch.from_numpy(cs.view(np.int32)).pin_memory()
    h_vals = torch.from_numpy(vs).pin_memory()
    h_cs = h_cols.numpy().view(np.uint32)
    h_vs = h_vals.numpy()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")  # > 126 MB L2

    sk = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=seed), device=device)

    def step_device():
        sk.append_csr_device(rp, d_cols.data_ptr(), d_vals.data_ptr())
        sk.finalize_device()
        if world > 1:
            merge_tree(P, torch, dist, sk, d, ell, device, rank, world)

    def step_host():
        sk.append_csr(rp, h_cs, h_vs)
        b = sk.finalize()  # B to host (the public API result)
        if world > 1:
            merge_tree(P, torch, dist, sk, d, ell, device, rank, world)
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
    pstats = sk.stats()
    accuracy = None
    if rank == 0 and world == 1 and not a.no_accuracy:
        # the paper's guarantee checked on the whole stream, on the device (SURVEY 8(d) accuracy
        # gate; cov_err = bench.cpp:171-183 with its default 1000 power steps, untimed)
        b = sk.sketch()
        t0 = time.time()
        ce, _ = P.cov_err((rp, cs, vs), d, b, P.RngState(4242), iterations=1000, device=device)
        alpha = 6.0 / 41.0
        fsq = float(np.dot(vs, vs))
        # the north_star bound at k = the planted rank: |A^T A - B^T B|_2 <= |A - A_k|_F^2 / (ell - k),
        # with |A - A_k|_F^2 from exact_tail (bench.cpp:68-137) on the device
        kp = {"c1": 10, "c2": 20, "c5": 32}.get(a.config, 0)
        tail, _, sweeps, _ = P.exact_tail((rp, cs, vs), d, kp, P.RngState(4243), device=device)
        accuracy = {"cov_err": ce, "definition": "|A^T A - B^T B|_2 / |A|_F^2 over the whole stream (1000 "
                                                 "power steps on the device, bench.cpp:171-183)",
                    "alpha_bound_k0": 1.0 / (alpha * ell), "within_alpha_bound": bool(ce <= 1.0 / (alpha * ell)),
                    "fd_bound_k0": 1.0 / ell, "within_fd_bound": bool(ce <= 1.0 / ell),
                    "k_planted": kp, "tail_k_over_fsq": tail / fsq, "exact_tail_sweeps": sweeps,
                    "north_star_bound_k": tail / fsq / (ell - kp),
                    "within_north_star_bound": bool(ce <= tail / fsq / (ell - kp)),
                    "seconds": round(time.time() - t0, 3)}

    value = world * nnz * a.steps / t_dev
    ms_step = 1e3 * t_dev / a.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "rows_per_sec": world * n * a.steps / t_dev,
            "config": {"workload": f"{a.config}: n={n} d={d} ell={ell} seed={cfg.seed}+rank, nnz={nnz}/rank "
                                   f"(BASELINE.json configs[1]); step = full-stream SfdSketcher + finalize"
                                   + (" + log2 merge tree" if world > 1 else ""),
                       "l2_flush": "256 MB write between timed steps", "parallelism": f"shards x{world}",
                       "flushes_per_step": stats["flushes"], "attempts_per_step": stats["attempts"]},
            "gpu_launches": int(launches), "clocks": clk}
    if t_e2e is not None:
        line["e2e"] = {"value": world * nnz * a.steps / t_e2e, "unit": UNIT,
                       "h2d_bytes_per_step": int(nnz * 12 + (n + stats["flushes"]) * 4),
                       "d2h_bytes_per_step": int(ell * d * 8)}
    line.update(roofline_from_profile(prof, pstats, n, d, ell, nnz))
    rl2 = line.get("roofline", {}).get("l2_gather")
    if rl2 and "spmm" in prof and prof["spmm"][1]:
        # Whole-step bound: the SpMM launches of one step move this many bytes L2 -> SM (one
        # ell-wide FP64 panel row per nonzero), so at the measured gather peak the step cannot
        # take less than floor_ms even with every other kernel hidden under them.
        nsp = prof["spmm"][1]
        gb = nsp * rl2["bytes_per_launch"] / 1e9
        bw = rl2.get("sustained_peak", rl2["peak"])
        floor_ms = 1e3 * gb / bw
        line["step_floor"] = {"bound": "l2_gather", "what": "SpMM gather bytes of one step at the sustained "
                              "L2 gather bandwidth", "spmm_launches": nsp, "gbytes": round(gb, 2),
                              "floor_ms": round(floor_ms, 2), "frac": round(floor_ms / ms_step, 4),
                              "serial_launch_ms": round(nsp * rl2["bytes_per_launch"] / (rl2["peak"] * 1e9) * 1e3, 2),
                              "note": "serial_launch_ms = the same launches back to back at the probe's "
                                      "same-size launch time; the lanes overlap launches, the ramp is the cost"}
    if accuracy is not None:
        line["accuracy"] = accuracy
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            t, nz, rows = reference_sample(a.config, 1, d)
            line["cpu_baseline"] = {"value": nz / t, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"first flush of {a.config} ({rows} rows, {nz} nnz) through the "
                                              f"unmodified reference (oracle/_ref), 1 thread: {t:.1f} s"}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def roofline_from_profile(prof: dict, st: dict, n: int, d: int, ell: int, nnz_stream: int) -> dict:
    """Roofline of the dominant kernel class from the profiled step (SURVEY sec 8(d) formulas)."""
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    fp64 = 36.9  # TFLOP/s, DMMA/DFMA measured on this pool: profiles/r01_fp64_peak.txt
    flushes = max(1, st["flushes"])
    m = d  # every flush of c2 has m = d rows (row trigger)
    nnz_f = nnz_stream / flushes
    kern = {}
    total_ms = sum(v[0] for k, v in prof.items() if k != "rng_gen")
    for k, (ms, cnt) in prof.items():
        kern[k] = {"ms": round(ms, 4), "launches": cnt, "share": round(ms / total_ms, 4) if total_ms else None}
    out = {"kernels": kern}
    # SpMM: bytes = 12 nnz_f + 8 (m+1) + 8 ell d + 8 ell m per launch
    if "spmm" in prof and prof["spmm"][1]:
        ms, cnt = prof["spmm"]
        byts = 12 * nnz_f + 8 * (m + 1) + 8 * ell * d + 8 * ell * m
        gbs = byts / (ms / cnt * 1e-3) / 1e9
        kern["spmm"].update({"alg_bytes_per_launch": byts, "achieved_gbs": round(gbs, 1),
                             "frac_of_measured_hbm": round(gbs / hbm, 4)})
    if "gram" in prof and prof["gram"][1]:
        ms, cnt = prof["gram"]
        att = max(1, st["attempts"])
        n_orth = prof.get("chol", (0, 0))[1]  # one pass-1 factorisation per CholeskyQR2
        # per CholeskyQR2: 2 Grams of m x ell; per attempt: W^T W (d x ell); per flush: [B;B'] (d x 2ell)
        flops = n_orth * 2 * (2 * m * ell * ell) + att * 2 * d * ell * ell + flushes * 2 * d * (2 * ell) ** 2
        tf = flops / (ms * 1e-3) / 1e12
        kern["gram"].update({"alg_flops_total": flops, "achieved_tflops": round(tf, 3),
                             "frac_of_fp64_peak": round(tf / fp64, 4)})
    # The metric names the SpMM's HBM roofline, so the roofline object is the SpMM (K3),
    # the path's memory-bound kernel; the largest time share is reported beside it.
    dom = max((k for k in prof if k != "rng_gen"), key=lambda k: prof[k][0]) if prof else None
    ks = kern.get("spmm", {})
    traffic = None
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = ncu.get("spmm_rows_kernel", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    out["roofline"] = {"bound": "hbm", "kernel": "spmm (CSR/CSC gather, ell-wide panels)",
                       "achieved": ks.get("achieved_gbs"), "peak": hbm, "unit": "GB/s",
                       "frac": ks.get("frac_of_measured_hbm"), "traffic": traffic,
                       "frac_of_nominal_8tbs": round(ks["achieved_gbs"] / 8000.0, 4) if ks.get("achieved_gbs") else None,
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)",
                       "alg_bytes_per_launch": ks.get("alg_bytes_per_launch"),
                       "note": "c2 panels (8 MB) are L2-resident: achieved uses SURVEY 8(d) algorithmic bytes; "
                               "traffic = ncu dram bytes per launch (profiles/)"}
    # The c2 panels are L2-resident, so the bound that actually applies is the L2 -> SM gather
    # bandwidth: measured by tools/probe_l2 (the same access pattern without arithmetic).
    l2 = None
    try:
        for line in open(os.path.join(ROOT, "profiles", "r01_l2_gather_peak.txt")):
            if line.startswith("l2_gather_gbs"):
                l2 = float(line.split()[1])
    except Exception:
        pass
    # Sustained rate of the same pattern in long launches (16x the gathers): a c2-sized launch
    # spends ~6.7 us of its ~10.6 us in launch ramp and tail (profiles/r01c_l2_gather_sustained.txt).
    l2s = None
    try:
        for line in open(os.path.join(ROOT, "profiles", "r01c_l2_gather_sustained.txt")):
            if line.startswith("l2_gather_sustained_gbs"):
                l2s = float(line.split()[1])
    except Exception:
        pass
    if l2 and "spmm" in prof and prof["spmm"][1]:
        ms, cnt = prof["spmm"]
        gath = 8 * ell * nnz_f + 12 * nnz_f  # one ell-wide panel row per nonzero + the CSR entry
        gbs = gath / (ms / cnt * 1e-3) / 1e9
        out["roofline"]["l2_gather"] = {"achieved": round(gbs, 1), "peak": l2, "unit": "GB/s",
                                        "frac": round(gbs / l2, 4), "bytes_per_launch": gath,
                                        "peak_source": "profiles/r01_l2_gather_peak.txt (tools/probe_l2: the same "
                                                       "gathers in one launch of the same size)"}
        if l2s:
            out["roofline"]["l2_gather"].update({"sustained_peak": l2s, "frac_of_sustained": round(gbs / l2s, 4),
                                                 "sustained_source": "profiles/r01c_l2_gather_sustained.txt"})
    out["dominant_kernel"] = {"class": dom, "share_of_step": kern[dom]["share"] if dom else None}
    return out


if __name__ == "__main__":
    sys.exit(main())
