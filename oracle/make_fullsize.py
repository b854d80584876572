"""Full-size parity fixtures from the UNMODIFIED reference (oracle/_ref/libsfdref.so).

TEST INFRASTRUCTURE ONLY. Runs the reference's own SfdSketcher (sketch.cpp:14-45, through
oracle/ref_shim.cpp `ref_sketch`: append every row, finalize) on prefixes of the BASELINE
streams at their FULL d and ell, and stores the sketch and the counters:

  c2_5f   c2 rows [0, 50_000)    d=1e4  ell=100  5 flushes      (~2.5 min on one core)
  c2_full c2 rows [0, 1_000_000) d=1e4  ell=100  100 flushes    (~50 min: the benched stream)
  c4_2f   c4 rows [0, 100_000)   d=5e4  ell=128  2 flushes      (~50 min)
  c3_1f   c3 rows [0, 100_000)   d=1e5  ell=200  1 flush        (~85 min)

Output: oracle/_ref/fullsize/<job>.npz (git-ignored like the rest of oracle/_ref; it travels
to the GPU box with the snapshot). tests/test_fullsize_parity.py (-m gpu) compares the
device sketcher against these: B^T B within 1e-8 relative Frobenius and the counters exactly.
Each file records a digest of the input CSR so a generator change is caught, not compared.

  python oracle/make_fullsize.py <job> [<job> ...]
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

JOBS = {
    "c2_5f": ("c2", 50_000),
    "c2_full": ("c2", 1_000_000),
    "c4_2f": ("c4", 100_000),
    "c3_1f": ("c3", 100_000),
}
OUT = os.path.join(ROOT, "oracle", "_ref", "fullsize")


def csr_digest(rp, cs, vs) -> str:
    h = hashlib.sha256()
    for a in (rp, cs, vs):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def run(job: str) -> None:
    from oracle.oracle import Reference
    from paper_1602_00412_b200 import synthetic as S

    name, rows = JOBS[job]
    cfg = S.CONFIGS[name]
    rp, cs, vs = S.generate(name, (0, rows))
    t = time.time()
    b, st = Reference().sketch(rp, cs, vs, cfg.d, cfg.ell, seed=cfg.seed)
    secs = time.time() - t
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, job + ".npz")
    np.savez(path + ".tmp.npz", b=b, flushes=st["flushes"], attempts=st["attempts"],
             verifier_i=st["verifier_i"], delta_spent=st["delta_spent"], rows=rows, d=cfg.d, ell=cfg.ell,
             seed=cfg.seed, nnz=int(rp[-1]), digest=csr_digest(rp, cs, vs), seconds=secs)
    os.replace(path + ".tmp.npz", path)
    print(f"{job}: {rows} rows, nnz {int(rp[-1])}, {st}, {secs:.1f} s -> {path}", flush=True)


if __name__ == "__main__":
    sys.path[0:1] = [ROOT]  # not oracle/ itself: `oracle` must resolve to the package dir
    for j in sys.argv[1:] or ["c2_5f"]:
        run(j)
