#!/usr/bin/env python
"""fuzz_diverge.py -- replay one fuzz case row by row through the device sketcher and the oracle
and report the first flush whose attempt / verifier counters differ, with that flush buffer's
singular values (test infrastructure: uses oracle/)."""
import sys, json, numpy as np
ROOT = __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + '/tools')
import paper_1602_00412_b200 as P
from oracle.oracle import Oracle, PowerConfig as OPower
import fuzz_parity as F
c = {"d": 9, "ell": 9, "n": 1637, "kind": "lognormal", "cols": "uniform", "structure": "none", "zmax": 5, "seed": 1444001220, "delta": 0.01, "q_override": 8}
rp, cs, vs = F.make_stream(c)
O = Oracle()
os_ = O.sketcher(9, 9, seed=c["seed"], delta=0.01, power=OPower(q_override=8))
g = P.SfdSketcher(P.SketchConfig(ell=9, d=9, seed=c["seed"], delta=0.01, power=P.PowerConfig(q_override=8)))
n = len(rp) - 1
for r in range(n):
    a, b = rp[r], rp[r + 1]
    before = os_.buffer_dense()
    os_.append(cs[a:b].astype(np.uint32), vs[a:b])
    g.append_csr(np.array([0, b - a], dtype=np.int64), cs[a:b].astype(np.uint32), vs[a:b])
    so, sg = os_.stats(), g.stats()
    if (so["attempts"], so["verifier_i"]) != (sg["attempts"], sg["verifier_i"]):
        buf = np.vstack([before, np.zeros((1, 9))]) if before is not None else None
        row = np.zeros(9); row[cs[a:b]] = vs[a:b]
        A = np.vstack([before, row]) if before is not None and len(before) else row[None, :]
        sv = np.linalg.svd(A, compute_uv=False)
        print("diverged at row", r, "oracle", so, "gpu", sg)
        print("flush buffer rows", A.shape[0], "singular values", sv, "sigma_min/sigma_max", sv[-1] / sv[0])
        print("tail energy fractions", np.cumsum(sv[::-1] ** 2)[:4] / (sv ** 2).sum())
        break
else:
    print("no divergence", os_.stats(), g.stats())
