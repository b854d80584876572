"""Regression test for the one fuzz divergence (profiles/r01_fuzz_parity.txt, seed 41 case 127).

A 9 x 9 lognormal stream (sigma 2, ~1e5 dynamic range) whose flush 93 holds a direction with
1.39e-12 of |A'|_F^2: the SparseShrink drop lands on the reference's Delta = 0 cut
(drop <= 1e-12 |A'|_F^2, core/src/shrink.cpp:112) to within roundoff, so which branch each
implementation takes is decided by the last bits of B'. The oracle replays the reference
bit-exactly (tests/test_oracle_pin.py); the device path may take the other branch there.

Pinned here:
* the oracle side of the tie does not move (CPU): its counters are exactly the reference's;
* on the device the sketch still matches at the north_star gate, and the counters agree or
  differ by exactly the one extra verified-and-rejected attempt the tie explains (one more
  attempt, one more verifier step) -- anything else is a new divergence, not this tie.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

CASE = {"d": 9, "ell": 9, "n": 1637, "kind": "lognormal", "cols": "uniform", "structure": "none", "zmax": 5,
        "seed": 1444001220, "delta": 0.01, "q_override": 8}
ORACLE_COUNTS = (181, 100)  # attempts, verifier i of the reference (profiles/r01_fuzz_parity.txt)


def _stream():
    import fuzz_parity as F
    return F.make_stream(CASE)


def _oracle_run(oracle):
    from oracle.oracle import PowerConfig as OPower
    rp, cs, vs = _stream()
    s = oracle.sketcher(9, 9, seed=CASE["seed"], delta=0.01, power=OPower(q_override=8))
    for r in range(len(rp) - 1):
        a, b = rp[r], rp[r + 1]
        s.append(cs[a:b].astype(np.uint32), vs[a:b])
    return s.finalize(), s.stats()


def test_near_tie_oracle_side(oracle):
    _, st = _oracle_run(oracle)
    assert (st["attempts"], st["verifier_i"]) == ORACLE_COUNTS


def test_near_tie_oracle_matches_reference(oracle, reference):
    from oracle.oracle import PowerConfig as OPower
    rp, cs, vs = _stream()
    b1, s1 = _oracle_run(oracle)
    s = reference.sketcher(9, 9, seed=CASE["seed"], delta=0.01, power=OPower(q_override=8)) \
        if hasattr(reference, "sketcher") else None
    if s is None:
        b2, s2 = reference.sketch(rp, cs, vs, 9, 9, seed=CASE["seed"], delta=0.01, power=OPower(q_override=8))
    else:
        for r in range(len(rp) - 1):
            a, b = rp[r], rp[r + 1]
            s.append(cs[a:b].astype(np.uint32), vs[a:b])
        b2, s2 = s.finalize(), s.stats()
    assert (s1["attempts"], s1["verifier_i"]) == (s2["attempts"], s2["verifier_i"])
    assert np.array_equal(b1, b2)


@pytest.mark.gpu
def test_near_tie_device(oracle):
    import paper_1602_00412_b200 as P
    rp, cs, vs = _stream()
    bo, so = _oracle_run(oracle)
    g = P.SfdSketcher(P.SketchConfig(ell=9, d=9, seed=CASE["seed"], delta=0.01, power=P.PowerConfig(q_override=8)))
    g.append_csr(rp, cs.astype(np.uint32), vs)
    b = g.finalize()
    sg = g.stats()
    go, gg = bo.T @ bo, b.T @ b
    assert np.linalg.norm(gg - go) / np.linalg.norm(go) <= 1e-8
    assert sg["flushes"] == so["flushes"]
    da, dv = sg["attempts"] - so["attempts"], sg["verifier_i"] - so["verifier_i"]
    assert (da, dv) in {(0, 0), (1, 1)}, (sg, so)
