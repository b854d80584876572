"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libsfdref.so).

Run in the build container (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/sfd_oracle.c) on machines without the
reference sources (tests/test_oracle_pin.py) and give the GPU parity tests fixed
expected outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference, VerifierState  # noqa: E402
from paper_1602_00412_b200 import synthetic as S  # noqa: E402


def main():
    R = Reference()
    out = {}
    # mt19937_64 + Rng draws (rng.hpp:12-31)
    r = R.rng(0)
    out["u64_seed0"] = np.array([r.next_u64() for _ in range(64)], dtype=np.uint64)
    r = R.rng(7)
    out["normals_seed7"] = np.array([r.normal() for _ in range(257)])
    r = R.rng(11)
    out["uniform_seed11"] = np.array([r.uniform() for _ in range(64)])
    # dense_shrink KAT (tests/test_shrink.cpp:24-32)
    a = np.zeros((3, 4))
    a[0, 0], a[1, 1], a[2, 2] = 3.0, 2.0, 1.0
    out["kat_dense_a"] = a
    out["kat_dense_b"] = R.dense_shrink(a, 2)
    # tall dense_shrink (tests/test_shrink.cpp:44-52 shape)
    g = R.rng(8)
    t = np.array([[g.normal() for _ in range(5)] for _ in range(8)])
    out["tall_a"] = t
    out["tall_b"] = R.dense_shrink(t, 4)
    # boosted_sparse_shrink on random_sparse(60, 30, 0.2) (tests/test_shrink.cpp:183-203)
    g = R.rng(1300)
    rp, cs, vs = S.random_sparse(g, 60, 30, 0.2)
    st = VerifierState()
    b, dh, att = R.boosted_sparse_shrink((rp, cs, vs), 30, 6, st, R.rng(99))
    out.update(boost_rp=rp, boost_cs=cs, boost_vs=vs, boost_b=b,
               boost_meta=np.array([dh, att, st.i, st.delta_spent]))
    # a small stream (tests/test_sketch.cpp:300-325 shape)
    g = R.rng(9000)
    rp, cs, vs = S.random_sparse(g, 300, 40, 0.2)
    b, stats = R.sketch(rp, cs, vs, 40, 12, seed=9000)
    out.update(small_rp=rp, small_cs=cs, small_vs=vs, small_b=b,
               small_stats=np.array([stats["flushes"], stats["attempts"], stats["verifier_i"],
                                     stats["delta_spent"]]))
    # first 3 flushes of BASELINE config c1 (n=3000 of 10000 rows, d=1000, ell=50, seed 0)
    rp, cs, vs = S.generate("c1", (0, 3000))
    b, stats = R.sketch(rp, cs, vs, 1000, 50, seed=0)
    out.update(c1p_b=b, c1p_stats=np.array([stats["flushes"], stats["attempts"], stats["verifier_i"],
                                            stats["delta_spent"]]))
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"))


if __name__ == "__main__":
    main()
