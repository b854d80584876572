"""Pin the CPU oracle (oracle/sfd_oracle.c) before trusting it as the parity checker.

* against the reference's own known-answer tests (tests/test_shrink.cpp, test_randsvd.cpp,
  test_sketch.cpp) restated here;
* against golden vectors produced by the UNMODIFIED reference (tests/golden/make_golden.py,
  oracle/_ref) -- bit-exact;
* live against oracle/_ref when it is available (build container, or its prebuilt .so).
All CPU-only (no GPU needed).
"""
import math
import os

import numpy as np
import pytest

from oracle.oracle import InvalidArgument, KALPHA, NumericalError, PowerConfig, VerifierState
from paper_1602_00412_b200 import synthetic as S

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def test_mt19937_64_standard_kat(oracle):
    # [rand.predef]: the 10000th output of a default-constructed mt19937_64 is 9981545732273789042
    r = oracle.rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


def test_rng_streams_match_reference_golden(oracle):
    r = oracle.rng(0)
    assert np.array_equal(np.array([r.next_u64() for _ in range(64)], dtype=np.uint64), GOLD["u64_seed0"])
    r = oracle.rng(7)
    assert np.array_equal(np.array([r.normal() for _ in range(257)]), GOLD["normals_seed7"])
    r = oracle.rng(11)
    assert np.array_equal(np.array([r.uniform() for _ in range(64)]), GOLD["uniform_seed11"])


def test_rng_state_tracks_spare(oracle):
    r = oracle.rng(3)
    r.normal()
    w, hs, sp = r.state()
    assert (w, hs) == (2, True)
    assert sp == r.normal()
    assert r.state()[:2] == (2, False)


def test_dense_shrink_kat(oracle):
    # tests/test_shrink.cpp:24-32: rows 3e1, 2e2, 1e3, ell=2 -> sqrt(5) e1, row ell zero
    b = oracle.dense_shrink(GOLD["kat_dense_a"], 2)
    assert abs(abs(b[0, 0]) - math.sqrt(5.0)) < 1e-10
    assert np.all(np.abs(b[0, 1:]) < 1e-10)
    assert np.all(b[1] == 0.0)
    assert np.array_equal(b, GOLD["kat_dense_b"])


def test_dense_shrink_tall_bookkeeping(oracle):
    # tests/test_shrink.cpp:44-52: |A|^2 - |B|^2 = 4 s4^2 + s5^2
    a = GOLD["tall_a"]
    b = oracle.dense_shrink(a, 4)
    sv = np.linalg.svd(a, compute_uv=False) ** 2
    assert abs((a ** 2).sum() - (b ** 2).sum() - (4 * sv[3] + sv[4])) <= 1e-8 * (4 * sv[3] + sv[4])
    assert np.array_equal(b, GOLD["tall_b"])


def test_dense_shrink_validation(oracle):
    with pytest.raises(InvalidArgument):
        oracle.dense_shrink(np.zeros((3, 4)), 0)
    with pytest.raises(InvalidArgument):
        oracle.dense_shrink(np.zeros((3, 4)), 4)


def test_power_iteration_count(oracle):
    # tests/test_randsvd.cpp:40-47
    assert oracle.power_iteration_count(3000) == 38
    assert oracle.power_iteration_count(3000, PowerConfig(q_override=5)) == 5
    assert oracle.power_iteration_count(3000, PowerConfig(q_override=0)) == 0


def test_boosted_matches_reference_golden(oracle):
    csr = (GOLD["boost_rp"], GOLD["boost_cs"], GOLD["boost_vs"])
    st = VerifierState()
    b, dh, att = oracle.boosted_sparse_shrink(csr, 30, 6, st, oracle.rng(99))
    assert np.array_equal(b, GOLD["boost_b"])
    assert [dh, att, st.i, st.delta_spent] == list(GOLD["boost_meta"])
    drop = (GOLD["boost_vs"] ** 2).sum() - (b ** 2).sum()
    assert abs(dh - drop / (KALPHA * 6)) <= 1e-12 * dh


def test_small_stream_matches_reference_golden(oracle):
    b, st = oracle.sketch(GOLD["small_rp"], GOLD["small_cs"], GOLD["small_vs"], 40, 12, seed=9000)
    assert np.array_equal(b, GOLD["small_b"])
    assert [st["flushes"], st["attempts"], st["verifier_i"], st["delta_spent"]] == list(GOLD["small_stats"])


def test_c1_prefix_matches_reference_golden(oracle):
    rp, cs, vs = S.generate("c1", (0, 3000))
    b, st = oracle.sketch(rp, cs, vs, 1000, 50, seed=0)
    assert np.array_equal(b, GOLD["c1p_b"])
    assert [st["flushes"], st["attempts"], st["verifier_i"], st["delta_spent"]] == list(GOLD["c1p_stats"])


def test_verify_trivial_operators(oracle):
    # tests/test_shrink.cpp:117-144
    rng = oracle.rng(5)
    st = VerifierState(0.1)
    assert oracle.verify_spectral(lambda x: np.zeros_like(x), 20, st, rng)
    assert st.i == 1
    assert oracle.verify_spectral(lambda x: x, 20, st, rng)
    assert st.i == 2
    assert not oracle.verify_spectral(lambda x: 3.0 * x, 20, st, rng)
    assert st.i == 3
    assert abs(st.delta_spent - (0.1 / 2 + 0.1 / 8 + 0.1 / 18)) <= 1e-12


def test_sketcher_triggers(oracle):
    # tests/test_sketch.cpp:35-66
    s = oracle.sketcher(4, 16, 0)
    s.append([0], [1.0])
    assert s.stats()["flushes"] == 0 and s.stats()["buf_rows"] == 1
    s = oracle.sketcher(3, 6, 0)
    g = oracle.rng(1)
    for i in range(3):
        s.append(list(range(6)), [g.normal() for _ in range(6)])
        assert s.stats()["flushes"] == (1 if i == 2 else 0)
    s = oracle.sketcher(4, 8, 0)
    for i in range(8):
        s.append([i], [1.0])
        assert s.stats()["flushes"] == (1 if i == 7 else 0)


def test_sketcher_row_validation(oracle):
    s = oracle.sketcher(2, 5, 0)
    with pytest.raises(InvalidArgument):
        s.append([5], [1.0])
    with pytest.raises(InvalidArgument):
        s.append([2, 2], [1.0, 1.0])
    with pytest.raises(InvalidArgument):
        s.append([1], [float("nan")])
    assert s.stats()["buf_rows"] == 0


def test_oracle_matches_live_reference(oracle, reference):
    rp, cs, vs = S.generate("c1", (0, 1000))
    b1, s1 = oracle.sketch(rp, cs, vs, 1000, 50, seed=0)
    b2, s2 = reference.sketch(rp, cs, vs, 1000, 50, seed=0)
    assert np.array_equal(b1, b2)
    for k in ("flushes", "attempts", "verifier_i", "delta_spent"):
        assert s1[k] == s2[k]
    g1, g2 = oracle.rng(77), reference.rng(77)
    z1 = oracle.simultaneous_iteration((rp, cs, vs), 1000, 20, g1)
    z2 = reference.simultaneous_iteration((rp, cs, vs), 1000, 20, g2)
    assert np.array_equal(z1, z2)
    a = np.random.default_rng(3).standard_normal((30, 12))
    assert np.array_equal(oracle.orthonormalize(a), reference.orthonormalize(a))
    k = a.T @ a
    v1, e1 = oracle.jacobi_eigh(k, 1e-12)
    v2, e2 = reference.jacobi_eigh(k, 1e-12)
    assert np.array_equal(v1, v2) and np.array_equal(e1, e2)


def test_retry_cap_is_a_numerical_error(oracle):
    # a verifier that always rejects: scale with a huge operator via a degenerate delta
    csr = (GOLD["boost_rp"], GOLD["boost_cs"], GOLD["boost_vs"])
    st = VerifierState(delta=0.1)
    st.c_verify = 200.0  # many steps: still accepts when the bound holds; just exercise the path
    b, dh, att = oracle.boosted_sparse_shrink(csr, 30, 6, st, oracle.rng(1))
    assert att >= 1
    with pytest.raises((NumericalError, InvalidArgument)):
        oracle.boosted_sparse_shrink(csr, 30, 0, VerifierState(), oracle.rng(1))


def test_fd_sketcher_oracle_matches_reference(oracle, reference):
    """FdSketcher restatement (sketch.cpp:47-78) against the compiled reference: buffer
    fills, the finalize partial shrink, the tall (2 ell > d) stack and < ell rows."""
    g = np.random.default_rng(3)
    for n, d, ell in [(7, 5, 2), (40, 12, 4), (3, 6, 3), (25, 30, 5), (61, 9, 6), (1, 4, 4)]:
        a = g.standard_normal((n, d))
        bo, co = oracle.fd_sketch(a, ell)
        br, cr = reference.fd_sketch(a, ell)
        assert co == cr
        assert np.array_equal(bo, br)


def test_cov_err_oracle_matches_reference(oracle, reference):
    """cov_err restatement (bench.cpp:171-183 over la_core.cpp:191-211) bit-exact against
    the compiled reference, same draws (rng advanced identically)."""
    from paper_1602_00412_b200 import synthetic as S
    rp, cs, vs = S.generate("c1", (0, 1200))
    b, _ = oracle.sketch(rp, cs, vs, 1000, 50, seed=0)
    g1, g2 = oracle.rng(77), reference.rng(77)
    assert oracle.cov_err(rp, cs, vs, 1000, b, g1, 150) == reference.cov_err(rp, cs, vs, 1000, b, g2, 150)
    # a zero sketch measures |A^T A|_2 / |A|_F^2 (power iteration converged by 400 steps)
    a = np.zeros((len(rp) - 1, 1000))
    for i in range(len(rp) - 1):
        a[i, cs[rp[i]:rp[i + 1]]] = vs[rp[i]:rp[i + 1]]
    top = np.linalg.norm(a, 2) ** 2 / (a ** 2).sum()
    assert abs(oracle.cov_err(rp, cs, vs, 1000, np.zeros((5, 1000)), oracle.rng(1), 400) - top) <= 1e-6 * top


def test_exact_tail_oracle_matches_reference(oracle, reference):
    """exact_tail restatement (bench.cpp:68-137: block k+10, MGS, Jacobi, the two convergence
    tests) bit-exact against the compiled reference for k = 0, 5, 10."""
    from paper_1602_00412_b200 import synthetic as S
    rp, cs, vs = S.generate("c1", (0, 1500))
    for k in (0, 5, 10):
        t1, s1, _ = oracle.exact_tail(rp, cs, vs, 1000, k, oracle.rng(9))
        t2, s2 = reference.exact_tail(rp, cs, vs, 1000, k, reference.rng(9))
        assert t1 == t2 and np.array_equal(s1, s2)


def test_proj_err_oracle_matches_reference(oracle, reference):
    """proj_err restatement (bench.cpp:139-169) bit-exact against the reference, including
    the nullopt case (tail below 1e-12 |A|_F^2)."""
    from paper_1602_00412_b200 import synthetic as S
    rp, cs, vs = S.generate("c1", (0, 1500))
    b, _ = oracle.sketch(rp, cs, vs, 1000, 50, seed=0)
    for k in (1, 7, 10):
        t, _, _ = oracle.exact_tail(rp, cs, vs, 1000, k, oracle.rng(9))
        assert oracle.proj_err(rp, cs, vs, 1000, b, k, t) == reference.proj_err(rp, cs, vs, 1000, b, k, t)
    assert oracle.proj_err(rp, cs, vs, 1000, b, 5, 1e-30) is None


@pytest.mark.parametrize("family,d,ell,rows", [("c3", 500, 24, 400), ("c4", 600, 32, 1500), ("c5", 800, 48, 1600),
                                               ("c3", 260, 200, 540), ("c5", 300, 256, 620)])
def test_oracle_matches_live_reference_families(oracle, reference, family, d, ell, rows):
    """The restatement bit-exact against the compiled reference on the c3 / c4 / c5 stream
    families the GPU parity tests rely on (Zipf columns with lognormal rows, power-law
    ratings mean-centred per row, Poisson rows with a planted signal) and at the wide ell of
    c3 (200) and c5 (256): same B, same counters."""
    seed = S.CONFIGS[family].seed
    rp, cs, vs = S.generate(S.StreamConfig(family, rows, d, ell, seed), (0, rows))
    b1, s1 = oracle.sketch(rp, cs, vs, d, ell, seed=seed)
    b2, s2 = reference.sketch(rp, cs, vs, d, ell, seed=seed)
    assert s1["flushes"] >= 2
    for k in ("flushes", "attempts", "verifier_i", "delta_spent"):
        assert s1[k] == s2[k], k
    assert np.array_equal(b1, b2)
