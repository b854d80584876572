"""ell above 256 (up to this build's 512; the reference accepts any 1 <= ell <= d,
core/src/sketch.cpp:9-12): every kernel on the flush path at lp = 264 .. 512 and the 2 ell
= 528 .. 1024 stacked rows of the dense shrink, against the oracle.

* CholeskyQR2 (chol_factor up to k = 512, the substitution TRSM above 256, exact_orth with its
  partials in dynamic shared memory) -- la_core.cpp:130-165;
* the eigensolver above 512 rows (dense_shrink of [B; B'], shrink.cpp:30-61; ell = 512 on
  d = 600 takes the tall path, whose Gram is d x d);
* the kernel-sequence verifier with 10 .. 16 values of t per lane (shrink.cpp:75-102);
* whole streams: SfdSketcher at ell = 320 and 512 (sketch.cpp:14-45), counters exact.
"""
import numpy as np
import pytest

import paper_1602_00412_b200 as P
from paper_1602_00412_b200 import synthetic as S

pytestmark = pytest.mark.gpu
BTB_TOL = 1e-8


def btb_rel(b, c):
    g, h = b.T @ b, c.T @ c
    return np.linalg.norm(g - h) / np.linalg.norm(h)


@pytest.mark.parametrize("n,k", [(1200, 264), (1500, 384), (1100, 512)])
def test_orthonormalize_wide_vs_oracle(oracle, n, k):
    a = np.random.default_rng(n + k).standard_normal((n, k))
    q = P.orthonormalize(a)
    qo = oracle.orthonormalize(a)
    assert np.max(np.abs(q.T @ q - np.eye(k))) <= 1e-13
    assert np.max(np.abs(q @ q.T - qo @ qo.T)) <= 1e-12


def test_orthonormalize_wide_drops_dependent_columns(oracle):
    """Dependent and zero columns past column 256: CholeskyQR's pivot test with exact_orth
    (k = 300) decides the drops like the reference's MGS."""
    rng = np.random.default_rng(5)
    a = rng.standard_normal((900, 300))
    a[:, 270] = a[:, 3] - 2.0 * a[:, 280]
    a[:, 299] = 0.0
    a[:, 290] = a[:, 10] + a[:, 20] + 1e-9 * rng.standard_normal(900)  # nearly dependent: kept by the reference
    q = P.orthonormalize(a)
    qo = oracle.orthonormalize(a)
    assert np.array_equal(np.abs(q).sum(axis=0) == 0, np.abs(qo).sum(axis=0) == 0)
    keep = np.abs(qo).sum(axis=0) > 0
    assert keep[290] and not keep[299]
    assert np.max(np.abs(q @ q.T - qo @ qo.T)) <= 1e-6


def test_dense_shrink_wide_vs_oracle(oracle):
    """540 stacked rows (the 16-CTA cluster row kernel) against the oracle."""
    a = np.random.default_rng(540).standard_normal((540, 700))
    assert btb_rel(P.dense_shrink(a, 270), oracle.dense_shrink(a, 270)) <= 1e-11


def test_dense_shrink_1024_rows_vs_svd():
    """1024 stacked rows (ell = 512, the global-memory tridiagonalisation): the reference's
    Jacobi takes minutes at this size, so the FD shrink is restated through LAPACK's SVD:
    B^T B = V diag(max(s_i^2 - s_ell^2, 0)) V^T over the top ell (shrink.cpp:30-61)."""
    a = np.random.default_rng(1024).standard_normal((1024, 1100))
    _, s, vt = np.linalg.svd(a, full_matrices=False)
    w = np.sqrt(np.maximum(s[:512] ** 2 - s[511] ** 2, 0.0))
    want = w[:, None] * vt[:512]
    assert btb_rel(P.dense_shrink(a, 512), want) <= 1e-10


@pytest.mark.parametrize("family,d,ell,rows", [("c5", 700, 320, 1400), ("c3", 600, 512, 600)])
def test_wide_ell_stream_vs_oracle(oracle, family, d, ell, rows):
    cfg = S.StreamConfig(family, rows, d, ell, 6)
    rp, cs, vs = S.generate(cfg, (0, rows))
    s = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=31))
    s.append_csr(rp, cs, vs)
    b = s.finalize()
    st = s.stats()
    s.close()
    bo, so = oracle.sketch(rp, cs, vs, d, ell, seed=31)
    assert so["flushes"] >= 1
    assert btb_rel(b, bo) <= BTB_TOL
    for key in ("flushes", "attempts", "verifier_i", "delta_spent"):
        assert st[key] == so[key], key


def test_ell_above_build_limit_rejected():
    with pytest.raises(P.InvalidArgument):
        P.SfdSketcher(P.SketchConfig(ell=513, d=2000, seed=0))


def test_large_d_stream_vs_oracle(oracle):
    """A wide, very sparse stream (d = 2e7 columns, ell = 3): panels of 2e7 x 8 doubles, the
    draw of d x ell = 6e7 normals per attempt, column ids above 2^24 -- the column and panel
    indexing at sizes the BASELINE configs do not reach (c5: d = 1e6)."""
    d, ell, rows = 20_000_000, 3, 40
    g = np.random.default_rng(9)
    rp = [0]
    cs, vs = [], []
    for _ in range(rows):
        c = np.sort(g.choice(d, size=g.integers(1, 6), replace=False))
        cs.append(c)
        vs.append(g.standard_normal(c.size))
        rp.append(rp[-1] + c.size)
    rp, cs, vs = np.array(rp, np.int64), np.concatenate(cs).astype(np.uint32), np.concatenate(vs)
    s = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=5))
    s.append_csr(rp, cs, vs)
    b = s.finalize()
    st = s.stats()
    s.close()
    bo, so = oracle.sketch(rp, cs, vs, d, ell, seed=5)
    for key in ("flushes", "attempts", "verifier_i", "delta_spent"):
        assert st[key] == so[key], key
    # B^T B is d x d here: compare through the 2 ell x 2 ell form of the difference
    r = np.linalg.qr(np.vstack([b, bo]).T, mode="r")
    x = r[:, :ell] @ r[:, :ell].T - r[:, ell:] @ r[:, ell:].T
    assert np.linalg.norm(x) <= BTB_TOL * np.linalg.norm(bo @ bo.T)


def test_cov_err_any_sketch_height_vs_oracle(oracle):
    """cov_err (bench.cpp:171-183) has no limit on the sketch's height: a 700-row B (above this
    build's sketching limit of 512) against the oracle, same draws."""
    rp, cs, vs = S.generate("c1", (0, 1500))
    b = np.random.default_rng(12).standard_normal((700, 1000)) * 0.05
    got, _ = P.cov_err((rp, cs, vs), 1000, b, P.RngState(31), iterations=150)
    want = oracle.cov_err(rp, cs, vs, 1000, b, oracle.rng(31), 150)
    assert abs(got - want) <= 1e-9 * abs(want)
