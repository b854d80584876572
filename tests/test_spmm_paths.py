"""The SpMM's alternative data paths give bit-identical sketches: staging the hot columns'
panel rows in shared memory (HotSet, TMA bulk copies) only changes where each row is read
from, and long rows / columns summed from pieces by their last piece keep the piece order."""
import numpy as np
import pytest

import paper_1602_00412_b200 as P
from paper_1602_00412_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _sketch(rp, cs, vs, d, ell, seed):
    s = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=seed))
    s.append_csr(rp, cs, vs)
    b = s.finalize()
    st = s.stats()
    s.close()
    return b, st


@pytest.mark.parametrize("family,d,ell,rows", [("c4", 3000, 64, 6000), ("c3", 2500, 96, 5000), ("c5", 4000, 128, 8000)])
def test_hot_column_staging_is_bit_identical(monkeypatch, family, d, ell, rows):
    rp, cs, vs = S.generate(S.StreamConfig(family, rows, d, ell, 5), (0, rows))
    monkeypatch.setenv("SFDG_HOT", "1")
    b_hot, st_hot = _sketch(rp, cs, vs, d, ell, 3)
    monkeypatch.setenv("SFDG_HOT", "0")
    b_plain, st_plain = _sketch(rp, cs, vs, d, ell, 3)
    assert np.array_equal(b_hot, b_plain) and st_hot == st_plain


def test_graphs_on_and_off_are_bit_identical(monkeypatch):
    rp, cs, vs = S.generate(S.StreamConfig("c4", 9000, 3000, 64, 6), (0, 9000))
    b_g, st_g = _sketch(rp, cs, vs, 3000, 64, 1)
    monkeypatch.setenv("SFDG_GRAPHS", "0")
    b_n, st_n = _sketch(rp, cs, vs, 3000, 64, 1)
    assert np.array_equal(b_g, b_n) and st_g == st_n


@pytest.mark.parametrize("family,d,ell,rows", [("c4", 3000, 64, 6000), ("c2", 4000, 100, 12000), ("c5", 2000, 200, 4000)])
def test_gram_tma_and_cp_async_are_bit_identical(monkeypatch, family, d, ell, rows):
    """The Gram's stages arrive by per-thread cp.async (default) or TMA bulk copies
    (SFDG_GRAM=tma): the same tiles, chunks and DMMA order, so the same bits -- including edge
    tiles (lp = 104 / 200: a 40- / 8-column last tile) and chunk tails."""
    rp, cs, vs = S.generate(S.StreamConfig(family, rows, d, ell, 7), (0, rows))
    b_c, st_c = _sketch(rp, cs, vs, d, ell, 2)
    monkeypatch.setenv("SFDG_GRAM", "tma")
    b_t, st_t = _sketch(rp, cs, vs, d, ell, 2)
    assert np.array_equal(b_t, b_c) and st_t == st_c


def test_gram_tma_dense_shrink_and_orthonormalize(monkeypatch):
    g = np.random.default_rng(11)
    a = g.standard_normal((333, 1001))  # 2 lp-wide Grams with odd row counts
    y = g.standard_normal((20011, 136))
    d_c, q_c = P.dense_shrink(a, 150), P.orthonormalize(y)
    monkeypatch.setenv("SFDG_GRAM", "tma")
    d_t, q_t = P.dense_shrink(a, 150), P.orthonormalize(y)
    assert np.array_equal(d_t, d_c) and np.array_equal(q_t, q_c)


@pytest.mark.parametrize("family,d,ell,rows", [("c4", 3000, 64, 6000), ("c3", 2500, 96, 5000), ("c5", 4000, 128, 8000)])
def test_piece_order_is_bit_identical(monkeypatch, family, d, ell, rows):
    """Pieces of long rows / columns run in the order of the first input index they gather
    (default for panels larger than L2; forced on here) or in piece order (SFDG_PIECE_ORDER=0):
    which warp runs a piece, and when, changes; the partials are summed in piece order either
    way, so the sketches are the same bits."""
    rp, cs, vs = S.generate(S.StreamConfig(family, rows, d, ell, 8), (0, rows))
    monkeypatch.setenv("SFDG_PIECE_ORDER", "1")
    b_o, st_o = _sketch(rp, cs, vs, d, ell, 4)
    monkeypatch.setenv("SFDG_PIECE_ORDER", "0")
    b_n, st_n = _sketch(rp, cs, vs, d, ell, 4)
    assert np.array_equal(b_o, b_n) and st_o == st_n


@pytest.mark.parametrize("family,d,ell,rows", [("c4", 3000, 64, 6000), ("c5", 4000, 128, 8000)])
def test_pieces_by_ticket_are_bit_identical(monkeypatch, family, d, ell, rows):
    """Pieces taken by ticket as warps become free (default for panels larger than L2; forced on
    here, with the first-index order) or statically strided: only which warp runs a piece, and
    when, changes -- the two-level sums keep the piece order -- so the sketches are the same bits,
    launch after launch (the ticket and arrival counters reset themselves)."""
    rp, cs, vs = S.generate(S.StreamConfig(family, rows, d, ell, 9), (0, rows))
    monkeypatch.setenv("SFDG_PIECE_ORDER", "1")
    monkeypatch.setenv("SFDG_SPMM_DYN", "1")
    b_t, st_t = _sketch(rp, cs, vs, d, ell, 5)
    monkeypatch.setenv("SFDG_SPMM_DYN", "0")
    b_s, st_s = _sketch(rp, cs, vs, d, ell, 5)
    assert np.array_equal(b_t, b_s) and st_t == st_s


def test_products_with_a_panel_larger_than_l2():
    """A'^T Z with a Z panel larger than the L2 (300k rows x 64 columns = 154 MB): the CSC plan
    shortens its pieces so the pieces in flight cover an L2-sized window, takes them by ticket in
    first-row order and sums columns of more than 64 pieces in two levels. Against scipy, and the
    same bits on a second run."""
    import scipy.sparse as sp

    rng = np.random.default_rng(23)
    m, d, k = 300_000, 5000, 64
    per = 5
    cols = rng.integers(20, d, size=(m, per))
    hot = rng.random((m, 3)) < np.array([0.9, 0.2, 0.02])  # columns 0, 1, 2: 270k / 60k / 6k entries
    rows = []
    for i in range(m):
        r = np.unique(cols[i])
        rows.append(np.concatenate([np.nonzero(hot[i])[0], r]))
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    cs = np.concatenate(rows).astype(np.uint32)
    vs = rng.standard_normal(cs.size)
    z = rng.standard_normal((m, k))
    a = sp.csr_matrix((vs, cs.astype(np.int64), rp), shape=(m, d))
    wa = a.T @ z
    _, w = P.csr_products((rp, cs, vs), d, z=z)
    assert np.max(np.abs(w - wa)) <= 1e-11 * np.abs(wa).max()
    _, w2 = P.csr_products((rp, cs, vs), d, z=z)
    assert np.array_equal(w, w2)
