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
