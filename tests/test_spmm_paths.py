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
