"""Numerical errors surface at the append that triggered the failing flush, with the
reference's post-exception state (core/src/sketch.cpp:20-32: append -> flush throws out of
boosted_sparse_shrink, so B, flush_count / attempt_total and the buffer stay as they were),
checked against the live reference sketcher (oracle/_ref, ref_sketcher_*)."""
import numpy as np
import pytest

import paper_1602_00412_b200 as P

pytestmark = pytest.mark.gpu


def _stream(d=40, flushes=3, big=1e308, bad_flush=1, seed=3):
    """d-row flushes of 6 random entries per row; every 7th row of `bad_flush` is scaled by
    `big`, so A'G overflows, the reference's orthonormalize produces NaN and
    simultaneous_iteration throws (randsvd.cpp:46-47) at that flush's trigger row."""
    g = np.random.default_rng(seed)
    rp, cs, vs = [0], [], []
    for i in range(flushes * d):
        cols = np.sort(g.choice(d, 6, replace=False))
        vals = g.standard_normal(6)
        if bad_flush * d <= i < (bad_flush + 1) * d and i % 7 == 0:
            vals = np.clip(vals, -1.5, 1.5) * big  # finite (|v| < DBL_MAX): the row is valid
        cs.append(cols)
        vs.append(vals)
        rp.append(rp[-1] + 6)
    return np.array(rp, np.int64), np.concatenate(cs).astype(np.uint32), np.concatenate(vs)


def _reference_run(reference, rp, cs, vs, d, ell, seed):
    from oracle.oracle import NumericalError, RefSketcher
    s = RefSketcher(reference, ell, d, seed=seed)
    for i in range(len(rp) - 1):
        try:
            s.append(cs[rp[i]:rp[i + 1]], vs[rp[i]:rp[i + 1]])
        except NumericalError as e:
            return i, str(e), s.sketch(), s.stats()
    raise AssertionError("the reference did not throw on this stream")


def _check_state(sk, ref_b, ref_st):
    st = sk.stats()
    b = sk.sketch()
    for key in ("flushes", "attempts", "verifier_i", "delta_spent"):
        assert st[key] == ref_st[key], key
    for key in ("buf_rows", "buf_nnz", "buf_frob_sq"):
        assert st[key] == ref_st[key], key
    g, gr = b.T @ b, ref_b.T @ ref_b
    assert np.linalg.norm(g - gr) <= 1e-8 * np.linalg.norm(gr)


@pytest.mark.parametrize("lanes", ["1", "4"])
def test_batch_append_raises_at_trigger_row(reference, monkeypatch, lanes):
    monkeypatch.setenv("SFDG_LANES", lanes)
    d, ell, seed = 40, 6, 5
    rp, cs, vs = _stream(d=d, flushes=4)
    row, msg, ref_b, ref_st = _reference_run(reference, rp, cs, vs, d, ell, seed)
    assert row == 2 * d - 1  # the trigger row of the bad flush
    sk = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=seed))
    h = P.lib()
    import ctypes as C
    rpa, csa, vsa = P._csr(rp, cs, vs)
    done = C.c_size_t()
    code = h.sfdg_sketcher_append_csr(sk._h, P._p(rpa, P._i64p), P._p(csa, P._u32p), P._p(vsa, P._dp),
                                      len(rpa) - 1, C.byref(done))
    assert code == 2, h.sfdg_last_error().decode()
    assert done.value == row + 1  # rows after the trigger row were never appended
    assert "non-finite" in h.sfdg_last_error().decode()
    _check_state(sk, ref_b, ref_st)
    brp, bcs, bvs = sk.buffer()  # the failing flush's rows, still buffered
    lo, hi = rp[d], rp[2 * d]
    assert np.array_equal(brp, rp[d:2 * d + 1] - lo)
    assert np.array_equal(bcs, cs[lo:hi]) and np.array_equal(bvs, vs[lo:hi])
    sk.close()


def test_row_by_row_append_raises_at_trigger_row(reference):
    d, ell, seed = 40, 6, 9
    rp, cs, vs = _stream(d=d, flushes=3, seed=4)
    row, _, ref_b, ref_st = _reference_run(reference, rp, cs, vs, d, ell, seed)
    sk = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=seed))
    raised = None
    for i in range(len(rp) - 1):
        try:
            sk.append(cs[rp[i]:rp[i + 1]], vs[rp[i]:rp[i + 1]])
        except P.NumericalError:
            raised = i
            break
    assert raised == row
    _check_state(sk, ref_b, ref_st)
    sk.close()


def test_device_append_raises_at_trigger_row(reference):
    import torch
    d, ell, seed = 40, 6, 5
    rp, cs, vs = _stream(d=d, flushes=4)
    row, _, ref_b, ref_st = _reference_run(reference, rp, cs, vs, d, ell, seed)
    dc = torch.from_numpy(cs.view(np.int32)).cuda()
    dv = torch.from_numpy(vs).cuda()
    sk = P.SfdSketcher(P.SketchConfig(ell=ell, d=d, seed=seed))
    with pytest.raises(P.NumericalError):
        sk.append_csr_device(rp, dc.data_ptr(), dv.data_ptr())
    _check_state(sk, ref_b, ref_st)
    sk.close()
