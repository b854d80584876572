"""verify_spectral over caller operators (shrink.hpp:35, shrink.cpp:75-102) through
sfdg_verify_spectral: the reference's own unit cases (tests/test_shrink.cpp:117-165) restated,
agreement with the oracle's verifier (sfd_oracle.c, pinned to the reference) on random PSD
operators, and the device-pointer operator mode."""
import numpy as np
import pytest

import paper_1602_00412_b200 as P
from oracle.oracle import VerifierState as OVer

pytestmark = pytest.mark.gpu


def test_trivial_operators_and_budget():
    # tests/test_shrink.cpp:117-144
    rng = P.RngState(5)
    st = P.VerifierState(delta=0.1)
    ok, rng = P.verify_spectral(lambda x: np.zeros_like(x), 20, st, rng)
    assert ok and st.i == 1
    ok, rng = P.verify_spectral(lambda x: x, 20, st, rng)
    assert ok and st.i == 2
    ok, rng = P.verify_spectral(lambda x: 3.0 * x, 20, st, rng)
    assert not ok and st.i == 3
    assert st.delta_spent == pytest.approx(0.1 / 2 + 0.1 / 8 + 0.1 / 18, rel=1e-12)
    assert st.delta_spent < st.delta


def test_planted_spike_is_rejected():
    # tests/test_shrink.cpp:146-165: C = 2.5 v v^T + 0.5 (I - v v^T), rejected >= 190 / 200
    d = 50
    v = np.random.default_rng(99).standard_normal(d)
    v /= np.linalg.norm(v)
    spike = lambda x: 0.5 * x + 2.0 * (v @ x) * v  # noqa: E731
    rng = P.RngState(99)
    rejected = 0
    for _ in range(200):
        ok, rng = P.verify_spectral(spike, d, P.VerifierState(delta=0.1), rng)
        rejected += not ok
    assert rejected >= 190


def test_matches_oracle_verifier(oracle):
    """Same operator, same stream position: the same verdict, the same draws consumed and the
    same verifier bookkeeping as the C restatement of shrink.cpp:75-102."""
    g = np.random.default_rng(7)
    for trial in range(12):
        d = int(g.integers(3, 60))
        m = g.standard_normal((d, d))
        c = m @ m.T
        c *= float(g.uniform(0.6, 1.4)) / np.linalg.eigvalsh(c).max()  # norm around the 1 threshold
        seed = 1000 + trial
        st, ost = P.VerifierState(delta=0.1, i=trial), OVer(delta=0.1, i=trial)
        ok, rng = P.verify_spectral(lambda x: c @ x, d, st, P.RngState(seed))
        orng = oracle.rng(seed)
        ook = oracle.verify_spectral(lambda x: c @ x, d, ost, orng)
        assert ok == ook, trial
        assert st.i == ost.i and st.delta_spent == ost.delta_spent
        assert rng.words == orng.state()[0]


def test_device_operator_mode():
    import torch
    d = 300
    g = np.random.default_rng(3)
    m = g.standard_normal((d, d))
    c = m @ m.T
    for scale, want in ((0.5, True), (2.0, False)):
        cs = c * scale / np.linalg.eigvalsh(c).max()
        ct = torch.from_numpy(cs).cuda()

        # device pointers wrapped without copies through __cuda_array_interface__
        class Buf:
            def __init__(self, ptr):
                self.__cuda_array_interface__ = {"shape": (d,), "typestr": "<f8", "data": (ptr, False),
                                                 "version": 3}

        def dev_op(xp, yp, n):
            x = torch.as_tensor(Buf(xp), device="cuda")
            y = torch.as_tensor(Buf(yp), device="cuda")
            torch.matmul(ct, x, out=y)
            torch.cuda.synchronize()

        st_d = P.VerifierState(delta=0.1)
        ok_d, r_d = P.verify_spectral(dev_op, d, st_d, P.RngState(11), on_device=True)
        st_h = P.VerifierState(delta=0.1)
        ok_h, r_h = P.verify_spectral(lambda x: cs @ x, d, st_h, P.RngState(11))
        assert ok_d == ok_h == want
        assert r_d.words == r_h.words and st_d.delta_spent == st_h.delta_spent
