"""ctypes bindings for the parity oracle.

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs -- never by the product package
``paper_1602_00412_b200``. Two back ends share one Python surface:

* ``Oracle()``   -- oracle/liboracle.so, the plain-C restatement (oracle/sfd_oracle.c)
* ``Reference()``-- oracle/_ref/libsfdref.so, the unmodified reference compiled from
                    /root/reference/proj/core/src plus oracle/ref_shim.cpp

Matrices are numpy float64, row-major, exactly the reference ``DenseMatrix`` layout
(core/include/sfd/dense_matrix.hpp:10-30). CSR inputs use int64 row_ptr, uint32 cols,
float64 vals like ``SparseBuffer`` (core/include/sfd/sparse.hpp:52-57).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libsfdref.so")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)
_szp = C.POINTER(C.c_size_t)

KALPHA = 6.0 / 41.0  # core/include/sfd/common.hpp:10


class OracleError(Exception):
    pass


class InvalidArgument(OracleError, ValueError):
    """std::invalid_argument (status 1)."""


class NumericalError(OracleError, ArithmeticError):
    """sfd::numerical_error (status 2)."""


def _raise(code: int, msg: str):
    if code == 1:
        raise InvalidArgument(msg)
    if code == 2:
        raise NumericalError(msg)
    raise OracleError(f"status {code}: {msg}")


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref when the reference sources are present)."""
    subprocess.run(["make", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def csr_arrays(row_ptr, cols, vals):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cs = np.ascontiguousarray(cols, dtype=np.uint32)
    vs = np.ascontiguousarray(vals, dtype=np.float64)
    return rp, cs, vs


class PowerConfig:
    """core/include/sfd/randsvd.hpp:10-14."""

    def __init__(self, epsilon=0.25, q_constant=1.0, q_override=None):
        self.epsilon = float(epsilon)
        self.q_constant = float(q_constant)
        self.q_override = q_override

    def as_tuple(self):
        return (self.epsilon, self.q_constant, -1 if self.q_override is None else int(self.q_override))


class _OrPower(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("q_constant", C.c_double), ("q_override", C.c_longlong)]


class _OrVerifier(C.Structure):
    _fields_ = [("i", C.c_size_t), ("delta", C.c_double), ("c_verify", C.c_double), ("delta_spent", C.c_double)]


class _OrCsr(C.Structure):
    _fields_ = [("row_ptr", _i64p), ("cols", _u32p), ("vals", _dp), ("m", C.c_size_t), ("d", C.c_size_t)]


class _OrSketchCfg(C.Structure):
    _fields_ = [("ell", C.c_size_t), ("d", C.c_size_t), ("delta", C.c_double), ("power", _OrPower),
                ("seed", C.c_uint64)]


class VerifierState:
    """core/include/sfd/shrink.hpp:11-16."""

    def __init__(self, delta=0.1, i=0, c_verify=2.0, delta_spent=0.0):
        self.i, self.delta, self.c_verify, self.delta_spent = i, delta, c_verify, delta_spent


_SYMOP = C.CFUNCTYPE(None, _dp, _dp, C.c_size_t, C.c_void_p)


class Oracle:
    """The plain-C restatement (oracle/sfd_oracle.c)."""

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.or_rng_new.restype = C.c_void_p
        L.or_rng_new.argtypes = [C.c_uint64]
        L.or_rng_free.argtypes = [C.c_void_p]
        for n, r in (("next_u64", C.c_uint64), ("uniform", C.c_double), ("normal", C.c_double),
                     ("normals_drawn", C.c_uint64)):
            f = getattr(L, "or_rng_" + n)
            f.restype = r
            f.argtypes = [C.c_void_p]
        L.or_rng_uniform_below.restype = C.c_uint64
        L.or_rng_uniform_below.argtypes = [C.c_void_p, C.c_uint64]
        L.or_rng_state.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int), _dp]
        L.or_last_error.restype = C.c_char_p
        L.or_power_iteration_count.argtypes = [C.c_size_t, C.c_double, C.c_double, C.c_longlong, _szp]
        L.or_jacobi_eigh.argtypes = [_dp, C.c_size_t, C.c_double, _dp, _dp]
        L.or_svd_top.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp, _dp, C.POINTER(C.c_int)]
        L.or_orthonormalize.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
        L.or_dense_shrink.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]
        L.or_fd_sketch.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, C.POINTER(C.c_size_t)]
        L.or_cov_err.argtypes = [C.POINTER(_OrCsr), _dp, C.c_size_t, C.c_void_p, C.c_size_t, C.POINTER(C.c_double)]
        L.or_proj_err.argtypes = [C.POINTER(_OrCsr), _dp, C.c_size_t, C.c_size_t, C.c_double,
                                  C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.or_exact_tail.argtypes = [C.POINTER(_OrCsr), C.c_size_t, C.c_void_p, _dp, C.POINTER(C.c_double),
                                    C.POINTER(C.c_size_t)]
        L.or_simultaneous_iteration.argtypes = [C.POINTER(_OrCsr), C.c_size_t, C.POINTER(_OrPower), C.c_void_p, _dp]
        L.or_sparse_shrink.argtypes = [C.POINTER(_OrCsr), C.c_size_t, C.POINTER(_OrPower), C.c_void_p, _dp]
        L.or_verify_spectral.argtypes = [_SYMOP, C.c_void_p, C.c_size_t, C.POINTER(_OrVerifier), C.c_void_p,
                                         C.POINTER(C.c_int)]
        L.or_boosted_sparse_shrink.argtypes = [C.POINTER(_OrCsr), C.c_size_t, C.POINTER(_OrVerifier),
                                               C.POINTER(_OrPower), C.c_void_p, _dp, _dp, _szp]
        L.or_merge.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]
        L.or_sketcher_new.argtypes = [C.POINTER(_OrSketchCfg), C.POINTER(C.c_void_p)]
        L.or_sketcher_free.argtypes = [C.c_void_p]
        L.or_sketcher_append_csr.argtypes = [C.c_void_p, _i64p, _u32p, _dp, C.c_size_t, _szp]
        L.or_sketcher_finalize.argtypes = [C.c_void_p, _dp]
        L.or_sketcher_get_sketch.argtypes = [C.c_void_p, _dp]
        L.or_sketcher_stats.argtypes = [C.c_void_p, _szp, _szp, _szp, _dp, _szp, _szp, _dp, C.POINTER(C.c_uint64)]
        L.or_sketcher_buffer_dense.argtypes = [C.c_void_p, _dp]

    def _chk(self, code):
        if code:
            _raise(code, self.L.or_last_error().decode())

    # ---- Rng ----
    def rng(self, seed: int) -> "Rng":
        return Rng(self, seed)

    def power_iteration_count(self, m, cfg: PowerConfig | None = None) -> int:
        cfg = cfg or PowerConfig()
        out = C.c_size_t()
        self._chk(self.L.or_power_iteration_count(m, *cfg.as_tuple(), C.byref(out)))
        return out.value

    def jacobi_eigh(self, sym, off_tol):
        s = _f64(sym)
        n = s.shape[0]
        vals = np.zeros(n)
        vecs = np.zeros((n, n))
        self._chk(self.L.or_jacobi_eigh(_ptr(s, _dp), n, off_tol, _ptr(vals, _dp), _ptr(vecs, _dp)))
        return vals, vecs

    def svd_top(self, a, r):
        a = _f64(a)
        m, d = a.shape
        sv = np.zeros(r)
        right = np.zeros((d, r))
        left = np.zeros((m, r))
        rd = C.c_int()
        self._chk(self.L.or_svd_top(_ptr(a, _dp), m, d, r, _ptr(sv, _dp), _ptr(right, _dp), _ptr(left, _dp),
                                    C.byref(rd)))
        return sv, right, left, bool(rd.value)

    def orthonormalize(self, a):
        a = _f64(a)
        n, k = a.shape
        out = np.zeros((n, k))
        self._chk(self.L.or_orthonormalize(_ptr(a, _dp), n, k, _ptr(out, _dp)))
        return out

    def dense_shrink(self, a, ell):
        a = _f64(a)
        rows, cols = a.shape
        out = np.zeros((ell, cols))
        self._chk(self.L.or_dense_shrink(_ptr(a, _dp), rows, cols, ell, _ptr(out, _dp)))
        return out

    def _csr(self, row_ptr, cols, vals, d):
        rp, cs, vs = csr_arrays(row_ptr, cols, vals)
        keep = (rp, cs, vs)
        return _OrCsr(_ptr(rp, _i64p), _ptr(cs, _u32p), _ptr(vs, _dp), len(rp) - 1, d), keep

    def simultaneous_iteration(self, csr, d, k, rng: "Rng", cfg: PowerConfig | None = None):
        c, keep = self._csr(*csr, d)
        pw = _OrPower(*(cfg or PowerConfig()).as_tuple())
        out = np.zeros((c.m, k))
        self._chk(self.L.or_simultaneous_iteration(C.byref(c), k, C.byref(pw), rng.h, _ptr(out, _dp)))
        return out

    def sparse_shrink(self, csr, d, ell, rng: "Rng", cfg: PowerConfig | None = None):
        c, keep = self._csr(*csr, d)
        pw = _OrPower(*(cfg or PowerConfig()).as_tuple())
        out = np.zeros((ell, d))
        self._chk(self.L.or_sparse_shrink(C.byref(c), ell, C.byref(pw), rng.h, _ptr(out, _dp)))
        return out

    def verify_spectral(self, op, d, state: VerifierState, rng: "Rng") -> bool:
        def _cb(xp, yp, n, _ctx):
            x = np.ctypeslib.as_array(xp, shape=(n,))
            y = np.ctypeslib.as_array(yp, shape=(n,))
            y[:] = op(x.copy())
        cb = _SYMOP(_cb)
        st = _OrVerifier(state.i, state.delta, state.c_verify, state.delta_spent)
        acc = C.c_int()
        self._chk(self.L.or_verify_spectral(cb, None, d, C.byref(st), rng.h, C.byref(acc)))
        state.i, state.delta_spent = st.i, st.delta_spent
        return bool(acc.value)

    def boosted_sparse_shrink(self, csr, d, ell, state: VerifierState, rng: "Rng", cfg: PowerConfig | None = None):
        c, keep = self._csr(*csr, d)
        pw = _OrPower(*(cfg or PowerConfig()).as_tuple())
        st = _OrVerifier(state.i, state.delta, state.c_verify, state.delta_spent)
        out = np.zeros((ell, d))
        dh = C.c_double()
        att = C.c_size_t()
        self._chk(self.L.or_boosted_sparse_shrink(C.byref(c), ell, C.byref(st), C.byref(pw), rng.h, _ptr(out, _dp),
                                                  C.byref(dh), C.byref(att)))
        state.i, state.delta_spent = st.i, st.delta_spent
        return out, dh.value, att.value

    def merge(self, b1, b2, ell):
        b1, b2 = _f64(b1), _f64(b2)
        if b1.shape[1] != b2.shape[1]:
            raise InvalidArgument("merge: column mismatch")
        d = b1.shape[1]
        out = np.zeros((ell, d))
        self._chk(self.L.or_merge(_ptr(b1, _dp), b1.shape[0], _ptr(b2, _dp), b2.shape[0], d, ell, _ptr(out, _dp)))
        return out

    def cov_err(self, row_ptr, cols, vals, d, sketch, rng: "Rng", iterations=1000):
        """cov_err (bench.cpp:171-183): |A^T A - B^T B|_2 / |A|_F^2; rng advanced."""
        keep = self._csr(row_ptr, cols, vals, d)
        b = _f64(sketch)
        out = C.c_double()
        self._chk(self.L.or_cov_err(C.byref(keep[0]), _ptr(b, _dp), b.shape[0], rng.h, iterations, C.byref(out)))
        return out.value

    def proj_err(self, row_ptr, cols, vals, d, sketch, k, tail_sq):
        """proj_err (bench.cpp:139-169): value or None (the reference's nullopt)."""
        keep = self._csr(row_ptr, cols, vals, d)
        b = _f64(sketch)
        out, has = C.c_double(), C.c_int()
        self._chk(self.L.or_proj_err(C.byref(keep[0]), _ptr(b, _dp), b.shape[0], k, tail_sq, C.byref(out),
                                     C.byref(has)))
        return out.value if has.value else None

    def exact_tail(self, row_ptr, cols, vals, d, k, rng: "Rng"):
        """exact_tail (bench.cpp:68-137): (tail_sq, sigma[k], sweeps); rng advanced."""
        keep = self._csr(row_ptr, cols, vals, d)
        sig = np.zeros(max(1, k))
        tail = C.c_double()
        sw = C.c_size_t()
        self._chk(self.L.or_exact_tail(C.byref(keep[0]), k, rng.h, _ptr(sig, _dp), C.byref(tail), C.byref(sw)))
        return tail.value, sig[:k], sw.value

    def fd_sketch(self, rows, ell):
        """FdSketcher whole-stream run (sketch.cpp:47-78): (B ell x d, shrink_count)."""
        a = _f64(np.atleast_2d(rows))
        n, d = a.shape
        out = np.zeros((ell, d))
        cnt = C.c_size_t()
        self._chk(self.L.or_fd_sketch(_ptr(a, _dp), n, d, ell, _ptr(out, _dp), C.byref(cnt)))
        return out, cnt.value

    def sketcher(self, ell, d, seed=0, delta=0.1, power: PowerConfig | None = None) -> "OracleSketcher":
        return OracleSketcher(self, ell, d, seed, delta, power or PowerConfig())

    def sketch(self, row_ptr, cols, vals, d, ell, seed=0, delta=0.1, power: PowerConfig | None = None):
        """Whole-stream run: returns (B, stats dict)."""
        s = self.sketcher(ell, d, seed, delta, power)
        s.append_csr(row_ptr, cols, vals)
        b = s.finalize()
        return b, s.stats()


class Rng:
    """core/include/sfd/rng.hpp:12-31 over the oracle's mt19937_64."""

    def __init__(self, lib: Oracle, seed: int):
        self.lib = lib
        self.seed = seed
        self.h = lib.L.or_rng_new(C.c_uint64(seed))

    def __del__(self):
        try:
            self.lib.L.or_rng_free(self.h)
        except Exception:
            pass

    def next_u64(self):
        return self.lib.L.or_rng_next_u64(self.h)

    def uniform(self):
        return self.lib.L.or_rng_uniform(self.h)

    def uniform_below(self, n):
        if n == 0:
            raise InvalidArgument("uniform_below: n must be positive")
        return self.lib.L.or_rng_uniform_below(self.h, n)

    def normal(self):
        return self.lib.L.or_rng_normal(self.h)

    def normals_drawn(self):
        return self.lib.L.or_rng_normals_drawn(self.h)

    def state(self):
        """(seed-relative raw words consumed, has_spare, spare) -- the full Rng draw state."""
        w, hs, sp = C.c_uint64(), C.c_int(), C.c_double()
        self.lib.L.or_rng_state(self.h, C.byref(w), C.byref(hs), C.byref(sp))
        return w.value, bool(hs.value), sp.value


class OracleSketcher:
    """core/include/sfd/sketch.hpp:22-49 (SfdSketcher) over the C restatement."""

    def __init__(self, lib: Oracle, ell, d, seed, delta, power: PowerConfig):
        self.lib, self.ell, self.d = lib, ell, d
        cfg = _OrSketchCfg(ell, d, delta, _OrPower(*power.as_tuple()), seed)
        h = C.c_void_p()
        lib._chk(lib.L.or_sketcher_new(C.byref(cfg), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.lib.L.or_sketcher_free(self.h)
        except Exception:
            pass

    def append(self, indices, values):
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        val = np.ascontiguousarray(values, dtype=np.float64)
        if len(idx) != len(val):
            raise InvalidArgument("append_row: index/value length mismatch")
        self.append_csr(np.array([0, len(idx)]), idx, val)

    def append_csr(self, row_ptr, cols, vals):
        rp, cs, vs = csr_arrays(row_ptr, cols, vals)
        done = C.c_size_t()
        if len(cs) == 0:
            cs = np.zeros(1, np.uint32)
            vs = np.zeros(1)
        self.lib._chk(self.lib.L.or_sketcher_append_csr(self.h, _ptr(rp, _i64p), _ptr(cs, _u32p), _ptr(vs, _dp),
                                                        len(rp) - 1, C.byref(done)))
        return done.value

    def finalize(self):
        out = np.zeros((self.ell, self.d))
        self.lib._chk(self.lib.L.or_sketcher_finalize(self.h, _ptr(out, _dp)))
        return out

    def sketch(self):
        out = np.zeros((self.ell, self.d))
        self.lib.L.or_sketcher_get_sketch(self.h, _ptr(out, _dp))
        return out

    def stats(self):
        f, a, i, r, z = (C.c_size_t() for _ in range(5))
        ds, fr = C.c_double(), C.c_double()
        nd = C.c_uint64()
        self.lib.L.or_sketcher_stats(self.h, C.byref(f), C.byref(a), C.byref(i), C.byref(ds), C.byref(r),
                                     C.byref(z), C.byref(fr), C.byref(nd))
        return {"flushes": f.value, "attempts": a.value, "verifier_i": i.value, "delta_spent": ds.value,
                "buf_rows": r.value, "buf_nnz": z.value, "buf_frob_sq": fr.value, "normals_drawn": nd.value}

    def buffer_dense(self):
        st = self.stats()
        out = np.zeros((st["buf_rows"], self.d))
        self.lib.L.or_sketcher_buffer_dense(self.h, _ptr(out, _dp))
        return out


class Reference:
    """The unmodified reference (oracle/_ref/libsfdref.so) -- same surface, fewer entry points."""

    def __init__(self, path: str = LIB_REF):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (reference sources absent?)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_free.argtypes = [C.c_void_p]
        for n, r in (("next_u64", C.c_uint64), ("uniform", C.c_double), ("normal", C.c_double)):
            f = getattr(L, "ref_rng_" + n)
            f.restype = r
            f.argtypes = [C.c_void_p]
        L.ref_rng_uniform_below.restype = C.c_uint64
        L.ref_rng_uniform_below.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_dense_shrink.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]
        L.ref_orthonormalize.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
        L.ref_jacobi_eigh.argtypes = [_dp, C.c_size_t, C.c_double, _dp, _dp]
        csr = [_i64p, _u32p, _dp, C.c_size_t, C.c_size_t]
        pw = [C.c_double, C.c_double, C.c_longlong]
        L.ref_sparse_shrink.argtypes = csr + [C.c_size_t] + pw + [C.c_void_p, _dp]
        L.ref_simultaneous_iteration.argtypes = csr + [C.c_size_t] + pw + [C.c_void_p, _dp]
        L.ref_boosted_sparse_shrink.argtypes = csr + [C.c_size_t, _dp] + pw + [C.c_void_p, _dp, _dp, _szp]
        L.ref_merge.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]
        L.ref_sketch.argtypes = csr + [C.c_size_t, C.c_double] + pw + [C.c_uint64, _dp, _dp]
        L.ref_cov_err.argtypes = csr + [_dp, C.c_size_t, C.c_void_p, C.c_size_t, C.POINTER(C.c_double)]
        L.ref_exact_tail.argtypes = csr + [C.c_size_t, C.c_void_p, _dp, C.POINTER(C.c_double)]
        L.ref_proj_err.argtypes = csr + [_dp, C.c_size_t, C.c_size_t, C.c_double, C.POINTER(C.c_double),
                                         C.POINTER(C.c_int)]

    def _chk(self, code):
        if code:
            _raise(code, self.L.ref_last_error().decode())

    def rng(self, seed):
        return RefRng(self, seed)

    def dense_shrink(self, a, ell):
        a = _f64(a)
        out = np.zeros((ell, a.shape[1]))
        self._chk(self.L.ref_dense_shrink(_ptr(a, _dp), a.shape[0], a.shape[1], ell, _ptr(out, _dp)))
        return out

    def orthonormalize(self, a):
        a = _f64(a)
        out = np.zeros_like(a)
        self._chk(self.L.ref_orthonormalize(_ptr(a, _dp), a.shape[0], a.shape[1], _ptr(out, _dp)))
        return out

    def jacobi_eigh(self, sym, off_tol):
        s = _f64(sym)
        n = s.shape[0]
        vals, vecs = np.zeros(n), np.zeros((n, n))
        self._chk(self.L.ref_jacobi_eigh(_ptr(s, _dp), n, off_tol, _ptr(vals, _dp), _ptr(vecs, _dp)))
        return vals, vecs

    def _csr(self, row_ptr, cols, vals, d):
        rp, cs, vs = csr_arrays(row_ptr, cols, vals)
        if len(cs) == 0:
            cs, vs = np.zeros(1, np.uint32), np.zeros(1)
        return (_ptr(rp, _i64p), _ptr(cs, _u32p), _ptr(vs, _dp), len(rp) - 1, d), (rp, cs, vs)

    def sparse_shrink(self, csr, d, ell, rng, cfg: PowerConfig | None = None):
        args, keep = self._csr(*csr, d)
        out = np.zeros((ell, d))
        self._chk(self.L.ref_sparse_shrink(*args, ell, *(cfg or PowerConfig()).as_tuple(), rng.h, _ptr(out, _dp)))
        return out

    def simultaneous_iteration(self, csr, d, k, rng, cfg: PowerConfig | None = None):
        args, keep = self._csr(*csr, d)
        out = np.zeros((args[3], k))
        self._chk(self.L.ref_simultaneous_iteration(*args, k, *(cfg or PowerConfig()).as_tuple(), rng.h,
                                                    _ptr(out, _dp)))
        return out

    def boosted_sparse_shrink(self, csr, d, ell, state: VerifierState, rng, cfg: PowerConfig | None = None):
        args, keep = self._csr(*csr, d)
        st = np.array([state.i, state.delta, state.c_verify, state.delta_spent], dtype=np.float64)
        out = np.zeros((ell, d))
        dh = C.c_double()
        att = C.c_size_t()
        self._chk(self.L.ref_boosted_sparse_shrink(*args, ell, _ptr(st, _dp), *(cfg or PowerConfig()).as_tuple(),
                                                   rng.h, _ptr(out, _dp), C.byref(dh), C.byref(att)))
        state.i, state.delta_spent = int(st[0]), st[3]
        return out, dh.value, att.value

    def merge(self, b1, b2, ell):
        b1, b2 = _f64(b1), _f64(b2)
        out = np.zeros((ell, b1.shape[1]))
        self._chk(self.L.ref_merge(_ptr(b1, _dp), b1.shape[0], _ptr(b2, _dp), b2.shape[0], b1.shape[1], ell,
                                   _ptr(out, _dp)))
        return out

    def fd_sketch(self, rows, ell):
        a = _f64(np.atleast_2d(rows))
        n, d = a.shape
        out = np.zeros((ell, d))
        cnt = C.c_size_t()
        self._chk(self.L.ref_fd_sketch(_ptr(a, _dp), C.c_size_t(n), C.c_size_t(d), C.c_size_t(ell), _ptr(out, _dp),
                                       C.byref(cnt)))
        return out, cnt.value

    def read_row_stream(self, path, plain_cols=0):
        """open_row_stream (io.cpp:170-189) read to the end by the compiled reference reader
        (oracle/_ref/refio): (row_ptr, cols, vals, d, error message or None)."""
        import subprocess
        exe = os.path.join(os.path.dirname(LIB_REF), "refio")
        raw = subprocess.run([exe, path, str(plain_cols)], capture_output=True, check=True).stdout
        n, d, z, err, ml = np.frombuffer(raw[:40], np.int64)
        off = 40
        msg = raw[off:off + ml].decode()
        off += ml
        rp = np.frombuffer(raw[off:off + 8 * (n + 1)], np.int64).copy()
        off += 8 * (n + 1)
        cs = np.frombuffer(raw[off:off + 4 * z], np.uint32).copy()
        off += 4 * z
        vs = np.frombuffer(raw[off:off + 8 * z], np.float64).copy()
        return rp, cs, vs, int(d), (msg if err else None)

    def proj_err(self, row_ptr, cols, vals, d, sketch, k, tail_sq):
        args, keep = self._csr(row_ptr, cols, vals, d)
        b = _f64(sketch)
        out, has = C.c_double(), C.c_int()
        self._chk(self.L.ref_proj_err(*args, _ptr(b, _dp), b.shape[0], k, tail_sq, C.byref(out), C.byref(has)))
        return out.value if has.value else None

    def exact_tail(self, row_ptr, cols, vals, d, k, rng):
        args, keep = self._csr(row_ptr, cols, vals, d)
        sig = np.zeros(max(1, k))
        tail = C.c_double()
        self._chk(self.L.ref_exact_tail(*args, k, rng.h, _ptr(sig, _dp), C.byref(tail)))
        return tail.value, sig[:k]

    def cov_err(self, row_ptr, cols, vals, d, sketch, rng, iterations=1000):
        args, keep = self._csr(row_ptr, cols, vals, d)
        b = _f64(sketch)
        out = C.c_double()
        self._chk(self.L.ref_cov_err(*args, _ptr(b, _dp), b.shape[0], rng.h, iterations, C.byref(out)))
        return out.value

    def power_sweep(self, row_ptr, cols, vals, d, y):
        """One simultaneous_iteration sweep (randsvd.cpp:39-48) from y (m x k): (y', seconds)."""
        args, keep = self._csr(row_ptr, cols, vals, d)
        y = _f64(y)
        out = np.zeros_like(y)
        secs = C.c_double()
        self.L.ref_power_sweep.argtypes = [_i64p, _u32p, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp,
                                           C.POINTER(C.c_double)]
        self._chk(self.L.ref_power_sweep(*args, y.shape[1], _ptr(y, _dp), _ptr(out, _dp), C.byref(secs)))
        return out, secs.value

    def sketch(self, row_ptr, cols, vals, d, ell, seed=0, delta=0.1, power: PowerConfig | None = None):
        args, keep = self._csr(row_ptr, cols, vals, d)
        out = np.zeros((ell, d))
        stats = np.zeros(4)
        self._chk(self.L.ref_sketch(*args, ell, delta, *(power or PowerConfig()).as_tuple(), seed, _ptr(out, _dp),
                                    _ptr(stats, _dp)))
        return out, {"flushes": int(stats[0]), "attempts": int(stats[1]), "verifier_i": int(stats[2]),
                     "delta_spent": float(stats[3])}


class RefSketcher:
    """A live reference SfdSketcher (oracle/ref_shim.cpp ref_sketcher_*), appended row by row."""

    def __init__(self, lib: Reference, ell, d, seed=0, delta=0.1):
        L = lib.L
        L.ref_sketcher_new.restype = C.c_void_p
        L.ref_sketcher_new.argtypes = [C.c_size_t, C.c_size_t, C.c_double, C.c_uint64]
        L.ref_sketcher_free.argtypes = [C.c_void_p]
        L.ref_sketcher_append.argtypes = [C.c_void_p, _u32p, _dp, C.c_size_t]
        L.ref_sketcher_sketch.argtypes = [C.c_void_p, _dp]
        L.ref_sketcher_stats.argtypes = [C.c_void_p, _dp]
        self.lib, self.ell, self.d = lib, ell, d
        self.h = L.ref_sketcher_new(ell, d, delta, C.c_uint64(seed))
        if not self.h:
            _raise(1, L.ref_last_error().decode())

    def __del__(self):
        try:
            self.lib.L.ref_sketcher_free(self.h)
        except Exception:
            pass

    def append(self, indices, values):
        cs = np.ascontiguousarray(indices, dtype=np.uint32)
        vs = np.ascontiguousarray(values, dtype=np.float64)
        if cs.size == 0:
            cs, vs = np.zeros(1, np.uint32), np.zeros(1)
            n = 0
        else:
            n = cs.size
        self.lib._chk(self.lib.L.ref_sketcher_append(self.h, _ptr(cs, _u32p), _ptr(vs, _dp), n))

    def sketch(self):
        out = np.zeros((self.ell, self.d))
        self.lib.L.ref_sketcher_sketch(self.h, _ptr(out, _dp))
        return out

    def stats(self):
        st = np.zeros(7)
        self.lib.L.ref_sketcher_stats(self.h, _ptr(st, _dp))
        return {"flushes": int(st[0]), "attempts": int(st[1]), "verifier_i": int(st[2]), "delta_spent": float(st[3]),
                "buf_rows": int(st[4]), "buf_nnz": int(st[5]), "buf_frob_sq": float(st[6])}


class RefRng:
    def __init__(self, lib: Reference, seed):
        self.lib = lib
        self.h = lib.L.ref_rng_new(C.c_uint64(seed))

    def __del__(self):
        try:
            self.lib.L.ref_rng_free(self.h)
        except Exception:
            pass

    def next_u64(self):
        return self.lib.L.ref_rng_next_u64(self.h)

    def uniform(self):
        return self.lib.L.ref_rng_uniform(self.h)

    def uniform_below(self, n):
        return self.lib.L.ref_rng_uniform_below(self.h, n)

    def normal(self):
        return self.lib.L.ref_rng_normal(self.h)
