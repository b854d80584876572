"""B200-native Sparse Frequent Directions (arXiv 1602.00412) -- host-side mirror.

The product is ``libsfdg.so`` (CUDA, sm_100a) behind the C ABI in ``include/sfdg.h``.
This module binds that ABI with ctypes and mirrors the reference C++ interface
(/root/reference/proj/core/include/sfd/sketch.hpp:9-71, shrink.hpp:11-41,
randsvd.hpp:10-26, la_core.hpp:23-41) so parity tests read like the reference's own:

    cfg = SketchConfig(ell=100, d=10_000, seed=1)
    s = SfdSketcher(cfg)              # SfdSketcher(const SketchConfig&)
    s.append(indices, values)         # append(const SparseRow&)
    s.append_csr(row_ptr, cols, vals) # many rows, same per-row trigger semantics
    B = s.finalize()                  # ell x d, float64

Errors map to the reference's exception classes: ``InvalidArgument`` (ValueError) for
std::invalid_argument, ``NumericalError`` (ArithmeticError) for sfd::numerical_error.
There is no CPU fallback: importing works anywhere, but every compute call needs the
CUDA library and a GPU and raises ``CudaError`` otherwise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = [
    "SketchConfig", "PowerConfig", "VerifierState", "RngState", "SfdSketcher", "merge", "merge_device",
    "dense_shrink", "sparse_shrink", "boosted_sparse_shrink", "verify_spectral", "simultaneous_iteration",
    "power_iteration_count",
    "gaussian_matrix", "eigh", "orthonormalize", "csr_products", "device_count", "launch_count", "lib",
    "InvalidArgument", "NumericalError", "CudaError", "KALPHA", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsfdg.so")
KALPHA = 6.0 / 41.0  # core/include/sfd/common.hpp:10


class SfdError(Exception):
    pass


class InvalidArgument(SfdError, ValueError):
    """std::invalid_argument (SFDG_INVALID_ARGUMENT)."""


class NumericalError(SfdError, ArithmeticError):
    """sfd::numerical_error (SFDG_NUMERICAL_ERROR)."""


class CudaError(SfdError, RuntimeError):
    """Device fault or no device (SFDG_CUDA_ERROR)."""


_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)
_szp = C.POINTER(C.c_size_t)


class _Power(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("q_constant", C.c_double), ("q_override", C.c_int64)]


class _SketchCfg(C.Structure):
    _fields_ = [("ell", C.c_size_t), ("d", C.c_size_t), ("delta", C.c_double), ("power", _Power),
                ("seed", C.c_uint64)]


class _Rng(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("words", C.c_uint64), ("has_spare", C.c_int32), ("spare", C.c_double)]


class _Verifier(C.Structure):
    _fields_ = [("i", C.c_size_t), ("delta", C.c_double), ("c_verify", C.c_double), ("delta_spent", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("flush_count", C.c_size_t), ("attempt_total", C.c_size_t), ("verifier", _Verifier),
                ("buffer_rows", C.c_size_t), ("buffer_nnz", C.c_size_t), ("buffer_frob_sq", C.c_double),
                ("rng", _Rng)]


_LIB = None


def lib() -> C.CDLL:
    """Load libsfdg.so (fails loudly when it was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `make -C {HERE}` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    L.sfdg_last_error.restype = C.c_char_p
    L.sfdg_version.restype = C.c_char_p
    L.sfdg_launch_count.restype = C.c_uint64
    L.sfdg_device_count.argtypes = [C.POINTER(C.c_int)]
    L.sfdg_sketcher_create.argtypes = [C.POINTER(_SketchCfg), C.c_int, C.POINTER(C.c_void_p)]
    L.sfdg_sketcher_destroy.argtypes = [C.c_void_p]
    L.sfdg_sketcher_append_csr.argtypes = [C.c_void_p, _i64p, _u32p, _dp, C.c_size_t, _szp]
    L.sfdg_sketcher_append_csr_device.argtypes = [C.c_void_p, _i64p, C.c_void_p, C.c_void_p, C.c_size_t, _szp]
    L.sfdg_sketcher_finalize.argtypes = [C.c_void_p, _dp]
    L.sfdg_sketcher_get_sketch.argtypes = [C.c_void_p, _dp]
    L.sfdg_sketcher_get_sketch_device.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    L.sfdg_sketcher_stats.argtypes = [C.c_void_p, C.POINTER(_Stats)]
    L.sfdg_sketcher_get_buffer.argtypes = [C.c_void_p, _i64p, _u32p, _dp]
    L.sfdg_sketcher_synchronize.argtypes = [C.c_void_p]
    L.sfdg_sketcher_reset.argtypes = [C.c_void_p, C.c_uint64]
    L.sfdg_sketcher_merge_device.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    L.sfdg_merge.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, C.c_int]
    L.sfdg_merge_device.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p, C.c_int,
                                    C.c_void_p]
    L.sfdg_dense_shrink.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, C.c_int]
    L.sfdg_sketch_file.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(_SketchCfg), C.c_int, _dp, C.POINTER(_Stats),
                                   _szp]
    L.sfdg_read_row_stream.argtypes = [C.c_char_p, C.c_size_t, _szp, _szp, _szp, _i64p, _u32p, _dp]
    L.sfdg_proj_err.argtypes = [_i64p, _u32p, _dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double,
                                C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int]
    L.sfdg_exact_tail.argtypes = [_i64p, _u32p, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.POINTER(_Rng), _dp,
                                  C.POINTER(C.c_double), _szp, C.c_int]
    L.sfdg_cov_err.argtypes = [_i64p, _u32p, _dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, C.c_size_t,
                               C.POINTER(_Rng), C.POINTER(C.c_double), C.c_int]
    L.sfdg_fd_create.argtypes = [C.c_size_t, C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]
    L.sfdg_fd_destroy.argtypes = [C.c_void_p]
    L.sfdg_fd_append.argtypes = [C.c_void_p, _dp, C.c_size_t]
    L.sfdg_fd_append_csr.argtypes = [C.c_void_p, _i64p, _u32p, _dp, C.c_size_t]
    L.sfdg_fd_finalize.argtypes = [C.c_void_p, _dp]
    L.sfdg_fd_shrink_count.argtypes = [C.c_void_p, C.POINTER(C.c_size_t)]
    L.sfdg_sharded_sketch.argtypes = [C.POINTER(_SketchCfg), _i64p, _u32p, _dp, C.c_size_t, C.c_int,
                                      C.POINTER(C.c_int), C.c_int, _dp, C.POINTER(_Stats)]
    csr = [_i64p, _u32p, _dp, C.c_size_t, C.c_size_t]
    L.sfdg_sparse_shrink.argtypes = csr + [C.c_size_t, C.POINTER(_Power), C.POINTER(_Rng), _dp, C.c_int]
    L.sfdg_boosted_sparse_shrink.argtypes = csr + [C.c_size_t, C.POINTER(_Verifier), C.POINTER(_Power),
                                                   C.POINTER(_Rng), _dp, _dp, _szp, C.c_int]
    L.sfdg_simultaneous_iteration.argtypes = csr + [C.c_size_t, C.POINTER(_Power), C.POINTER(_Rng), _dp, C.c_int]
    L.sfdg_power_iteration_count.argtypes = [C.c_size_t, C.POINTER(_Power), _szp]
    L.sfdg_gaussian_matrix.argtypes = [C.POINTER(_Rng), C.c_size_t, C.c_size_t, _dp, C.c_int]
    L.sfdg_eigh.argtypes = [_dp, C.c_size_t, C.c_double, _dp, _dp, C.c_int]
    L.sfdg_orthonormalize.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_int]
    L.sfdg_csr_products.argtypes = csr + [C.c_size_t, _dp, _dp, _dp, _dp, C.c_int]
    L.sfdg_profile_end.argtypes = [C.c_char_p, C.c_size_t]
    _LIB = L
    return L


def profile_begin() -> None:
    """Start per-kernel-class CUDA-event timing inside the library."""
    lib().sfdg_profile_begin()


def profile_end() -> dict:
    """Stop timing; returns {kernel_class: (total_ms, launches, flops, bytes)} -- the flops /
    bytes are the algorithmic work the library declared for those launches."""
    import json
    buf = C.create_string_buffer(1 << 16)
    lib().sfdg_profile_end(buf, len(buf))
    return {k: (v[0], v[1], v[2], v[3]) for k, v in json.loads(buf.value.decode()).items()}


def _check(code: int) -> None:
    if code == 0:
        return
    msg = lib().sfdg_last_error().decode(errors="replace")
    if code == 1:
        raise InvalidArgument(msg)
    if code == 2:
        raise NumericalError(msg)
    raise CudaError(msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _csr(row_ptr, cols, vals):
    """Host CSR in the C ABI's types. The C side trusts row_ptr for its reads, so the array
    shapes are checked here: row_ptr non-decreasing from >= 0, row_ptr[-1] <= len(cols) ==
    len(vals) (the reference rejects an index/value length mismatch, sparse.cpp:9-10), and
    column ids representable as uint32 (a wider id must not wrap onto a valid column)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    c_in = np.asarray(cols)
    if c_in.size and c_in.dtype != np.uint32:
        if c_in.dtype.kind not in "iu":
            raise InvalidArgument("SparseRow: column indices must be integers")
        if int(c_in.min()) < 0 or int(c_in.max()) > 0xFFFFFFFF:
            raise InvalidArgument("SparseRow: index out of range")
    cs = np.ascontiguousarray(c_in, dtype=np.uint32)
    vs = np.ascontiguousarray(vals, dtype=np.float64)
    if rp.ndim != 1 or rp.size < 1:
        raise InvalidArgument("row_ptr must be a 1-d array of n+1 offsets")
    if cs.size != vs.size:
        raise InvalidArgument("SparseRow: indices and values size mismatch")
    if rp[0] < 0 or (rp.size > 1 and bool(np.any(np.diff(rp) < 0))):
        raise InvalidArgument("row_ptr must be non-decreasing from a non-negative offset")
    if int(rp[-1]) > cs.size:
        raise InvalidArgument("row_ptr[-1] exceeds the number of stored entries")
    if cs.size == 0:  # keep valid pointers for empty inputs
        cs, vs = np.zeros(1, np.uint32), np.zeros(1)
    return rp, cs, vs


class PowerConfig:
    """randsvd.hpp:10-14 (q_override None = unset)."""

    def __init__(self, epsilon: float = 0.25, q_constant: float = 1.0, q_override: int | None = None):
        self.epsilon, self.q_constant, self.q_override = float(epsilon), float(q_constant), q_override

    def _c(self) -> _Power:
        return _Power(self.epsilon, self.q_constant, -1 if self.q_override is None else int(self.q_override))


class SketchConfig:
    """sketch.hpp:9-17."""

    def __init__(self, ell: int = 0, d: int = 0, delta: float = 0.1, power: PowerConfig | None = None, seed: int = 0):
        self.ell, self.d, self.delta, self.seed = int(ell), int(d), float(delta), int(seed)
        self.power = power or PowerConfig()

    def _c(self) -> _SketchCfg:
        return _SketchCfg(self.ell, self.d, self.delta, self.power._c(), self.seed)


class VerifierState:
    """shrink.hpp:11-16."""

    def __init__(self, delta: float = 0.1, i: int = 0, c_verify: float = 2.0, delta_spent: float = 0.0):
        self.i, self.delta, self.c_verify, self.delta_spent = int(i), float(delta), float(c_verify), float(delta_spent)

    def _c(self) -> _Verifier:
        return _Verifier(self.i, self.delta, self.c_verify, self.delta_spent)

    def _update(self, v: _Verifier) -> None:
        self.i, self.delta_spent = int(v.i), float(v.delta_spent)

    def __repr__(self):
        return f"VerifierState(i={self.i}, delta={self.delta}, delta_spent={self.delta_spent})"


class RngState:
    """Position in sfd::Rng's stream (rng.hpp:12-31): Rng(seed) after `words` raw draws."""

    def __init__(self, seed: int = 0, words: int = 0, has_spare: bool = False, spare: float = 0.0):
        self.seed, self.words, self.has_spare, self.spare = int(seed), int(words), bool(has_spare), float(spare)

    def _c(self) -> _Rng:
        return _Rng(self.seed, self.words, 1 if self.has_spare else 0, self.spare)

    def _update(self, r: _Rng) -> None:
        self.words, self.has_spare, self.spare = int(r.words), bool(r.has_spare), float(r.spare)

    def __repr__(self):
        return f"RngState(seed={self.seed}, words={self.words}, has_spare={self.has_spare})"


def device_count() -> int:
    n = C.c_int()
    lib().sfdg_device_count(C.byref(n))
    return n.value


def launch_count() -> int:
    return int(lib().sfdg_launch_count())


class SfdSketcher:
    """sfd::SfdSketcher (sketch.hpp:22-49) running on one B200."""

    def __init__(self, cfg: SketchConfig, device: int = 0):
        self.cfg = cfg
        self.device = device
        self._h = C.c_void_p()
        c = cfg._c()
        _check(lib().sfdg_sketcher_create(C.byref(c), device, C.byref(self._h)))

    def close(self) -> None:
        if self._h:
            lib().sfdg_sketcher_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- append ------------------------------------------------------------
    def append(self, indices, values) -> None:
        """append(const SparseRow&) (sketch.cpp:20-23)."""
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        val = np.ascontiguousarray(values, dtype=np.float64)
        if idx.shape != val.shape:
            raise InvalidArgument("append_row: index/value length mismatch")
        if idx.size and (idx.min() < 0 or idx.max() >= 2 ** 32):
            raise InvalidArgument("append_row: column index out of range")
        self.append_csr(np.array([0, idx.size], dtype=np.int64), idx.astype(np.uint32), val)

    def append_csr(self, row_ptr, cols, vals) -> int:
        """Append many rows; returns rows committed. Raises on the first bad row."""
        rp, cs, vs = _csr(row_ptr, cols, vals)
        done = C.c_size_t()
        _check(lib().sfdg_sketcher_append_csr(self._h, _p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1,
                                              C.byref(done)))
        return done.value

    def append_csr_device(self, h_row_ptr, d_cols_ptr: int, d_vals_ptr: int) -> int:
        """Rows whose cols/vals already live in this GPU's memory (raw device pointers)."""
        rp = np.ascontiguousarray(h_row_ptr, dtype=np.int64)
        done = C.c_size_t()
        _check(lib().sfdg_sketcher_append_csr_device(self._h, _p(rp, _i64p), C.c_void_p(d_cols_ptr),
                                                     C.c_void_p(d_vals_ptr), len(rp) - 1, C.byref(done)))
        return done.value

    # ---- results / accessors -------------------------------------------------
    def finalize(self) -> np.ndarray:
        out = np.zeros((self.cfg.ell, self.cfg.d))
        _check(lib().sfdg_sketcher_finalize(self._h, _p(out, _dp)))
        return out

    def sketch(self) -> np.ndarray:
        out = np.zeros((self.cfg.ell, self.cfg.d))
        _check(lib().sfdg_sketcher_get_sketch(self._h, _p(out, _dp)))
        return out

    def sketch_device_t(self, d_out_ptr: int, ld: int) -> None:
        """B^T (d x ell, leading dimension ld) into device memory (merge tree input)."""
        _check(lib().sfdg_sketcher_get_sketch_device(self._h, C.c_void_p(d_out_ptr), ld))

    def _stats(self) -> _Stats:
        s = _Stats()
        _check(lib().sfdg_sketcher_stats(self._h, C.byref(s)))
        return s

    def flush_count(self) -> int:
        return int(self._stats().flush_count)

    def attempt_total(self) -> int:
        return int(self._stats().attempt_total)

    def verifier(self) -> VerifierState:
        v = self._stats().verifier
        return VerifierState(v.delta, v.i, v.c_verify, v.delta_spent)

    def rng_state(self) -> RngState:
        r = self._stats().rng
        return RngState(r.seed, r.words, bool(r.has_spare), r.spare)

    def stats(self) -> dict:
        s = self._stats()
        return {"flushes": s.flush_count, "attempts": s.attempt_total, "verifier_i": s.verifier.i,
                "delta_spent": s.verifier.delta_spent, "buf_rows": s.buffer_rows, "buf_nnz": s.buffer_nnz,
                "buf_frob_sq": s.buffer_frob_sq, "rng_words": s.rng.words, "rng_has_spare": bool(s.rng.has_spare)}

    def buffer(self):
        """buffer(): (row_ptr int64, cols uint32, vals float64) of the unflushed rows."""
        s = self._stats()
        rp = np.zeros(s.buffer_rows + 1, np.int64)
        cs = np.zeros(max(1, s.buffer_nnz), np.uint32)
        vs = np.zeros(max(1, s.buffer_nnz))
        _check(lib().sfdg_sketcher_get_buffer(self._h, _p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp)))
        return rp, cs[: s.buffer_nnz], vs[: s.buffer_nnz]

    def buffer_dense(self) -> np.ndarray:
        rp, cs, vs = self.buffer()
        out = np.zeros((len(rp) - 1, self.cfg.d))
        for i in range(len(rp) - 1):
            out[i, cs[rp[i]:rp[i + 1]]] = vs[rp[i]:rp[i + 1]]
        return out

    def synchronize(self) -> None:
        _check(lib().sfdg_sketcher_synchronize(self._h))

    def reset(self, seed: int | None = None) -> None:
        """Back to the just-constructed state (optionally with a new seed); keeps allocations."""
        if seed is not None:
            self.cfg.seed = int(seed)
        _check(lib().sfdg_sketcher_reset(self._h, C.c_uint64(self.cfg.seed)))

    def merge_device(self, d_other_bt: int, ld: int) -> None:
        """B <- merge(B, other) with other's B^T (d x ell, leading dim ld) on this device."""
        _check(lib().sfdg_sketcher_merge_device(self._h, C.c_void_p(d_other_bt), ld))

    def finalize_device(self) -> None:
        """finalize() leaving B on the device (no host copy)."""
        _check(lib().sfdg_sketcher_finalize(self._h, None))


# ---- free functions ------------------------------------------------------------

def merge(b1, b2, ell: int, device: int = 0) -> np.ndarray:
    """merge(b1, b2, ell) = dense_shrink(vstack(b1, b2), ell) (sketch.cpp:80-83)."""
    b1, b2 = _f64(b1), _f64(b2)
    if b1.ndim != 2 or b2.ndim != 2 or b1.shape[1] != b2.shape[1]:
        raise InvalidArgument("merge: column mismatch")
    d = b1.shape[1]
    out = np.zeros((ell, d))
    _check(lib().sfdg_merge(_p(b1, _dp), b1.shape[0], _p(b2, _dp), b2.shape[0], d, ell, _p(out, _dp), device))
    return out


class FdSketcher:
    """FdSketcher (sketch.hpp:53-67): dense Frequent Directions on the device."""

    def __init__(self, ell: int, d: int, device: int = 0):
        self.ell, self.d = int(ell), int(d)
        self._h = C.c_void_p()
        _check(lib().sfdg_fd_create(self.ell, self.d, device, C.byref(self._h)))

    def append(self, row) -> None:
        self.append_rows(np.atleast_2d(row))

    def append_rows(self, rows) -> None:
        a = _f64(np.atleast_2d(rows))
        if a.shape[1] != self.d:
            raise InvalidArgument("FdSketcher: row dimension mismatch")
        _check(lib().sfdg_fd_append(self._h, _p(a, _dp), a.shape[0]))

    def append_csr(self, row_ptr, cols, vals) -> None:
        rp, cs, vs = _csr(row_ptr, cols, vals)
        _check(lib().sfdg_fd_append_csr(self._h, _p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1))

    def finalize(self) -> np.ndarray:
        out = np.zeros((self.ell, self.d))
        _check(lib().sfdg_fd_finalize(self._h, _p(out, _dp)))
        return out

    def shrink_count(self) -> int:
        c = C.c_size_t()
        _check(lib().sfdg_fd_shrink_count(self._h, C.byref(c)))
        return c.value

    def close(self) -> None:
        if self._h:
            lib().sfdg_fd_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sharded_sketch(row_ptr, cols, vals, cfg: "SketchConfig", shards: int, devices=(0,)):
    """sfdg_sharded_sketch: G contiguous row shards sketched with seed + g on
    devices[g % len(devices)], merged in the log2 tree (shards.py order). Returns
    (B ell x d, [per-shard stats dicts])."""
    rp, cs, vs = _csr(row_ptr, cols, vals)
    devs = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    out = np.zeros((cfg.ell, cfg.d))
    st = (_Stats * shards)()
    c = cfg._c()
    _check(lib().sfdg_sharded_sketch(C.byref(c), _p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1, shards,
                                     devs.ctypes.data_as(C.POINTER(C.c_int)), len(devs), _p(out, _dp), st))
    stats = [{"flushes": s.flush_count, "attempts": s.attempt_total, "verifier_i": s.verifier.i,
              "delta_spent": s.verifier.delta_spent} for s in st]
    return out, stats


def merge_device(d_b1t: int, d_b2t: int, ell: int, d: int, ld: int, d_outt: int, device: int = 0,
                 stream: int = 0) -> None:
    """Device merge of two B^T (d x ell, leading dim ld) into d_outt."""
    _check(lib().sfdg_merge_device(C.c_void_p(d_b1t), C.c_void_p(d_b2t), ell, d, ld, C.c_void_p(d_outt), device,
                                   C.c_void_p(stream) if stream else None))


def dense_shrink(a, ell: int, device: int = 0) -> np.ndarray:
    """dense_shrink(a, ell) (shrink.cpp:30-61)."""
    a = _f64(a)
    out = np.zeros((ell, a.shape[1]))
    _check(lib().sfdg_dense_shrink(_p(a, _dp), a.shape[0], a.shape[1], ell, _p(out, _dp), device))
    return out


def _rng_arg(rng) -> RngState:
    if isinstance(rng, RngState):
        return rng
    if hasattr(rng, "state") and hasattr(rng, "seed"):  # oracle Rng: adopt its draw position
        w, hs, sp = rng.state()
        return RngState(rng.seed, w, hs, sp)
    return RngState(int(rng))


def sparse_shrink(csr, d: int, ell: int, rng, power: PowerConfig | None = None, device: int = 0):
    """sparse_shrink(buffer, ell, power, rng) (shrink.cpp:63-73). Returns (B', RngState after)."""
    rp, cs, vs = _csr(*csr)
    st = _rng_arg(rng)
    c = st._c()
    pw = (power or PowerConfig())._c()
    out = np.zeros((ell, d))
    _check(lib().sfdg_sparse_shrink(_p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1, d, ell, C.byref(pw),
                                    C.byref(c), _p(out, _dp), device))
    st = RngState(st.seed)
    st._update(c)
    return out, st


def read_row_stream(path: str, plain_cols: int = 0):
    """open_row_stream (io.cpp:170-189) through the parallel reader: (row_ptr, cols, vals, d).
    Host-only (no GPU needed)."""
    n, d, z = C.c_size_t(), C.c_size_t(), C.c_size_t()
    _check(lib().sfdg_read_row_stream(path.encode(), plain_cols, C.byref(n), C.byref(d), C.byref(z), None, None,
                                      None))
    rp = np.zeros(n.value + 1, np.int64)
    cs = np.zeros(max(1, z.value), np.uint32)
    vs = np.zeros(max(1, z.value))
    _check(lib().sfdg_read_row_stream(path.encode(), plain_cols, C.byref(n), C.byref(d), C.byref(z), _p(rp, _i64p),
                                      _p(cs, _u32p), _p(vs, _dp)))
    return rp, cs[: z.value], vs[: z.value], d.value


def sketch_file(path: str, cfg: "SketchConfig", plain_cols: int = 0, device: int = 0):
    """sfdg_sketch_file: the reference's run_sketch over a file (tools/sfd_main.cpp:65-69).
    cfg.d = 0 takes the file's width. Returns (B, stats dict)."""
    d = C.c_size_t()
    # the sketch width is the file's; read the header first when cfg.d is 0
    width = cfg.d or read_row_stream_width(path, plain_cols)
    out = np.zeros((cfg.ell, width))
    st = _Stats()
    c = cfg._c()
    _check(lib().sfdg_sketch_file(path.encode(), plain_cols, C.byref(c), device, _p(out, _dp), C.byref(st),
                                  C.byref(d)))
    return out, {"flushes": st.flush_count, "attempts": st.attempt_total, "verifier_i": st.verifier.i,
                 "delta_spent": st.verifier.delta_spent}


def read_row_stream_width(path: str, plain_cols: int = 0) -> int:
    if plain_cols:
        return plain_cols
    with open(path) as f:
        for line in f:
            if line.startswith("%") or not line.strip():
                continue
            return int(line.split()[1])
    raise InvalidArgument(path + ": missing MatrixMarket size line")


def proj_err(csr, d: int, sketch, k: int, tail_sq: float, device: int = 0):
    """proj_err (bench.cpp:139-169) on the device: value or None (the reference's nullopt)."""
    rp, cs, vs = _csr(*csr)
    b = _f64(np.atleast_2d(sketch))
    out, has = C.c_double(), C.c_int()
    _check(lib().sfdg_proj_err(_p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1, d, _p(b, _dp), b.shape[0], k,
                               tail_sq, C.byref(out), C.byref(has), device))
    return out.value if has.value else None


def exact_tail(csr, d: int, k: int, rng, device: int = 0):
    """exact_tail(a, k, rng) (bench.cpp:68-137) on the device: (tail_sq, sigma[k], sweeps, RngState)."""
    rp, cs, vs = _csr(*csr)
    st = _rng_arg(rng)
    c = st._c()
    sig = np.zeros(max(1, k))
    tail = C.c_double()
    sw = C.c_size_t()
    _check(lib().sfdg_exact_tail(_p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1, d, k, C.byref(c),
                                 _p(sig, _dp), C.byref(tail), C.byref(sw), device))
    st = RngState(st.seed)
    st._update(c)
    return tail.value, sig[:k], sw.value, st


def cov_err(csr, d: int, sketch, rng, iterations: int = 1000, device: int = 0):
    """cov_err(a, sketch, rng, iterations) (bench.cpp:171-183): |A^T A - B^T B|_2 / |A|_F^2 over
    the whole CSR stream, on the device. Returns (value, RngState after)."""
    rp, cs, vs = _csr(*csr)
    b = _f64(np.atleast_2d(sketch))
    if b.shape[1] != d:
        raise InvalidArgument("cov_err: dimension mismatch")
    st = _rng_arg(rng)
    c = st._c()
    out = C.c_double()
    _check(lib().sfdg_cov_err(_p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1, d, _p(b, _dp), b.shape[0],
                              iterations, C.byref(c), C.byref(out), device))
    st = RngState(st.seed)
    st._update(c)
    return out.value, st


def boosted_sparse_shrink(csr, d: int, ell: int, state: VerifierState, rng, power: PowerConfig | None = None,
                          device: int = 0):
    """boosted_sparse_shrink (shrink.cpp:104-131). Returns (B', delta_hat, attempts, RngState after)."""
    rp, cs, vs = _csr(*csr)
    st = _rng_arg(rng)
    c = st._c()
    v = state._c()
    pw = (power or PowerConfig())._c()
    out = np.zeros((ell, d))
    dh = C.c_double()
    att = C.c_size_t()
    _check(lib().sfdg_boosted_sparse_shrink(_p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), len(rp) - 1, d, ell,
                                            C.byref(v), C.byref(pw), C.byref(c), _p(out, _dp), C.byref(dh),
                                            C.byref(att), device))
    state._update(v)
    st = RngState(st.seed)
    st._update(c)
    return out, dh.value, att.value, st


_SYMOP = C.CFUNCTYPE(C.c_int, _dp, _dp, C.c_size_t, C.c_void_p)


def verify_spectral(op, d: int, state: VerifierState, rng, device: int = 0, on_device: bool = False) -> tuple:
    """verify_spectral(apply, d, state, rng) (shrink.hpp:35, shrink.cpp:75-102) over a caller
    operator. op(x) -> y: numpy arrays (on_device=False), or op(x_ptr, y_ptr, d) on raw device
    pointers of `device` (on_device=True). Returns (accepted, RngState after); state updated."""
    err = []

    def _cb(xp, yp, n, _ctx):
        try:
            if on_device:
                op(C.cast(xp, C.c_void_p).value, C.cast(yp, C.c_void_p).value, n)
            else:
                x = np.ctypeslib.as_array(xp, shape=(n,)).copy()
                y = np.asarray(op(x), dtype=np.float64)
                if y.shape != (n,):
                    raise ValueError("verify_spectral: operator output has the wrong shape")
                np.ctypeslib.as_array(yp, shape=(n,))[:] = y
            return 0
        except Exception as e:  # reported after the call
            err.append(e)
            return 1

    cb = _SYMOP(_cb)
    st = _rng_arg(rng)
    c = st._c()
    v = state._c()
    acc = C.c_int()
    L = lib()
    L.sfdg_verify_spectral.argtypes = [_SYMOP, C.c_void_p, C.c_int, C.c_size_t, C.POINTER(_Verifier),
                                       C.POINTER(_Rng), C.POINTER(C.c_int), C.c_int]
    code = L.sfdg_verify_spectral(cb, None, 1 if on_device else 0, d, C.byref(v), C.byref(c), C.byref(acc), device)
    if err:
        raise err[0]
    _check(code)
    state._update(v)
    st = RngState(st.seed)
    st._update(c)
    return bool(acc.value), st


def simultaneous_iteration(csr, d: int, k: int, rng, power: PowerConfig | None = None, device: int = 0):
    """simultaneous_iteration (randsvd.cpp:18-51). Returns (Z m x k, RngState after)."""
    rp, cs, vs = _csr(*csr)
    st = _rng_arg(rng)
    c = st._c()
    pw = (power or PowerConfig())._c()
    m = len(rp) - 1
    out = np.zeros((m, k))
    _check(lib().sfdg_simultaneous_iteration(_p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), m, d, k, C.byref(pw),
                                             C.byref(c), _p(out, _dp), device))
    st = RngState(st.seed)
    st._update(c)
    return out, st


def power_iteration_count(m: int, power: PowerConfig | None = None) -> int:
    pw = (power or PowerConfig())._c()
    q = C.c_size_t()
    _check(lib().sfdg_power_iteration_count(m, C.byref(pw), C.byref(q)))
    return q.value


def gaussian_matrix(rows: int, cols: int, rng, device: int = 0):
    """gaussian_matrix (la_core.cpp:167-172) on the device. Returns (G, RngState after)."""
    st = _rng_arg(rng)
    c = st._c()
    out = np.zeros((rows, cols))
    _check(lib().sfdg_gaussian_matrix(C.byref(c), rows, cols, _p(out, _dp), device))
    st = RngState(st.seed)
    st._update(c)
    return out, st


def eigh(sym, off_tol: float, device: int = 0):
    """jacobi_eigh contract (la_core.cpp:24-80): (values desc, vectors columns)."""
    s = _f64(sym)
    n = s.shape[0]
    vals, vecs = np.zeros(n), np.zeros((n, n))
    _check(lib().sfdg_eigh(_p(s, _dp), n, off_tol, _p(vals, _dp), _p(vecs, _dp), device))
    return vals, vecs


def orthonormalize(a, device: int = 0) -> np.ndarray:
    """orthonormalize contract (la_core.cpp:130-165) via device CholeskyQR2."""
    a = _f64(a)
    out = np.zeros_like(a)
    _check(lib().sfdg_orthonormalize(_p(a, _dp), a.shape[0], a.shape[1], _p(out, _dp), device))
    return out


def csr_products(csr, d: int, x=None, z=None, device: int = 0):
    """(A x, A^T z) for panels x (d x k) and z (m x k) (sparse.cpp:32-69)."""
    rp, cs, vs = _csr(*csr)
    m = len(rp) - 1
    k = (x if x is not None else z).shape[1]
    y = np.zeros((m, k)) if x is not None else None
    w = np.zeros((d, k)) if z is not None else None
    xx = _f64(x) if x is not None else None
    zz = _f64(z) if z is not None else None
    _check(lib().sfdg_csr_products(_p(rp, _i64p), _p(cs, _u32p), _p(vs, _dp), m, d, k,
                                   _p(xx, _dp) if xx is not None else None, _p(y, _dp) if y is not None else None,
                                   _p(zz, _dp) if zz is not None else None, _p(w, _dp) if w is not None else None,
                                   device))
    return y, w
