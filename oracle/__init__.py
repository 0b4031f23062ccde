"""CPU oracle for the reduced QMC matrix product -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may import this.
The product path (paper_2305_11645_b200) never imports it and shares no code with it.

Thin ctypes wrapper over oracle/rqmc_oracle.c (plain C, fp64, -ffp-contract=off), which computes
the plain definitions of PAPER.md (P:n = line n):
  points  x_{k,j} = {k z_j / N} + shift / digital net / reduced MC
          (Eq. randpts) + Phi^-1 map
  product Y = X A, naive triple loop in increasing j
  Q_N     N^-1 sum_k f(x_k^T A) with Neumaier summation
Every function is pinned by tests/test_oracle_pins.py.
f = MEAN_SQ (C4) is pinned by an exact-rational brute force of Q_N, f = CALL_MEAN_EXP (C2) by a
40-digit mpmath evaluation of the definition on exact rational points (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rqmc_oracle.c")
_LIB = os.path.join(_HERE, "librqmc_oracle.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


class _Prob(C.Structure):
    _fields_ = [("b", C.c_int), ("m", C.c_int), ("s", C.c_int),
                ("w", C.POINTER(C.c_int32)), ("kind", C.c_int),
                ("z", C.POINTER(C.c_uint64)), ("C", C.POINTER(C.c_uint64)),
                ("shift", C.POINTER(C.c_double)), ("dshift", C.POINTER(C.c_uint64)),
                ("map", C.c_int), ("seed", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp, u64p, i64p = C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.POINTER(C.c_int64)
        _lib.orc_invnorm.restype = C.c_double
        _lib.orc_invnorm.argtypes = [C.c_double]
        _lib.orc_tent.restype = C.c_double
        _lib.orc_tent.argtypes = [C.c_double]
        _lib.orc_points.argtypes = [C.POINTER(_Prob), C.c_int64, C.c_int64, dp, u64p]
        _lib.orc_product.argtypes = [C.c_int64, C.c_int, C.c_int, dp, dp, dp]
        _lib.orc_f.argtypes = [C.c_int64, C.c_int, dp, C.c_int, dp, dp]
        _lib.orc_neumaier.restype = C.c_double
        _lib.orc_neumaier.argtypes = [dp, C.c_int64]
        _lib.orc_f_rows.argtypes = [C.POINTER(_Prob), dp, C.c_int, C.c_int, dp, i64p, C.c_int64, dp, dp, C.c_int]
        _lib.orc_f_rows_meanid.argtypes = [C.POINTER(_Prob), dp, C.c_int, C.c_int, i64p, C.c_int64, dp, C.c_int]
        _lib.orc_points_rows.argtypes = [C.POINTER(_Prob), i64p, C.c_int64, dp, C.c_int]
        _lib.orc_f_all_meanid_tab.argtypes = [C.POINTER(_Prob), dp, C.c_int, C.c_int, dp, C.c_int]
        _lib.orc_f_all_tab.argtypes = [C.POINTER(_Prob), dp, C.c_int, C.c_int, dp, dp, C.c_int]
        _lib.orc_alg4_product.argtypes = [C.POINTER(_Prob), dp, C.c_int, dp]
        _lib.orc_mc_bank_index.restype = C.c_uint64
        _lib.orc_mc_bank_index.argtypes = [C.POINTER(_Prob), C.c_uint64, C.c_int]
        _lib.orc_mc_bank_indices.argtypes = [C.POINTER(_Prob), C.c_uint64, u64p]
        _lib.orc_mc_word.restype = C.c_uint64
        _lib.orc_mc_word.argtypes = [C.c_uint64, C.c_int, C.c_uint64]
        _lib.orc_mc_points_bank.argtypes = [C.POINTER(_Prob), dp, i64p, C.c_int64, C.c_int64, dp]
    return _lib


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


class _Holder:
    """Keeps numpy arrays alive while the C struct points at them."""

    def __init__(self, prob):
        self.w = np.ascontiguousarray(prob.w, dtype=np.int32)
        self.z = None if prob.z is None else np.ascontiguousarray(prob.z, dtype=np.uint64)
        self.Cm = None if prob.C is None else np.ascontiguousarray(prob.C, dtype=np.uint64)
        self.sh = None if prob.shift is None else np.ascontiguousarray(prob.shift, dtype=np.float64)
        self.ds = None if prob.dshift is None else np.ascontiguousarray(prob.dshift, dtype=np.uint64)
        self.s = _Prob(prob.b, prob.m, prob.s, _ptr(self.w, C.c_int32), prob.kind,
                       _ptr(self.z, C.c_uint64), _ptr(self.Cm, C.c_uint64),
                       _ptr(self.sh, C.c_double), _ptr(self.ds, C.c_uint64), prob.map,
                       int(getattr(prob, "mc_seed", 0)))


def mc_bank_index(prob, n: int, j: int) -> int:
    """Reduced MC (Eq. randpts): bank sample number used by coordinate j (0-based) of point n."""
    h = _Holder(prob)
    return int(lib().orc_mc_bank_index(C.byref(h.s), n, j))


def mc_bank_indices(prob, n: int) -> np.ndarray:
    """Reduced MC (Eq. randpts): the bank sample numbers of every coordinate of point n, one digit pass."""
    h = _Holder(prob)
    out = np.empty(prob.s, dtype=np.uint64)
    lib().orc_mc_bank_indices(C.byref(h.s), n, _ptr(out, C.c_uint64))
    return out


def mc_word(seed: int, j: int, r: int) -> int:
    """The counter-based draw y_{j,r} as its 53-bit word (u = (word | 1) 2^-53)."""
    return int(lib().orc_mc_word(seed, j, r))


def mc_points_bank(prob, bank_cols, k0: int = 0, n: int | None = None) -> np.ndarray:
    """Sample matrix of Eq. randpts from explicit banks: bank_cols[j] holds N_j values of coordinate j."""
    n = prob.N - k0 if n is None else n
    h = _Holder(prob)
    off = np.zeros(prob.s, dtype=np.int64)
    off[1:] = np.cumsum([len(c) for c in bank_cols])[:-1]
    bank = np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.float64) for c in bank_cols]))
    X = np.empty((n, prob.s), dtype=np.float64)
    lib().orc_mc_points_bank(C.byref(h.s), _ptr(bank, C.c_double), _ptr(off, C.c_int64), k0, n, _ptr(X, C.c_double))
    return X


def tent(u: float) -> float:
    """phi(u) = 1 - |1 - 2u|, the oracle's C evaluation."""
    return lib().orc_tent(float(u))


def invnorm(u: float) -> float:
    return lib().orc_invnorm(float(u))


def points(prob, k0: int = 0, n: int | None = None):
    """(X, T): rows k0..k0+n of the point matrix X and the integer word of each entry."""
    n = prob.N - k0 if n is None else n
    h = _Holder(prob)
    X = np.empty((n, prob.s), dtype=np.float64)
    T = np.empty((n, prob.s), dtype=np.uint64)
    lib().orc_points(C.byref(h.s), k0, n, _ptr(X, C.c_double), _ptr(T, C.c_uint64))
    return X, T


def points_rows(prob, ks, nthreads: int = 0) -> np.ndarray:
    """Rows ks (any order) of the point matrix X."""
    h = _Holder(prob)
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.int64))
    X = np.empty((len(ks), prob.s), dtype=np.float64)
    lib().orc_points_rows(C.byref(h.s), _ptr(ks, C.c_int64), len(ks), _ptr(X, C.c_double), nthreads)
    return X


def product(X: np.ndarray, A: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float64)
    A = np.ascontiguousarray(A, dtype=np.float64)
    n, s = X.shape
    tau = A.shape[1]
    Y = np.empty((n, tau), dtype=np.float64)
    lib().orc_product(n, s, tau, _ptr(X, C.c_double), _ptr(A, C.c_double), _ptr(Y, C.c_double))
    return Y


def f_of_y(Y: np.ndarray, f: int, fparam) -> np.ndarray:
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    fp = np.ascontiguousarray(np.asarray(fparam, dtype=np.float64).reshape(-1)[:2].copy() if fparam is not None else np.zeros(2))
    fk = np.empty(Y.shape[0])
    lib().orc_f(Y.shape[0], Y.shape[1], _ptr(Y, C.c_double), f, _ptr(fp, C.c_double), _ptr(fk, C.c_double))
    return fk


def neumaier(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return lib().orc_neumaier(_ptr(v, C.c_double), len(v))


def f_rows(prob, ks, with_y: bool = False, nthreads: int = 0, f: int | None = None):
    """f_k (and optionally Y rows) for the given global row indices k, via O1+O2+O3."""
    h = _Holder(prob)
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.int64))
    A = np.ascontiguousarray(prob.A, dtype=np.float64)
    fp = np.ascontiguousarray(np.asarray(prob.fparam, dtype=np.float64))
    fk = np.empty(len(ks))
    Y = np.empty((len(ks), prob.tau)) if with_y else None
    ff = prob.f if f is None else f
    err = lib().orc_f_rows(C.byref(h.s), _ptr(A, C.c_double), prob.tau, ff, _ptr(fp, C.c_double),
                           _ptr(ks, C.c_int64), len(ks), _ptr(fk, C.c_double), _ptr(Y, C.c_double), nthreads)
    if err:
        raise MemoryError("oracle f_rows allocation failed")
    return (fk, Y) if with_y else fk


def f_rows_meanid(prob, ks, nthreads: int = 0):
    """O3' mean identity (g = id only): f_k = F(x_k . abar), abar = tau^-1 A 1."""
    h = _Holder(prob)
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.int64))
    A = np.ascontiguousarray(prob.A, dtype=np.float64)
    fk = np.empty(len(ks))
    if lib().orc_f_rows_meanid(C.byref(h.s), _ptr(A, C.c_double), prob.tau, prob.f,
                               _ptr(ks, C.c_int64), len(ks), _ptr(fk, C.c_double), nthreads):
        raise ValueError("mean identity needs g = id (f in {EXP_MEAN, MEAN})")
    return fk


def f_all_meanid_tab(prob, nthreads: int = 0) -> np.ndarray:
    """O3' over all N rows with column tabulation (g = id only); returns f_k for k = 0..N-1."""
    h = _Holder(prob)
    A = np.ascontiguousarray(prob.A, dtype=np.float64)
    fk = np.empty(prob.N)
    err = lib().orc_f_all_meanid_tab(C.byref(h.s), _ptr(A, C.c_double), prob.tau, prob.f, _ptr(fk, C.c_double), nthreads)
    if err:
        raise ValueError({1: "mean identity needs g = id", 3: "row-zeroed nets are not periodic"}.get(
            err, "allocation failed"))
    return fk


def f_all_tab(prob, f: int | None = None, nthreads: int = 0) -> np.ndarray:
    """f_k for k = 0..N-1 by O1+O2+O3 with column tabulation and row/column cache blocking (same
    arithmetic order per entry as f_rows; any f; periodic kinds only)."""
    h = _Holder(prob)
    A = np.ascontiguousarray(prob.A, dtype=np.float64)
    fp = np.ascontiguousarray(np.asarray(prob.fparam, dtype=np.float64))
    fk = np.empty(prob.N)
    err = lib().orc_f_all_tab(C.byref(h.s), _ptr(A, C.c_double), prob.tau, prob.f if f is None else f,
                              _ptr(fp, C.c_double), _ptr(fk, C.c_double), nthreads)
    if err:
        raise ValueError({1: "row-zeroed nets are not periodic"}.get(err, "allocation failed"))
    return fk


def alg4_xa(prob) -> np.ndarray:
    """All N rows of XA by the paper's Alg. 4 for an unshifted, unmapped row-zeroed net
    (kind 3): a second product path, from the FULL net and the table c_k = (k/b^{m-w_j}) a_j."""
    h = _Holder(prob)
    A = np.ascontiguousarray(prob.A, dtype=np.float64)
    Y = np.empty((prob.N, prob.tau))
    err = lib().orc_alg4_product(C.byref(h.s), _ptr(A, C.c_double), prob.tau, _ptr(Y, C.c_double))
    if err:
        raise ValueError("Alg. 4 needs an unshifted, unmapped row-zeroed net (kind 3)" if err == 1
                         else "allocation failed")
    return Y


def xa(prob, k0: int = 0, n: int | None = None) -> np.ndarray:
    """Y rows k0..k0+n of XA by the naive definition."""
    X, _ = points(prob, k0, n)
    return product(X, prob.A)


def qn_sum(prob, ks=None, nthreads: int = 0) -> float:
    """sum_k f(x_k^T A) over rows ks (default all N), Neumaier in increasing k (times N)."""
    ks = np.arange(prob.N, dtype=np.int64) if ks is None else ks
    return neumaier(f_rows(prob, ks, nthreads=nthreads))
