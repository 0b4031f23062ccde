"""B200-native reduced QMC matrix product (Dick, Ebert, Herrmann, Kritzer, Longo; arXiv 2305.11645).

Thin Python binding over the C ABI in include/rqmc.h (librqmc.so, built in-tree for sm_100a).
Argument marshalling only: every step of the path (points, per-level GEMMs, tile-accumulate, f and
its reduction) runs in the library's CUDA kernels.  PyTorch provides device memory, streams and
torch.distributed (the one all-reduce of the local f-sums across ranks).

    plan = Plan(b=2, m=24, s=4096, tau=2048, w=w, z=z, shift=delta, map=MAP_INVNORM)
    Y = plan.xa(A)                          # N x tau, Y = X A
    q = plan.qn(A, F_EXP_MEAN)              # Q_N = N^-1 sum_k f(x_k^T A)

There is no CPU fallback: if librqmc.so is missing or CUDA is unavailable the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from ._build import LIB as _LIB_PATH

# A/B experiments only: RQMC_LIB may name another in-tree build (librqmc_<variant>.so)
_LIB_PATH = os.environ.get("RQMC_LIB", _LIB_PATH)

LATTICE, DIGITAL_NET, REDUCED_MC, DIGITAL_NET_ROWS = 0, 1, 2, 3
MAP_UNIT, MAP_INVNORM, MAP_TENT = 0, 1, 2
F_NONE, F_EXP_MEAN, F_CALL_MEAN_EXP, F_MEAN_SQ, F_MEAN = -1, 0, 1, 2, 3

STATUS = {0: "OK", 1: "EINVAL", 2: "ENOTPRIME", 3: "EWORDER", 4: "EZUNIT", 5: "ESHIFT", 6: "ENETMAT",
          7: "EDIM", 8: "EDOMAIN", 9: "ECUDA", 10: "ENOMEM", 11: "EUNSUPPORTED"}


class RqmcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class _Desc(C.Structure):
    _fields_ = [("b", C.c_int), ("m", C.c_int), ("s", C.c_int), ("tau", C.c_int),
                ("w", C.POINTER(C.c_int32)), ("kind", C.c_int),
                ("z", C.POINTER(C.c_uint64)), ("C", C.POINTER(C.c_uint64)),
                ("shift", C.POINTER(C.c_double)), ("dshift", C.POINTER(C.c_uint64)),
                ("map", C.c_int), ("rank", C.c_int), ("world", C.c_int), ("seed", C.c_uint64)]


class LevelInfo(C.Structure):
    _fields_ = [("w", C.c_int), ("j_lo", C.c_int), ("s_w", C.c_int), ("M", C.c_int64),
                ("M_local", C.c_int64), ("parent", C.c_int), ("coarse", C.c_int), ("fft", C.c_int),
                ("absorbed", C.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Summary(C.Structure):
    _fields_ = [("n_levels", C.c_int), ("checkpoint", C.c_int), ("n_fine", C.c_int),
                ("n_bundles", C.c_int64), ("N_local", C.c_int64), ("s_star", C.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["rqmc_plan_create", "rqmc_plan_destroy", "rqmc_strerror", "rqmc_plan_last_error",
           "rqmc_plan_summary_get", "rqmc_plan_level", "rqmc_plan_global_row", "rqmc_plan_stats",
           "rqmc_workspace_size", "rqmc_xa", "rqmc_qn", "rqmc_qn_host", "rqmc_xa_host", "rqmc_points",
           "rqmc_profile_enable", "rqmc_profile_read", "rqmc_workspace_size_batch", "rqmc_qn_batch",
           "rqmc_plan_summary_batch", "rqmc_plan_dispatch", "rqmc_plan_partition"]

_lib = None


def lib():
    """Load librqmc.so (fails loudly if it has not been built: python -m paper_2305_11645_b200._build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python paper_2305_11645_b200/_build.py` "
                               "(or __graft_entry__.build()); there is no fallback path")
        L = C.CDLL(_LIB_PATH)
        vp, dp, i64 = C.c_void_p, C.POINTER(C.c_double), C.c_int64
        L.rqmc_plan_create.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
        L.rqmc_plan_destroy.argtypes = [vp]
        L.rqmc_plan_destroy.restype = None
        L.rqmc_strerror.restype = C.c_char_p
        L.rqmc_plan_last_error.argtypes = [vp]
        L.rqmc_plan_last_error.restype = C.c_char_p
        L.rqmc_plan_summary_get.argtypes = [vp, C.POINTER(Summary)]
        L.rqmc_plan_level.argtypes = [vp, C.c_int, C.POINTER(LevelInfo)]
        L.rqmc_plan_global_row.argtypes = [vp, i64]
        L.rqmc_plan_global_row.restype = i64
        L.rqmc_plan_stats.argtypes = [vp, C.c_int, C.POINTER(i64), dp, dp]
        L.rqmc_workspace_size.argtypes = [vp, C.POINTER(C.c_size_t)]
        L.rqmc_xa.argtypes = [vp, vp, i64, vp, i64, C.c_int, dp, vp, vp, C.c_size_t, vp]
        L.rqmc_qn.argtypes = [vp, vp, i64, C.c_int, dp, vp, vp, C.c_size_t, vp]
        L.rqmc_qn_host.argtypes = [vp, dp, i64, C.c_int, dp, dp, vp, C.c_size_t, vp]
        L.rqmc_xa_host.argtypes = [vp, dp, i64, vp, i64, C.c_int, dp, dp, vp, C.c_size_t, vp]
        L.rqmc_points.argtypes = [vp, C.c_int, i64, i64, vp, vp, vp]
        L.rqmc_profile_enable.argtypes = [vp, C.c_int]
        L.rqmc_workspace_size_batch.argtypes = [vp, C.c_int, C.POINTER(C.c_size_t)]
        L.rqmc_plan_summary_batch.argtypes = [vp, C.c_int, C.c_int, C.POINTER(Summary)]
        L.rqmc_qn_batch.argtypes = [vp, C.c_int, dp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), vp, i64,
                                    C.c_int, dp, vp, vp, C.c_size_t, vp]
        L.rqmc_plan_dispatch.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.rqmc_plan_partition.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
        L.rqmc_profile_read.argtypes = [vp, C.POINTER(C.c_int), dp, dp, dp, dp]
        _lib = L
    return _lib


def _arr(x, dt):
    return None if x is None else np.ascontiguousarray(np.asarray(x, dtype=dt))


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def _stream_ptr(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


class Plan:
    """rqmc_plan_t: immutable description of one reduced point set (+ shift/map) and A's shape."""

    def __init__(self, b: int, m: int, s: int, tau: int, w: Sequence[int], kind: int = LATTICE,
                 z=None, C_words=None, shift=None, dshift=None, map: int = MAP_UNIT,
                 rank: int = 0, world: int = 1, seed: int = 0):
        self._keep = dict(w=_arr(w, np.int32), z=_arr(z, np.uint64), C=_arr(C_words, np.uint64),
                          shift=_arr(shift, np.float64), dshift=_arr(dshift, np.uint64))
        k = self._keep
        d = _Desc(b, m, s, tau, _p(k["w"], C.c_int32), kind, _p(k["z"], C.c_uint64), _p(k["C"], C.c_uint64),
                  _p(k["shift"], C.c_double), _p(k["dshift"], C.c_uint64), map, rank, world, seed)
        h = C.c_void_p()
        st = lib().rqmc_plan_create(C.byref(d), C.byref(h))
        if st != 0:
            raise RqmcError(st, lib().rqmc_plan_last_error(None).decode())
        self._h = h
        self.b, self.m, self.s, self.tau, self.rank, self.world = b, m, s, tau, rank, world
        self.N = b ** m
        self._ws = None

    @classmethod
    def from_problem(cls, prob, rank: int = 0, world: int = 1) -> "Plan":
        return cls(prob.b, prob.m, prob.s, prob.tau, prob.w, prob.kind, prob.z, prob.C, prob.shift,
                   prob.dshift, prob.map, rank, world, getattr(prob, "mc_seed", 0))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.rqmc_plan_destroy(h)
            self._h = None

    def _check(self, st):
        if st != 0:
            raise RqmcError(st, lib().rqmc_plan_last_error(self._h).decode())

    # ---- inspection (host only, no GPU needed)
    def summary(self) -> dict:
        s = Summary()
        self._check(lib().rqmc_plan_summary_get(self._h, C.byref(s)))
        return s.as_dict()

    def levels(self) -> list:
        out = []
        for i in range(self.summary()["n_levels"]):
            li = LevelInfo()
            self._check(lib().rqmc_plan_level(self._h, i, C.byref(li)))
            out.append(li.as_dict())
        return out

    def dispatch(self, f: int = F_MEAN, want_y: bool = False, R: int = 1) -> str:
        """Name of the fused fine-level kernel template a run with these arguments launches (host only)."""
        buf = C.create_string_buffer(96)
        self._check(lib().rqmc_plan_dispatch(self._h, R, f, int(want_y), buf, len(buf)))
        return buf.value.decode()

    def partition(self) -> dict:
        """Residue classes of this rank: {"classes": ncls, "first": c0, "count": nc}; local row i is
        global point c0 + (i mod nc) + ncls (i div nc)."""
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(lib().rqmc_plan_partition(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"classes": a.value, "first": b.value, "count": c.value}

    def global_rows(self):
        """Global point indices k of this rank's local rows (numpy int64, N_local entries)."""
        pt = self.partition()
        i = np.arange(self.summary()["N_local"], dtype=np.int64)
        return pt["first"] + i % pt["count"] + pt["classes"] * (i // pt["count"])

    def global_row(self, i: int) -> int:
        return lib().rqmc_plan_global_row(self._h, i)

    def stats(self, want_y: bool = False) -> dict:
        rows, macs, byt = C.c_int64(), C.c_double(), C.c_double()
        self._check(lib().rqmc_plan_stats(self._h, int(want_y), C.byref(rows), C.byref(macs), C.byref(byt)))
        return {"local_rows": rows.value, "macs": macs.value, "min_bytes": byt.value}

    def workspace_size(self) -> int:
        n = C.c_size_t()
        self._check(lib().rqmc_workspace_size(self._h, C.byref(n)))
        return n.value

    # ---- device runs
    def workspace(self, device=None):
        import torch
        dev = torch.device("cuda") if device is None else torch.device(device)
        need = self.workspace_size()
        if self._ws is None or self._ws.device != dev or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=dev)
        return self._ws

    @staticmethod
    def _check_A(A, s, tau):
        import torch
        if not (isinstance(A, torch.Tensor) and A.is_cuda and A.dtype == torch.float64):
            raise TypeError("A must be a CUDA float64 tensor")
        if A.dim() != 2 or A.shape[0] != s or A.shape[1] != tau or A.stride(1) != 1:
            raise ValueError(f"A must be {s} x {tau} with unit column stride")

    def xa(self, A, f: int = F_NONE, fparam=None, Y=None, fsum=None, stream=None):
        """Y = X A on this rank's rows; with f, also returns the local sum of f (device tensor)."""
        import torch
        self._check_A(A, self.s, self.tau)
        nl = self.summary()["N_local"]
        if Y is None:
            Y = torch.empty((nl, self.tau), dtype=torch.float64, device=A.device)
        if fsum is None and f != F_NONE:
            fsum = torch.empty(1, dtype=torch.float64, device=A.device)
        ws = self.workspace(A.device)
        fp = _arr(fparam if fparam is not None else [0.0, 0.0], np.float64)
        self._check(lib().rqmc_xa(self._h, C.c_void_p(A.data_ptr()), A.stride(0), C.c_void_p(Y.data_ptr()),
                                  Y.stride(0), f, _p(fp, C.c_double),
                                  C.c_void_p(fsum.data_ptr()) if fsum is not None else None,
                                  C.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream)))
        return (Y, fsum) if f != F_NONE else Y

    def qn_sum(self, A, f: int, fparam=None, out=None, stream=None):
        """Local sum over this rank's rows of f(x_k^T A), as a 1-element device tensor."""
        import torch
        self._check_A(A, self.s, self.tau)
        out = torch.empty(1, dtype=torch.float64, device=A.device) if out is None else out
        ws = self.workspace(A.device)
        fp = _arr(fparam if fparam is not None else [0.0, 0.0], np.float64)
        self._check(lib().rqmc_qn(self._h, C.c_void_p(A.data_ptr()), A.stride(0), f, _p(fp, C.c_double),
                                  C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(),
                                  _stream_ptr(stream)))
        return out

    def qn(self, A, f: int, fparam=None, group=None) -> float:
        """Q_N = N^-1 sum_k f(x_k^T A); with world > 1 the local sums meet in one all_reduce."""
        part = self.qn_sum(A, f, fparam)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(part, group=group)
        return float(part.item()) / self.N

    def summary_batch(self, R: int, f: int = F_MEAN) -> dict:
        """Summary of the layout a batch of R replicas with integrand f runs with (checkpoint may differ
        from summary())."""
        o = Summary()
        self._check(lib().rqmc_plan_summary_batch(self._h, R, f, C.byref(o)))
        return o.as_dict()

    def workspace_size_batch(self, R: int) -> int:
        n = C.c_size_t()
        self._check(lib().rqmc_workspace_size_batch(self._h, R, C.byref(n)))
        return n.value

    def qn_batch(self, A, f: int, fparam=None, shifts=None, dshifts=None, seeds=None, out=None,
                 max_workspace_bytes: Optional[int] = None, stream=None):
        """Batched randomisation (rqmc_qn_batch): local f-sums for R shifts (lattice: R x s array),
        digital shifts (net: R x s words) or seeds (reduced MC: R); returns an R-element device tensor."""
        import torch
        self._check_A(A, self.s, self.tau)
        src = shifts if shifts is not None else (dshifts if dshifts is not None else seeds)
        if src is None:
            raise ValueError("qn_batch needs shifts, dshifts or seeds")
        R = len(src)
        sh = None if shifts is None else _arr(np.asarray(shifts, dtype=np.float64).reshape(R, self.s), np.float64)
        ds = None if dshifts is None else _arr(np.asarray(dshifts, dtype=np.uint64).reshape(R, self.s), np.uint64)
        sd = None if seeds is None else _arr(np.asarray(seeds, dtype=np.uint64).reshape(R), np.uint64)
        need = self.workspace_size_batch(R)
        if max_workspace_bytes is not None:
            need = max(min(need, max_workspace_bytes), self.workspace_size_batch(1))
        if self._ws is None or self._ws.device != A.device or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=A.device)
        ws = self._ws
        out = torch.empty(R, dtype=torch.float64, device=A.device) if out is None else out
        fp = _arr(fparam if fparam is not None else [0.0, 0.0], np.float64)
        self._check(lib().rqmc_qn_batch(self._h, R, _p(sh, C.c_double), _p(ds, C.c_uint64), _p(sd, C.c_uint64),
                                        C.c_void_p(A.data_ptr()), A.stride(0), f, _p(fp, C.c_double),
                                        C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()),
                                        min(ws.numel(), need), _stream_ptr(stream)))
        return out

    def rqmc_estimate(self, A, f: int, fparam=None, shifts=None, dshifts=None, seeds=None, group=None):
        """(Q_N mean over the R randomisations, standard error, per-replica Q_N) -- torch.distributed
        aware like qn(): the per-replica local sums are all-reduced over `group` when initialised."""
        import torch
        sums = self.qn_batch(A, f, fparam, shifts=shifts, dshifts=dshifts, seeds=seeds)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(sums, group=group)
        q = (sums / self.N).cpu().numpy()
        R = len(q)
        se = float(np.std(q, ddof=1) / np.sqrt(R)) if R > 1 else float("nan")
        return float(np.mean(q)), se, q

    def qn_host(self, A_host: np.ndarray, f: int, fparam=None, device=None, stream=None) -> float:
        """End-to-end: host A in, host local f-sum out (H2D and D2H inside the C call)."""
        A_host = np.asarray(A_host)
        if A_host.dtype != np.float64 or A_host.shape != (self.s, self.tau) or not A_host.flags.c_contiguous:
            raise ValueError("A_host must be a C-contiguous float64 s x tau array")
        ws = self.workspace(device)
        fp = _arr(fparam if fparam is not None else [0.0, 0.0], np.float64)
        out = C.c_double()
        self._check(lib().rqmc_qn_host(self._h, A_host.ctypes.data_as(C.POINTER(C.c_double)), self.tau, f,
                                       _p(fp, C.c_double), C.byref(out), C.c_void_p(ws.data_ptr()),
                                       ws.numel(), _stream_ptr(stream)))
        return out.value

    def xa_host(self, A_host: np.ndarray, Y, f: int = F_NONE, fparam=None, stream=None):
        """End-to-end XA: host A in (H2D inside the C call, overlapped with the run), Y = X A into the
        device tensor Y (N_local x tau, unit column stride); with f, returns the local f-sum (host float)."""
        import torch
        A_host = np.asarray(A_host)
        if A_host.dtype != np.float64 or A_host.shape != (self.s, self.tau) or not A_host.flags.c_contiguous:
            raise ValueError("A_host must be a C-contiguous float64 s x tau array")
        nl = self.summary()["N_local"]
        if not (isinstance(Y, torch.Tensor) and Y.is_cuda and Y.dtype == torch.float64 and Y.dim() == 2
                and Y.shape[0] == nl and Y.shape[1] == self.tau and Y.stride(1) == 1):
            raise ValueError(f"Y must be a CUDA float64 {nl} x {self.tau} tensor with unit column stride")
        ws = self.workspace(Y.device)
        fp = _arr(fparam if fparam is not None else [0.0, 0.0], np.float64)
        out = C.c_double()
        self._check(lib().rqmc_xa_host(self._h, A_host.ctypes.data_as(C.POINTER(C.c_double)), self.tau,
                                       C.c_void_p(Y.data_ptr()), Y.stride(0), f, _p(fp, C.c_double),
                                       C.byref(out) if f != F_NONE else None, C.c_void_p(ws.data_ptr()),
                                       ws.numel(), _stream_ptr(stream)))
        return out.value if f != F_NONE else None

    def points(self, level_idx: int, r0: int = 0, count: Optional[int] = None):
        """Reduced points of one level: (integer words, fp64 values), each count x s_w."""
        import torch
        lv = self.levels()[level_idx]
        count = lv["M_local"] - r0 if count is None else count
        words = torch.empty((count, lv["s_w"]), dtype=torch.int64, device="cuda")
        vals = torch.empty((count, lv["s_w"]), dtype=torch.float64, device="cuda")
        self._check(lib().rqmc_points(self._h, level_idx, r0, count, C.c_void_p(words.data_ptr()),
                                      C.c_void_p(vals.data_ptr()), _stream_ptr()))
        return words, vals

    # ---- device-side phase timing (CUDA events recorded by the library on the run's stream)
    def profile_enable(self, max_runs: int):
        self._check(lib().rqmc_profile_enable(self._h, max_runs))

    def profile_read(self) -> dict:
        n = C.c_int()
        v = [C.c_double() for _ in range(4)]
        self._check(lib().rqmc_profile_read(self._h, C.byref(n), *[C.byref(x) for x in v]))
        return {"runs": n.value, "gen_ms": v[0].value, "coarse_ms": v[1].value, "fine_ms": v[2].value,
                "reduce_ms": v[3].value}

