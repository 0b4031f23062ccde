"""Seeded synthetic inputs for the reduced QMC matrix product (shared by oracle, CUDA path, bench).

This module holds NO arithmetic of the method: it only draws the *inputs* of the
paper's problem statement (Alg. 1 input line; Alg. 2):
reduction indices w, generating vector z', random shift Delta,
digital-net generating matrices C^(j) and a digital shift, and the dense
matrix A.  Both sides (oracle/ and the CUDA path) consume identical arrays.

Streams are counter-based SplitMix64: value i of stream (seed, sid) is
mix64(key(seed, sid) + (i+1)*GOLDEN), so any prefix/subset is reproducible.

Configurations C1..C5 mirror BASELINE.json `configs`; the readings
of under-specified parts (C-10..C-17 in SURVEY §8(c)) are listed in DESIGN.md.
"""
from __future__ import annotations

import dataclasses
import math
import os
from typing import Optional

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# stream ids
S_Z, S_SHIFT, S_NETC, S_DSHIFT, S_A = 1, 2, 3, 4, 5


def _mix64(x: np.ndarray) -> np.ndarray:
    x = x.copy()
    x ^= x >> np.uint64(30)
    x *= _M1
    x ^= x >> np.uint64(27)
    x *= _M2
    x ^= x >> np.uint64(31)
    return x


def stream(seed: int, sid: int, n: int, offset: int = 0) -> np.ndarray:
    """n uint64 values of counter-based stream (seed, sid), starting at counter `offset`."""
    with np.errstate(over="ignore"):
        key = _mix64(np.array([np.uint64(seed) * GOLDEN + np.uint64(sid)], dtype=np.uint64))[0]
        ctr = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return _mix64(key + ctr * GOLDEN)


def uniform53(seed: int, sid: int, n: int) -> np.ndarray:
    """Dyadic uniforms (u64 >> 11) * 2^-53 in [0, 1) (reading C-10)."""
    return (stream(seed, sid, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normals(seed: int, sid: int, n: int) -> np.ndarray:
    """Box-Muller N(0,1) draws (reading C-16)."""
    u = stream(seed, sid, 2 * ((n + 1) // 2))
    u1 = ((u[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53  # (0, 1]
    u2 = (u[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * len(u1))
    z[0::2] = r * np.cos(2.0 * math.pi * u2)
    z[1::2] = r * np.sin(2.0 * math.pi * u2)
    return z[:n]


def ilog_floor(j: int, b: int) -> int:
    """Largest e with b^e <= j, in integers (reading C-12: float log misrounds at powers)."""
    e, p = 0, b
    while p <= j:
        e += 1
        p *= b
    return e


def w_log(b: int, m: int, s: int, c: float = 1.0) -> np.ndarray:
    """w_j = min(floor(log_b j^c), m), j = 1..s (SPEC S:636-644 `log:c`)."""
    out = np.empty(s, dtype=np.int32)
    for j in range(1, s + 1):
        if c == 1.0:
            e = ilog_floor(j, b)
        else:  # floor(c*log_b j) by integer comparison: largest e with b^e <= j^c
            e = 0
            while float(b) ** (e + 1) <= float(j) ** c * (1 + 1e-15):
                e += 1
        out[j - 1] = min(e, m)
    return out


def draw_z(seed: int, b: int, m: int, w: np.ndarray) -> np.ndarray:
    """z'_j in [1, b^m) coprime to b, then reduced mod M_j = b^{m-w_j}; z'_j = 1 if w_j >= m (C-11)."""
    s = len(w)
    u = stream(seed, S_Z, s)
    N = b ** m
    z = np.empty(s, dtype=np.uint64)
    for j in range(s):
        if b == 2:
            v = (int(u[j]) % (N // 2)) * 2 + 1
        else:
            q = int(u[j] >> np.uint64(8)) % (b ** (m - 1))
            v = q * b + 1 + (int(u[j]) % (b - 1))
        Mj = b ** (m - min(int(w[j]), m))
        z[j] = 1 if Mj == 1 else v % Mj
    return z


def draw_net_matrices(seed: int, m: int, w: np.ndarray, delete_cols: bool = True) -> np.ndarray:
    """Unit upper-triangular m x m GF(2) matrices with columns m-w_j..m-1 zeroed (BASELINE C3, reading C-7);
    delete_cols=False keeps every column (full nonsingular matrices for the row-zeroed nets of
    Alg. 3/4, KIND_NET_ROWS, whose row zeroing the plan applies).

    Returned as column words: C[j*m + q] holds column q (input digit q, LSB-first digit of n);
    bit (m-1-p) is entry C_{p+1, q+1} (output digit p+1 has weight 2^-(p+1))  (reading C-8).
    """
    s = len(w)
    u = stream(seed, S_NETC, s * m)
    C = np.zeros(s * m, dtype=np.uint64)
    for j in range(s):
        keep = m - min(int(w[j]), m) if delete_cols else m  # columns q < keep survive
        for q in range(m):
            if q >= keep:
                continue
            # column q of an upper-triangular matrix: rows p <= q (0-based), diagonal p == q is 1
            rnd = int(u[j * m + q]) & ((1 << q) - 1) if q > 0 else 0  # rows 0..q-1 random
            col = 0
            for p in range(q):
                if (rnd >> p) & 1:
                    col |= 1 << (m - 1 - p)
            col |= 1 << (m - 1 - q)
            C[j * m + q] = col
    return C


def a_iid(seed: int, s: int, tau: int, sd: float) -> np.ndarray:
    return (normals(seed, S_A, s * tau) * sd).reshape(s, tau)


def a_brownian_chol(s: int, tau: int) -> np.ndarray:
    """Upper Cholesky factor R of Sigma_ij = min(i,j)/s: R_ji = s^-1/2 for j <= i (reading C-15)."""
    assert s == tau
    return np.triu(np.full((s, tau), 1.0 / math.sqrt(s)))


def a_exp_chol(s: int, tau: int, ell: float) -> np.ndarray:
    """First s rows of the upper Cholesky factor of Sigma_ij = rho^|i-j| (tau x tau), rho = exp(-1/ell).

    AR(1) closed form (reading C-14): R_{1,i} = rho^(i-1); R_{j,i} = rho^(i-j) sqrt(1-rho^2), 2 <= j <= i.
    """
    rho = math.exp(-1.0 / ell)
    i = np.arange(tau)[None, :]
    j = np.arange(s)[:, None]
    R = np.where(i >= j, rho ** np.maximum(i - j, 0).astype(np.float64), 0.0)
    R[1:, :] *= math.sqrt(1.0 - rho * rho)
    return R


def a_kl(s: int, tau: int) -> np.ndarray:
    """A_ji = j^-2 sin(j pi t_i), t_i = (i+0.5)/tau, j = 1..s (BASELINE C3; reading C-13)."""
    j = np.arange(1, s + 1, dtype=np.float64)[:, None]
    t = (np.arange(tau, dtype=np.float64)[None, :] + 0.5) / tau
    return j ** -2.0 * np.sin(j * math.pi * t)


# f ids (match include/rqmc.h rqmc_f)
F_NONE, F_EXP_MEAN, F_CALL_MEAN_EXP, F_MEAN_SQ, F_MEAN = -1, 0, 1, 2, 3
KIND_LATTICE, KIND_NET, KIND_MC, KIND_NET_ROWS = 0, 1, 2, 3
MAP_UNIT, MAP_INVNORM, MAP_TENT = 0, 1, 2   # TENT: phi(x) = 1 - |1 - 2x|


@dataclasses.dataclass
class Problem:
    """All inputs of one reduced-QMC problem (P:390-391 / P:473-475 plus shift, map and f)."""
    name: str
    kind: int
    b: int
    m: int
    s: int
    tau: int
    w: np.ndarray                      # int32[s]
    z: Optional[np.ndarray]            # uint64[s]  lattice z'_j
    C: Optional[np.ndarray]            # uint64[s*m] net column words
    shift: Optional[np.ndarray]        # float64[s] lattice shift Delta
    dshift: Optional[np.ndarray]       # uint64[s] 53-bit digital shift words
    map: int
    A: np.ndarray                      # float64[s, tau]
    f: int
    fparam: np.ndarray                 # float64[2]
    store_y: bool
    seed: int
    mc_seed: int = 0                   # reduced MC (KIND_MC): seed of the counter-based draws

    @property
    def N(self) -> int:
        return self.b ** self.m


def as_reduced_mc(prob: Problem, mc_seed: Optional[int] = None) -> Problem:
    """The same layout (b, m, w), map, A and f with reduced Monte Carlo points (Sec. 5,
    P:975-1000): no generating vector / matrices / shifts, draws seeded by
    mc_seed (default: the problem's seed)."""
    return dataclasses.replace(prob, name=prob.name + "MC", kind=KIND_MC, z=None, C=None, shift=None,
                               dshift=None, mc_seed=int(prob.seed if mc_seed is None else mc_seed))


def make_config(cfg: str, seed: Optional[int] = None) -> Problem:
    """BASELINE.json configs C1..C5 (SURVEY §8(d) 'Inputs (exact)'); a suffix "MC" (e.g. C5MC) gives
    the same workload with reduced Monte Carlo points (as_reduced_mc).  "C3R" is C3 with the paper's
    row-zeroed net (Alg. 3/4): full unit upper-triangular C^(j), the plan zeroes
    their last w_j rows; same shift, A and f."""
    cfg = cfg.upper()
    if cfg.endswith("MC"):
        return as_reduced_mc(make_config(cfg[:-2], seed))
    if cfg in ("C1U", "C5U"):
        # NEXT-4 workloads: the config without its random shift (unshifted lattice: every coordinate
        # of a level has the same map, so the per-level FFT product applies)
        p = make_config(cfg[:-1], seed)
        return dataclasses.replace(p, name=cfg, shift=None)
    if cfg == "C3R":
        p = make_config("C3", seed)
        return dataclasses.replace(p, name="C3R", kind=KIND_NET_ROWS,
                                   C=draw_net_matrices(p.seed, p.m, p.w, delete_cols=False))
    seeds = {"C1": 1001, "C2": 1002, "C3": 1003, "C4": 1004, "C5": 1005}
    sd = seeds[cfg] if seed is None else seed
    fp = np.zeros(2)
    if cfg == "C1":
        b, m, s, tau = 2, 10, 32, 32
        w = w_log(b, m, s)
        return Problem(cfg, KIND_LATTICE, b, m, s, tau, w, draw_z(sd, b, m, w), None, None, None,
                       MAP_UNIT, a_iid(sd, s, tau, 1.0), F_EXP_MEAN, fp, True, sd)
    if cfg == "C2":
        b, m, s, tau = 2, 16, 256, 256
        w = w_log(b, m, s)
        return Problem(cfg, KIND_LATTICE, b, m, s, tau, w, draw_z(sd, b, m, w), None,
                       uniform53(sd, S_SHIFT, s), None, MAP_INVNORM, a_brownian_chol(s, tau),
                       F_CALL_MEAN_EXP, np.array([0.2, 1.0]), False, sd)
    if cfg == "C3":
        b, m, s, tau = 2, 20, 1024, 1024
        w = w_log(b, m, s)
        return Problem(cfg, KIND_NET, b, m, s, tau, w, None, draw_net_matrices(sd, m, w), None,
                       stream(sd, S_DSHIFT, s) >> np.uint64(11), MAP_UNIT, a_kl(s, tau),
                       F_EXP_MEAN, fp, False, sd)
    if cfg == "C4":
        b, m, s, tau = 3, 12, 2000, 4096
        w = w_log(b, m, s)
        return Problem(cfg, KIND_LATTICE, b, m, s, tau, w, draw_z(sd, b, m, w), None,
                       uniform53(sd, S_SHIFT, s), None, MAP_INVNORM, a_exp_chol(s, tau, 0.1 * s),
                       F_MEAN_SQ, fp, True, sd)
    if cfg == "C5":
        b, m, s, tau = 2, 24, 4096, 2048
        w = w_log(b, m, s)
        return Problem(cfg, KIND_LATTICE, b, m, s, tau, w, draw_z(sd, b, m, w), None,
                       uniform53(sd, S_SHIFT, s), None, MAP_INVNORM, a_iid(sd, s, tau, 1.0 / math.sqrt(s)),
                       F_EXP_MEAN, fp, False, sd)
    raise ValueError(cfg)


def make_random(seed: int, b: int, m: int, s: int, tau: int, kind: int = KIND_LATTICE,
                shifted: bool = False, mapping: int = MAP_UNIT, wmode: str = "log",
                f: int = F_EXP_MEAN, int_a: bool = False) -> Problem:
    """Small random problems for property sweeps: random nondecreasing w with w_1 = 0."""
    # RQMC_TEST_SEED_OFFSET (tools/fuzz_parity.sh): the same sweeps on other seeds; both sides get the same inputs
    seed = seed + int(os.environ.get("RQMC_TEST_SEED_OFFSET", "0") or 0)
    rng = stream(seed, 99, 4 * s + 8)
    if wmode == "log":
        w = w_log(b, m, s)
    elif wmode == "zero":
        w = np.zeros(s, dtype=np.int32)
    else:  # random nondecreasing, may exceed m
        steps = (rng[:s] % np.uint64(3)).astype(np.int64)
        steps[0] = 0
        w = np.minimum(np.cumsum(steps * (rng[s:2 * s] % np.uint64(2)).astype(np.int64)), m + 2).astype(np.int32)
        w[0] = 0
    if int_a:
        A = ((stream(seed, S_A, s * tau) % np.uint64(17)).astype(np.int64) - 8).astype(np.float64).reshape(s, tau)
    else:
        A = (uniform53(seed, S_A, s * tau) * 2.0 - 1.0).reshape(s, tau)
    if kind == KIND_MC:
        return Problem(f"rand{seed}", kind, b, m, s, tau, w, None, None, None, None, mapping, A, f,
                       np.array([0.2, 1.0]), True, seed, mc_seed=seed * 7 + 1)
    if kind == KIND_LATTICE:
        z = draw_z(seed, b, m, w)
        sh = uniform53(seed, S_SHIFT, s) if shifted else None
        if shifted and int_a:  # dyadic shift with <= 30 bits keeps every partial sum exact
            sh = (stream(seed, S_SHIFT, s) >> np.uint64(34)).astype(np.float64) * 2.0 ** -30
        return Problem(f"rand{seed}", kind, b, m, s, tau, w, z, None, sh, None, mapping, A, f,
                       np.array([0.2, 1.0]), True, seed)
    assert b == 2
    C = draw_net_matrices(seed, m, w, delete_cols=kind != KIND_NET_ROWS)
    ds = None
    if shifted:
        ds = stream(seed, S_DSHIFT, s) >> np.uint64(11)
        if int_a:
            ds = ds & np.uint64(((1 << 30) - 1) << 23)  # top 30 of 53 digits only
    return Problem(f"rand{seed}", kind, b, m, s, tau, w, None, C, None, ds, mapping, A, f,
                   np.array([0.2, 1.0]), True, seed)
