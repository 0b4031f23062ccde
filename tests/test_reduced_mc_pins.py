"""Pins for the reduced Monte Carlo oracle (Sec. 5).

The oracle builds x_{j,n} = y_{j, m_s N_{s+1} + ... + m_j N_{j+1}} from the mixed-radix digits of n
(Eq. randpts).  What pins it (not itself):
  * the paper's displayed point pattern (P:99-120 display, golden paper_example_p99.txt);
  * the closed form of the truncated index: it equals n mod N_j (N_{j+1} | N_j);
  * multiplicity: each bank value is used exactly b^{w_j} times (counting over all n);
  * Theorem 5: the variance of the estimator, computed by EXHAUSTIVE enumeration of
    all Bernoulli banks through the oracle, equals the theorem's formula with mu_u evaluated from
    its definition -- an exact, deterministic check of the sharing structure;
  * unbiasedness E Q(f) = E f, exactly by the same enumeration;
  * the counter-based draws: uniform moments (closed forms 1/2, 1/12) and no repeated words.
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W


def mc(b, m, w, A=None, f=W.F_EXP_MEAN, mapping=W.MAP_UNIT, seed=1):
    s = len(w)
    A = np.ones((s, 1)) if A is None else np.asarray(A, dtype=np.float64)
    return W.Problem("mc", W.KIND_MC, b, m, s, A.shape[1], np.array(w, np.int32), None, None, None, None,
                     mapping, A, f, np.zeros(2), True, 0, mc_seed=seed)


def _golden(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as fh:
        return [l.split() for l in fh if l.strip() and not l.startswith("#")]


def test_randpts_paper_display(golden_dir):
    """P:99-120 / SPEC reduced-MC example: N_1=4, N_2=2, N_3=1 (w = 0, 1, 2; m = 2) -> point k uses
    (y_{1,k}, y_{2,k mod 2}, y_{3,0}); SPEC: n = 3 -> (y_{1,3}, y_{2,1}, y_{3,0})."""
    p = mc(2, 2, [0, 1, 2])
    for k, i1, i2, i3 in (map(int, r) for r in _golden(golden_dir, "paper_example_p99.txt")):
        assert [oracle.mc_bank_index(p, k, j) for j in range(3)] == [i1, i2, i3]
    X = oracle.mc_points_bank(p, [[10, 11, 12, 13], [20, 21], [30]])
    np.testing.assert_array_equal(X, [[10, 20, 30], [11, 21, 30], [12, 20, 30], [13, 21, 30]])


@pytest.mark.parametrize("b,m,seed", [(2, 5, 1), (3, 3, 2), (2, 6, 3), (5, 2, 4)])
def test_truncated_index_is_n_mod_Nj_and_multiplicity(b, m, seed):
    """Eq. randpts' index sum_{i>=j} m_i N_{i+1} < N_j and n - index is a multiple of N_j, i.e. the
    index is n mod N_j; every bank value of coordinate j is used b^{w_j} times (S: multiplicity)."""
    rng = np.random.default_rng(seed)
    s = 7
    w = np.concatenate([[0], np.sort(rng.integers(0, m + 2, s - 1))]).astype(np.int32)
    p = mc(b, m, w)
    N = b ** m
    for j in range(s):
        Nj = b ** (m - min(int(w[j]), m))
        idx = [oracle.mc_bank_index(p, n, j) for n in range(N)]
        assert idx == [n % Nj for n in range(N)]
        counts = np.bincount(idx, minlength=Nj)
        assert (counts == b ** min(int(w[j]), m)).all()


def _theorem5(mu, M):
    """Var Q = sum_{k=1}^s mu_{k..s} prod_{j=k}^s M_j^-1 (1 - 1/M_{k-1}) - mu_0 / M_s, 1 - 1/M_0 := 1."""
    s = len(M)
    v = 0.0
    for k in range(1, s + 1):
        prod = 1.0
        for j in range(k, s + 1):
            prod /= M[j - 1]
        fac = 1.0 if k == 1 else 1.0 - 1.0 / M[k - 2]
        v += mu[k] * prod * fac
    return v - mu[0] / M[s - 1]


@pytest.mark.parametrize("b,m,w,support", [
    (2, 2, [0, 1, 2], (0.0, 1.0)),
    (2, 3, [0, 1, 1], (0.0, 1.0)),
    (2, 2, [0, 0, 1], (-1.0, 2.0)),
    (3, 1, [0, 0, 1], (0.0, 1.0)),
    (2, 3, [0, 2, 3], (0.0, 1.0)),
])
def test_variance_theorem_exhaustive(b, m, w, support):
    """Theorem 5: exact variance of Q(f) = N^-1 sum_n f(x_n) over ALL bank realizations
    (each y_{j,r} uniform on a 2-point support) equals the formula; also E Q = E f (unbiased)."""
    s = len(w)
    A = np.array([[0.7, -0.2], [0.3, 0.9], [-0.5, 0.4]])[:s]
    p = mc(b, m, w, A=A, f=W.F_EXP_MEAN)
    wc = [min(x, m) for x in w]
    Nj = [b ** (m - x) for x in wc]
    M = [b ** ((wc[j + 1] if j + 1 < s else m) - wc[j]) for j in range(s)]   # M_j = N_j / N_{j+1}

    def f(x):  # the integrand f(x) = exp(mean(x^T A)) by its definition (reading C-17)
        return math.exp(float(np.mean(np.asarray(x) @ A)))

    # mu_u for tail sets u = {k..s}: E_{x_u}[(E_{x_-u} f(x_u, x_-u))^2], iid coordinates
    mu = {0: sum(f(x) for x in itertools.product(support, repeat=s)) ** 2 / len(support) ** (2 * s)}
    for k in range(1, s + 1):
        u = list(range(k - 1, s))
        rest = list(range(0, k - 1))
        tot = 0.0
        for xu in itertools.product(support, repeat=len(u)):
            g = 0.0
            for xr in itertools.product(support, repeat=len(rest)):
                x = [0.0] * s
                for i, v in zip(u, xu):
                    x[i] = v
                for i, v in zip(rest, xr):
                    x[i] = v
                g += f(x)
            g /= len(support) ** len(rest)
            tot += g * g
        mu[k] = tot / len(support) ** len(u)
    # exhaustive enumeration of the banks through the oracle's reduced-MC sample matrix + product + f
    nb = sum(Nj)
    assert len(support) ** nb <= 1 << 17
    q1 = q2 = 0.0
    cnt = 0
    for vals in itertools.product(support, repeat=nb):
        cols, o = [], 0
        for n_j in Nj:
            cols.append(vals[o:o + n_j])
            o += n_j
        X = oracle.mc_points_bank(p, cols)
        Q = float(np.mean(oracle.f_of_y(oracle.product(X, A), W.F_EXP_MEAN, None)))
        q1 += Q
        q2 += Q * Q
        cnt += 1
    EQ = q1 / cnt
    var = q2 / cnt - EQ * EQ
    assert abs(EQ - math.sqrt(mu[0])) <= 1e-12 * abs(EQ)           # unbiased: E Q = E f
    assert abs(var - _theorem5(mu, M)) <= 1e-10 * max(1.0, abs(var))


def test_theorem5_classical_special_cases():
    """S: s = 1, M_1 = N gives (mu_1 - mu_0)/N; all M_j = 1 gives mu_{1..s} - mu_0."""
    mu = {0: 2.0, 1: 5.0}
    assert _theorem5(mu, [8]) == pytest.approx((5.0 - 2.0) / 8)
    mu = {0: 2.0, 1: 9.0, 2: 4.0, 3: 3.0}
    assert _theorem5(mu, [1, 1, 1]) == pytest.approx(9.0 - 2.0)


def test_counter_draws_uniform_and_distinct():
    """u = (word|1) 2^-53 of the counter-based stream: mean 1/2 and variance 1/12 (closed forms of
    U(0,1)) within 6 standard errors over 2^17 draws from 8 coordinates; no repeated words."""
    words = np.array([oracle.mc_word(12345, j, r) for j in range(8) for r in range(1 << 14)], dtype=np.uint64)
    assert len(np.unique(words)) == len(words)
    assert (words < (np.uint64(1) << np.uint64(53))).all()
    u = (words | np.uint64(1)).astype(np.float64) * 2.0 ** -53
    n = len(u)
    assert 0.0 < u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 6 * math.sqrt(1 / 12 / n)
    assert abs(u.var() - 1 / 12) < 6 * math.sqrt(1 / 180 / n)
    # different coordinates are different streams: correlation of paired draws ~ 0
    a = u[: 1 << 14]
    c = u[1 << 14: 2 << 14]
    assert abs(np.corrcoef(a, c)[0, 1]) < 6 / math.sqrt(1 << 14)


def test_points_follow_bank_draws():
    """orc_point for reduced MC = the bank of counter draws read through Eq. randpts (Phi^-1 map too)."""
    p = mc(2, 4, [0, 1, 1, 2, 3, 5], mapping=W.MAP_INVNORM, seed=99)
    X, T = oracle.points(p)
    for n in range(p.N):
        for j in range(p.s):
            r = oracle.mc_bank_index(p, n, j)
            wd = oracle.mc_word(99, j, r)
            assert int(T[n, j]) == wd
            assert X[n, j] == oracle.invnorm((wd | 1) * 2.0 ** -53)


def test_bank_indices_one_pass_equals_per_coordinate():
    """orc_mc_bank_indices (one digit pass per point, used by the full-N tabulation) equals the
    per-coordinate Eq. randpts index orc_mc_bank_index for every coordinate (random layouts, w > m)."""
    rng = np.random.default_rng(17)
    for b, m in ((2, 9), (3, 6), (5, 4)):
        prob = W.make_random(60 + b, b, m, 40, 3, kind=W.KIND_MC, wmode="rand")
        for n in list(rng.integers(0, prob.N, 40)) + [0, prob.N - 1]:
            got = oracle.mc_bank_indices(prob, int(n))
            assert [int(v) for v in got] == [oracle.mc_bank_index(prob, int(n), j) for j in range(prob.s)]
