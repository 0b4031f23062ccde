"""Pins for the CPU oracle against what the paper and mathematics fix (not against itself).

Each test names the passage it follows (P:n = PAPER.md line, S:n = SPEC.md line).
A plausible oracle bug -- dropped term, wrong sign/index, transposed operand, wrong periodicity
reading, wrong digit order -- fails at least one of these.
"""
import math
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
import workloads as W


def _golden(golden_dir, name):
    rows = []
    with open(os.path.join(golden_dir, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def lattice(b, m, w, z, shift=None, mapping=W.MAP_UNIT, A=None):
    s = len(w)
    A = np.zeros((s, 1)) if A is None else np.asarray(A, dtype=np.float64)
    return W.Problem("t", W.KIND_LATTICE, b, m, s, A.shape[1], np.array(w, np.int32),
                     np.array(z, np.uint64), None, None if shift is None else np.array(shift, np.float64),
                     None, mapping, A, W.F_MEAN, np.zeros(2), True, 0)


def net(m, w, cols, dshift=None, mapping=W.MAP_UNIT, A=None):
    s = len(w)
    A = np.zeros((s, 1)) if A is None else np.asarray(A, dtype=np.float64)
    return W.Problem("t", W.KIND_NET, 2, m, s, A.shape[1], np.array(w, np.int32), None,
                     np.array(cols, np.uint64), None, None if dshift is None else np.array(dshift, np.uint64),
                     mapping, A, W.F_MEAN, np.zeros(2), True, 0)


# ---------------------------------------------------------------- point sets (O1)

def test_paper_example_periodicity(golden_dir):
    """with N_1=4, N_2=2, N_3=1 coordinate j of point k uses y_{j, k mod N_j}."""
    # reduced lattice with b=2, m=2, w=(0,1,2): N_j = 4, 2, 1
    p = lattice(2, 2, [0, 1, 2], [1, 1, 1])
    X, T = oracle.points(p)
    for k, i1, i2, i3 in (map(int, r) for r in _golden(golden_dir, "paper_example_p99.txt")):
        # value of coordinate j equals the value at the representative index i_j
        assert X[k, 0] == X[i1, 0] and X[k, 1] == X[i2, 1] and X[k, 2] == X[i3, 2]
    assert len(set(X[:, 0])) == 4 and len(set(X[:, 1])) == 2 and len(set(X[:, 2])) == 1


def test_spec_reduced_column_and_full_sets(golden_dir):
    g = {r[0]: r[1:] for r in _golden(golden_dir, "spec_reduced_column.txt")}
    # S:59 reduced column (b=2, m=3, z_j=3, w_j=1): rows 0..3, tiled twice
    p = lattice(2, 3, [0, 1], [1, 3])
    X, _ = oracle.points(p)
    col = [float(Fr(v)) for v in g["reduced_column"]]
    assert list(X[:4, 1]) == col and list(X[4:, 1]) == col
    # S:68
    X, _ = oracle.points(lattice(2, 2, [0, 2], [1, 1]))
    exp = [[float(Fr(a)) for a in r.split(",")] for r in g["full_b2m2"]]
    assert X.tolist() == exp
    # S:70
    X, _ = oracle.points(lattice(3, 1, [0], [1]))
    assert X[:, 0].tolist() == [float(Fr(v)) for v in g["full_b3m1"]]


@pytest.mark.parametrize("name,b,m,w,z,shift", [
    ("g1_lattice.txt", 2, 3, [0, 1, 2], [3, 1, 1], None),
    ("g1s_lattice_shift.txt", 2, 3, [0, 1, 2], [3, 1, 1], [1 / 16, 3 / 8, 1 / 2]),
])
def test_golden_g1(golden_dir, name, b, m, w, z, shift):
    A = np.array([[1, 2], [-1, 0], [2, -3]], dtype=np.float64)
    p = lattice(b, m, w, z, shift, A=A)
    X, _ = oracle.points(p)
    Y = oracle.product(X, A)
    for r in _golden(golden_dir, name):
        k = int(r[0])
        assert X[k].tolist() == [float(Fr(v)) for v in r[1:4]]      # bit-exact (dyadic)
        assert Y[k].tolist() == [float(Fr(v)) for v in r[4:6]]


def test_golden_g2_base3(golden_dir):
    p = lattice(3, 2, [0, 0, 1], [1, 2, 1], A=np.ones((3, 1)))
    X, _ = oracle.points(p)
    Y = oracle.product(X, p.A)
    for r in _golden(golden_dir, "g2_lattice_b3.txt"):
        k = int(r[0])
        np.testing.assert_allclose(X[k], [float(Fr(v)) for v in r[1:4]], rtol=0, atol=1e-16)
        assert abs(Y[k, 0] - float(Fr(r[4]))) <= 1e-15   # 3 rounded thirds: a few ulp


def test_golden_g3_net(golden_dir):
    # C1 = I; C2 = [[1,1,0],[0,1,0],[0,0,0]] as column words (bit m-p for row p)
    cols = [4, 2, 1, 4, 6, 0]
    X, _ = oracle.points(net(3, [0, 1], cols))
    for r in _golden(golden_dir, "g3_net.txt"):
        assert X[int(r[0])].tolist() == [float(Fr(v)) for v in r[1:3]]


def _radical_inverse(n, m):
    """Textbook van der Corput radical inverse in base 2 of n < 2^m."""
    x, f = Fr(0), Fr(1, 2)
    while n:
        if n & 1:
            x += f
        n >>= 1
        f /= 2
    return x


def test_net_identity_is_van_der_corput():
    """C = I gives the van der Corput sequence (m=3, n=5 -> 0.625)."""
    m = 6
    cols = [1 << (m - 1 - q) for q in range(m)]  # identity: column q has output digit q+1
    X, T = oracle.points(net(m, [0], cols))
    for n in range(2 ** m):
        assert X[n, 0] == float(_radical_inverse(n, m))
    X3, _ = oracle.points(net(3, [0], [4, 2, 1]))
    assert X3[5, 0] == 0.625


def test_net_row_zeroing_matches_paper_equation():
    """Eq. reduced_genmat_net2: the last min(w_j,m) rows are dropped; for w_j >= m the
    matrix is zero. With a full (non-column-deleted) C, values lie on the grid of step
    2^-(m-w_j) and the oracle must NOT keep the dropped rows."""
    m = 5
    rng = np.random.default_rng(3)
    full = [int(rng.integers(1, 2 ** m)) for _ in range(m)]
    for wj in (0, 1, 3, 5, 7):
        X, T = oracle.points(net(m, [0, wj], [1 << (m - 1 - q) for q in range(m)] + full))
        step = 2.0 ** -(m - min(wj, m))
        assert np.all(np.mod(X[:, 1], step) == 0.0)
        if wj >= m:
            assert np.all(X[:, 1] == 0.0)
        # brute force: y_p = sum_q C_pq kappa_q mod 2 with rows p > m - w zeroed
        for n in range(2 ** m):
            y = Fr(0)
            for pp in range(1, m - min(wj, m) + 1):
                bit = sum(((full[q] >> (m - pp)) & 1) * ((n >> q) & 1) for q in range(m)) % 2
                y += Fr(bit, 2 ** pp)
            assert X[n, 1] == float(y)


@pytest.mark.parametrize("b,m,s", [(2, 8, 20), (3, 5, 14), (5, 3, 9)])
def test_lattice_periodicity_multiplicity_and_means(b, m, s):
    """coordinate j takes values t/b^{m-min(w_j,m)}, each exactly b^{min(w_j,m)} times,
    column j is periodic with period M_j; closed-form mean (1 - b^{-(m-w_j)})/2 (B.ns)."""
    w = W.w_log(b, m, s)
    z = W.draw_z(7, b, m, w)
    X, T = oracle.points(lattice(b, m, w, z))
    N = b ** m
    for j in range(s):
        Mj = b ** (m - min(int(w[j]), m))
        col = X[:, j]
        assert np.array_equal(col, np.tile(col[:Mj], N // Mj))
        vals, cnt = np.unique(col, return_counts=True)
        assert len(vals) == Mj and np.all(cnt == N // Mj)
        assert np.all(np.mod(T[:, j], N // Mj) == 0)     # numerator k z_j mod N is a multiple of b^{w_j}
        mean = math.fsum(col) / N
        assert abs(mean - (1 - 1 / Mj) / 2) <= 1e-15
    if m > 0:
        jj = int(np.nonzero(w >= m)[0][0]) if np.any(w >= m) else None
        if jj is not None:
            assert np.all(X[:, jj] == 0.0)               # j > s*: zero column


@pytest.mark.parametrize("b,m,s", [(2, 8, 20), (3, 5, 14), (5, 3, 9)])
def test_tent_map_definition_and_means(b, m, s):
    """Tent transformation phi(x) = 1 - |1 - 2x| (the alternative to the random shift):
    phi(0) = 0, phi(1/4) = phi(3/4) = 1/2, phi(1/2) = 1.  An unshifted reduced lattice column is a
    permutation of the grid {t / M_j}, so its tent-mapped mean is sum_t phi(t/M)/M = 1/2 for
    even M and 1/2 - 1/(2 M^2) for odd M (pairs t, M - t; 0 for M = 1), and the map acts entry by entry on
    the unmapped points (by exact rationals for b = 2, where t/M is dyadic)."""
    assert (oracle.tent(0.0), oracle.tent(0.25), oracle.tent(0.5), oracle.tent(0.75)) == (0.0, 0.5, 1.0, 0.5)
    w = W.w_log(b, m, s)
    z = W.draw_z(7, b, m, w)
    X, _ = oracle.points(lattice(b, m, w, z, mapping=W.MAP_TENT))
    Xu, _ = oracle.points(lattice(b, m, w, z))
    N = b ** m
    for j in range(s):
        Mj = b ** (m - min(int(w[j]), m))
        exp = Fr(1, 2) if Mj % 2 == 0 else Fr(1, 2) - Fr(1, 2 * Mj * Mj)
        assert abs(math.fsum(X[:, j]) / N - float(exp)) <= 1e-15
        assert np.array_equal(X[:, j], np.tile(X[:Mj, j], N // Mj))
        for k in range(0, N, max(1, N // 37)):
            t = 1 - abs(1 - 2 * Fr(Xu[k, j]))
            if b == 2:
                assert Fr(X[k, j]) == t
            else:
                assert abs(Fr(X[k, j]) - t) <= Fr(1, 2 ** 52)


def test_shifted_means_closed_form():
    """psi(x) = {x + Delta}: mean of M equispaced shifted values = (1-1/M)/2 + {M Delta}/M."""
    b, m, s = 2, 9, 40
    w = W.w_log(b, m, s)
    z = W.draw_z(11, b, m, w)
    sh = W.uniform53(11, W.S_SHIFT, s)
    X, _ = oracle.points(lattice(b, m, w, z, sh))
    for j in range(s):
        M = b ** (m - min(int(w[j]), m))
        exp = (1 - 1 / M) / 2 + (M * sh[j] - math.floor(M * sh[j])) / M
        assert abs(math.fsum(X[:, j]) / b ** m - exp) <= 4e-16
        assert np.array_equal(X[:, j], np.tile(X[:M, j], b ** m // M))


def test_net_c3_style_periodic_permutation():
    """Reading C-7: unit upper-triangular C with columns >= m-w_j deleted gives points that are
    periodic with period 2^{m-w_j} and each period is a permutation of the grid; digital shift mean."""
    m, s = 8, 24
    w = W.w_log(2, m, s)
    Cw = W.draw_net_matrices(5, m, w)
    ds = W.stream(5, W.S_DSHIFT, s) >> np.uint64(11)
    X0, T0 = oracle.points(net(m, w, Cw))
    X1, T1 = oracle.points(net(m, w, Cw, ds))
    N = 2 ** m
    for j in range(s):
        M = 2 ** (m - min(int(w[j]), m))
        assert np.array_equal(X0[:, j], np.tile(X0[:M, j], N // M))
        assert sorted(X0[:M, j].tolist()) == [t / M for t in range(M)]
        assert np.array_equal(T1[:, j], (T0[:, j] << np.uint64(53 - m)) ^ ds[j])
        sig_low = int(ds[j]) % (2 ** (53 - (m - min(int(w[j]), m))))
        exp = (1 - 1 / M) / 2 + sig_low * 2.0 ** -53
        assert abs(math.fsum(X1[:, j]) / N - exp) <= 4e-16


# ---------------------------------------------------------------- Phi^-1

def test_invnorm_values_and_symmetry():
    assert abs(oracle.invnorm(0.975) - 1.959963984540054) <= 2e-15
    assert oracle.invnorm(0.5) == 0.0
    for u in (2.0 ** -53, 2.0 ** -30, 3 * 2.0 ** -20, 0.25, 0.375, 0.5 - 2.0 ** -40):
        assert oracle.invnorm(1 - u) == -oracle.invnorm(u)   # S:282; u dyadic so 1-u is exact


def test_invnorm_against_library_and_roundtrip():
    """Independent library routine (scipy ndtri) and the defining equation Phi(x) = u (math.erfc)."""
    from scipy.special import ndtri
    rng = np.random.default_rng(0)
    us = np.concatenate([rng.random(3000), 2.0 ** -np.arange(2, 60, 3.0), 1 - 2.0 ** -np.arange(2, 53, 3.0)])
    for u in us:
        x = oracle.invnorm(u)
        assert abs(x - ndtri(u)) <= 2e-15 * max(1.0, abs(x))
        q = 0.5 * math.erfc(-x / math.sqrt(2))
        assert abs(q - u) <= 4e-16 * max(u, 1e-300) * max(1.0, x * x) + 1e-300


def test_zero_rule():
    """Reading C-5: unshifted Phi^-1 maps u=0 to b^-m/2."""
    p = lattice(2, 4, [0, 1], [1, 1], mapping=W.MAP_INVNORM)
    X, _ = oracle.points(p)
    assert X[0, 0] == oracle.invnorm(0.5 / 16) and X[0, 1] == oracle.invnorm(0.5 / 16)
    assert X[8, 0] == 0.0 and X[4, 1] == 0.0       # u = 1/2 -> 0


def test_zero_rule_shifted():
    """Reading C-5, shifted branch: a shifted coordinate that wraps to exactly u = 0 is mapped as
    u = 2^-53.  G1s (tests/golden/g1s_lattice_shift.txt) has x_{k,3} = {k/2 + 1/2} = 0 for every
    odd k, so with Phi^-1 those entries are Phi^-1(2^-53) -- pinned against scipy's ndtri (an
    independent library routine), like every other G1s entry against ndtri of its golden value."""
    from scipy.special import ndtri
    p = lattice(2, 3, [0, 1, 2], [3, 1, 1], [1 / 16, 3 / 8, 1 / 2], mapping=W.MAP_INVNORM)
    X, T = oracle.points(p)
    unit = oracle.points(lattice(2, 3, [0, 1, 2], [3, 1, 1], [1 / 16, 3 / 8, 1 / 2]))[0]
    for k in range(8):
        for j in range(3):
            u = unit[k, j]
            ref = ndtri(2.0 ** -53) if u == 0.0 else ndtri(u)
            assert abs(X[k, j] - ref) <= 2e-15 * max(1.0, abs(ref)), (k, j)
    assert all(unit[k, 2] == 0.0 for k in (1, 3, 5, 7))          # the wrap happens (golden table)
    assert abs(X[1, 2] - (-8.209536151601387)) <= 2e-14            # Phi^-1(2^-53) (scipy ndtri)


def test_f_all_tab_equals_rowwise():
    """The full-N oracle with column tabulation and cache blocking (orc_f_all_tab) is the plain
    O1+O2+O3 path reorganised without changing any per-entry operation order: bit-identical to
    f_rows on every kind, map, shift and f (including ragged row / column blocks)."""
    for kind, b, m in ((W.KIND_LATTICE, 2, 7), (W.KIND_LATTICE, 3, 5), (W.KIND_NET, 2, 7), (W.KIND_MC, 2, 6)):
        for f in (W.F_EXP_MEAN, W.F_CALL_MEAN_EXP, W.F_MEAN_SQ, W.F_MEAN):
            prob = W.make_random(90 + f, b, m, 71, 131, kind=kind, shifted=kind != W.KIND_MC,
                                 mapping=W.MAP_INVNORM if f % 2 else W.MAP_UNIT, wmode="rand", f=f)
            assert np.array_equal(oracle.f_all_tab(prob), oracle.f_rows(prob, np.arange(prob.N)))


# ---------------------------------------------------------------- product (O2) and Q_N (O3)

def _frac_points(b, m, w, z, shift_fr=None):
    """Exact rationals x_{k,j} = (k z'_j mod M_j)/M_j (second form of P:308-309) + {x + Delta}."""
    N = b ** m
    out = []
    for k in range(N):
        row = []
        for j in range(len(w)):
            M = b ** (m - min(w[j], m))
            x = Fr(k * z[j] % M, M)
            if shift_fr is not None:
                x += shift_fr[j]
                if x >= 1:
                    x -= 1
            row.append(x)
        out.append(row)
    return out


def _alg2_exact(b, m, w, Xfr, A):
    """PAPER Alg. 2 in exact rationals, including empty levels and w_j >= m columns
    dropped (s*): P_I = tile(P_{I+1}, b) + X_I A_I, descending I."""
    tau = len(A[0])
    sstar = max(j for j in range(len(w)) if w[j] < m) + 1
    P = [[Fr(0)] * tau]
    for I in range(m - 1, -1, -1):
        rows = b ** (m - I)
        js = [j for j in range(sstar) if w[j] == I]
        newP = []
        for r in range(rows):
            row = list(P[r % len(P)])
            for j in js:
                x = Xfr[r][j]            # reduced point row r of coordinate j (k = r < b^{m-I})
                row = [row[c] + x * A[j][c] for c in range(tau)]
            newP.append(row)
        P = newP
    return P


@pytest.mark.parametrize("seed,b,m,s,tau", [(1, 2, 5, 9, 3), (2, 3, 3, 7, 4), (3, 2, 4, 5, 6), (4, 5, 2, 8, 2)])
def test_product_exact_bruteforce_and_alg2(seed, b, m, s, tau):
    """Naive product equals exact rational brute force sum_j x_kj A_jc and PAPER Alg. 2;
    A is non-square with small-integer entries so any transposed operand or wrong index fails."""
    rng = np.random.default_rng(seed)
    w = sorted([0] + list(rng.integers(0, m + 2, s - 1)))
    z = W.draw_z(seed, b, m, np.array(w))
    A = rng.integers(-8, 9, (s, tau)).astype(np.float64)
    p = lattice(b, m, w, z, A=A)
    X, _ = oracle.points(p)
    Y = oracle.product(X, A)
    Xfr = _frac_points(b, m, w, [int(v) for v in z])
    Afr = [[Fr(int(v)) for v in row] for row in A]
    exact = [[sum(Xfr[k][j] * Afr[j][c] for j in range(s)) for c in range(tau)] for k in range(b ** m)]
    alg2 = _alg2_exact(b, m, w, Xfr, Afr)
    assert exact == alg2                                  # Alg. 2 reaches the plain result exactly
    tol = 0.0 if b == 2 else 1e-13
    for k in range(b ** m):
        for c in range(tau):
            assert abs(Y[k, c] - float(exact[k][c])) <= tol


def test_product_identity_matrix():
    """A = I_s makes XA = X (pins product indexing)."""
    prob = W.make_random(21, 2, 7, 12, 12, shifted=True)
    X, _ = oracle.points(prob)
    assert np.array_equal(oracle.product(X, np.eye(12)), X)


def test_qn_linear_closed_form():
    """Linear f (B.ns): Q_N = xbar^T A 1 / tau with the closed-form column means."""
    b, m, s, tau = 2, 10, 48, 16
    prob = W.make_random(5, b, m, s, tau, shifted=True, f=W.F_MEAN)
    xbar = []
    for j in range(s):
        M = b ** (m - min(int(prob.w[j]), m))
        d = prob.shift[j]
        xbar.append((1 - 1 / M) / 2 + (M * d - math.floor(M * d)) / M)
    exp = float(np.dot(np.array(xbar), prob.A.sum(axis=1)) / tau)
    got = oracle.qn_sum(prob) / prob.N
    assert abs(got - exp) <= 1e-13 * max(1.0, abs(exp))


def test_qn_exp_mean_identity():
    """O3' (g = id): exp(mean(x^T A)) == exp(x . abar); independent O(Ns) path agrees with naive."""
    prob = W.make_config("C1")
    ks = np.arange(prob.N)
    a = oracle.f_rows(prob, ks)
    b = oracle.f_rows_meanid(prob, ks)
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=0)
    assert abs(oracle.neumaier(a) - oracle.neumaier(b)) <= 1e-13 * abs(oracle.neumaier(a))


def test_f_definitions_by_hand():
    """C-17 definitions of the five f's on a hand-checkable row."""
    Y = np.array([[0.0, 1.0, -1.0, 2.0]])
    assert oracle.f_of_y(Y, W.F_MEAN, None)[0] == 0.5
    assert oracle.f_of_y(Y, W.F_EXP_MEAN, None)[0] == math.exp(0.5)
    assert oracle.f_of_y(Y, W.F_MEAN_SQ, None)[0] == 1.5
    exp = (1 + math.exp(0.2) + math.exp(-0.2) + math.exp(0.4)) / 4 - 1
    assert abs(oracle.f_of_y(Y, W.F_CALL_MEAN_EXP, [0.2, 1.0])[0] - max(exp, 0)) <= 1e-16
    assert oracle.f_of_y(Y, W.F_CALL_MEAN_EXP, [0.2, 5.0])[0] == 0.0


def test_neumaier():
    assert oracle.neumaier(np.array([1e16, 1.0, -1e16])) == 1.0
    v = np.random.default_rng(1).standard_normal(10000) * 1e3
    assert oracle.neumaier(v) == math.fsum(v)


# ---------------------------------------------------------------- inputs (workloads)

def test_w_rule():
    assert W.w_log(2, 4, 8).tolist() == [0, 1, 1, 2, 2, 2, 2, 3]
    w3 = W.w_log(3, 12, 3 ** 10 + 2)
    assert w3[3 ** 5 - 1] == 5 and w3[3 ** 5 - 2] == 4 and w3[3 ** 10 - 1] == 10   # reading C-12
    assert W.w_log(2, 3, 40).max() == 3                                 # clamp at m


def test_cholesky_closed_forms():
    s = 64
    R = W.a_brownian_chol(s, s)
    i = np.arange(1, s + 1)
    np.testing.assert_allclose(R.T @ R, np.minimum.outer(i, i) / s, atol=1e-15)   # C-15
    R2 = W.a_exp_chol(s, s, 7.0)
    rho = math.exp(-1 / 7.0)
    np.testing.assert_allclose(R2.T @ R2, rho ** np.abs(np.subtract.outer(i, i)), atol=2e-15)  # C-14
    np.testing.assert_allclose(R2, np.linalg.cholesky(rho ** np.abs(np.subtract.outer(i, i))).T, atol=1e-14)


def test_configs_valid():
    for c in ("C1", "C2", "C3", "C4"):
        p = W.make_config(c)
        assert p.A.shape == (p.s, p.tau) and p.w[0] == 0 and np.all(np.diff(p.w) >= 0)
        if p.kind == W.KIND_LATTICE:
            for j in range(p.s):
                M = p.b ** (p.m - min(int(p.w[j]), p.m))
                assert 1 <= int(p.z[j]) < max(M, 2) and math.gcd(int(p.z[j]), p.b) == 1


def test_meanid_tabulated_equals_rowwise():
    """The tabulated O3' (column periodicity) equals the row-wise O3' and the naive O3."""
    for prob in (W.make_random(31, 2, 9, 70, 8, shifted=True, mapping=W.MAP_INVNORM),
                 W.make_random(32, 3, 5, 30, 5, shifted=True, mapping=W.MAP_INVNORM),
                 W.make_random(33, 2, 8, 20, 6, kind=W.KIND_NET, shifted=True)):
        ks = np.arange(prob.N)
        tab = oracle.f_all_meanid_tab(prob)
        assert np.array_equal(tab, oracle.f_rows_meanid(prob, ks))
        np.testing.assert_allclose(tab, oracle.f_rows(prob, ks), rtol=1e-13)


# ---------------------------------------------------------------- Q_N for the C2 / C4 integrands

def _exact_points(b, m, w, z, shift):
    """x_{k,j} = {k z_j / N + Delta_j} in exact rationals, z_j = b^{w_j} z'_j."""
    N = b ** m
    pts = []
    for k in range(N):
        row = []
        for j in range(len(w)):
            zj = (b ** min(w[j], m)) * z[j] % N if w[j] < m else 0
            x = Fr(k * zj % N, N) + Fr(shift[j])
            row.append(x - 1 if x >= 1 else x)
        pts.append(row)
    return pts


def test_qn_mean_sq_exact_rational():
    """C4's f = mean(y^2) (reading C-17): the oracle's Q_N sum over a b = 3 shifted lattice with an
    integer A equals the exact rational sum of the definition (brute force) to 1e-15."""
    b, m, w, z = 3, 3, [0, 0, 1, 2], [1, 2, 4, 1]
    shift = [Fr(1, 8), Fr(3, 4), Fr(0), Fr(5, 16)]   # dyadic shifts: exact in fp64
    A = np.array([[1, -2, 3], [2, 0, -1], [-1, 1, 1], [3, 2, -2]], dtype=np.float64)
    p = W.Problem("t", W.KIND_LATTICE, b, m, 4, 3, np.array(w, np.int32), np.array(z, np.uint64), None,
                  np.array([float(s) for s in shift]), None, W.MAP_UNIT, A, W.F_MEAN_SQ, np.zeros(2), True, 0)
    exact = Fr(0)
    for x in _exact_points(b, m, w, z, shift):
        y = [sum(x[j] * int(A[j, c]) for j in range(4)) for c in range(3)]
        exact += sum(v * v for v in y) / 3
    q = oracle.qn_sum(p)
    assert abs(q - float(exact)) <= 1e-15 * float(exact)


def test_qn_call_mean_exp_high_precision():
    """C2's f = max(mean exp(0.2 y) - 1, 0) (reading C-17): the oracle's Q_N sum over a b = 2 shifted
    lattice equals the definition evaluated on the exact rational points in 40-digit arithmetic
    (mpmath, an exp implementation independent of libm) to 1e-14 relative."""
    import mpmath as mp
    mp.mp.dps = 40
    b, m, w, z = 2, 5, [0, 1, 1, 2, 3], [3, 1, 5, 3, 1]
    shift = [Fr(1, 32), Fr(7, 16), Fr(3, 8), Fr(0), Fr(9, 64)]
    A = np.array([[2.5, -1.0], [1.0, 3.0], [-2.0, 0.5], [4.0, 1.5], [0.25, -3.0]])
    p = W.Problem("t", W.KIND_LATTICE, b, m, 5, 2, np.array(w, np.int32), np.array(z, np.uint64), None,
                  np.array([float(s) for s in shift]), None, W.MAP_UNIT, A, W.F_CALL_MEAN_EXP,
                  np.array([0.2, 1.0]), True, 0)
    ref = mp.mpf(0)
    Am = [[mp.mpf(float(v)) for v in row] for row in A]
    for x in _exact_points(b, m, w, z, shift):
        y = [mp.fsum(mp.mpf(x[j].numerator) / x[j].denominator * Am[j][c] for j in range(5)) for c in range(2)]
        ref += max(mp.fsum(mp.exp(mp.mpf("0.2") * v) for v in y) / 2 - 1, 0)
    q = oracle.qn_sum(p)
    assert abs(q - float(ref)) <= 1e-14 * float(ref)
