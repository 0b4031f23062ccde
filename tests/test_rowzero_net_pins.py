"""Pins for the row-zeroed digital nets of Alg. 3/4.

The oracle has two independent product paths for them: O1 (Eq. reduced_genmat_net2 row zeroing,
then Eq. def:digital) + O2 (naive product), and Alg. 4 step by step (full net y_n, the table
c_k = (k/b^{m-w_j}) a_j and the gather floor(y_{n,j} b^{m-w_j})).  They must agree, and both are
pinned to a hand-derived worked example and to closed forms.
"""
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
import workloads as W


def rnet(m, w, cols, A, dshift=None, mapping=W.MAP_UNIT):
    s = len(w)
    A = np.asarray(A, dtype=np.float64)
    return W.Problem("t", W.KIND_NET_ROWS, 2, m, s, A.shape[1], np.array(w, np.int32), None,
                     np.array(cols, np.uint64), None, None if dshift is None else np.array(dshift, np.uint64),
                     mapping, A, W.F_MEAN, np.zeros(2), True, 0)


def test_golden_g4_rowzero_net(golden_dir):
    """Hand-derived example (tests/golden/g4_rowzero_net.txt): points, product by O1+O2 and by Alg. 4."""
    p = rnet(3, [0, 1], [4, 2, 1, 4, 6, 7], [[1.0], [1.0]])
    X, _ = oracle.points(p)
    Y2 = oracle.xa(p)
    Y4 = oracle.alg4_xa(p)
    rows = []
    with open(os.path.join(golden_dir, "g4_rowzero_net.txt")) as fh:
        rows = [ln.split() for ln in fh if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 8
    for r in rows:
        n = int(r[0])
        assert X[n].tolist() == [float(Fr(r[1])), float(Fr(r[2]))]
        assert Y2[n, 0] == float(Fr(r[3])) and Y4[n, 0] == float(Fr(r[3]))


def test_antidiagonal_generator_closed_form():
    """C^(j) = anti-identity (output digit p = input digit m-p) gives y_n = n / 2^m; zeroing the last
    w rows truncates it to z_{j,n} = floor(n / 2^w) / 2^{m-w}: blocks of 2^w equal values, the opposite
    of the lattice's periodic pattern."""
    m, w = 7, [0, 1, 2, 2, 3, 5, 7, 9]
    s = len(w)
    cols = [1 << q for q in range(m)] * s
    rng = np.random.default_rng(5)
    A = rng.integers(-8, 9, size=(s, 3)).astype(np.float64)
    p = rnet(m, w, cols, A)
    X, T = oracle.points(p)
    n = np.arange(2 ** m)
    for j in range(s):
        wj = min(w[j], m)
        expect = (n >> wj).astype(np.float64) * 2.0 ** -(m - wj)
        assert np.array_equal(X[:, j], expect)
        assert np.array_equal(T[:, j], ((n >> wj) << wj).astype(np.uint64))
    # exact product: every term is a dyadic with <= m bits times a small integer
    expect_y = sum(np.outer((n >> min(w[j], m)) * 2 ** min(w[j], m), A[j]) for j in range(s)) / 2.0 ** m
    assert np.array_equal(oracle.xa(p), expect_y)
    assert np.array_equal(oracle.alg4_xa(p), expect_y)


@pytest.mark.parametrize("seed,m,s,wmode", [(1, 8, 20, "rand"), (2, 9, 33, "log"), (3, 7, 50, "rand")])
def test_value_multiplicity_and_grid(seed, m, s, wmode):
    """For nonsingular C^(j), component j of the reduced net lies on {k / b^{m-w_j}} and takes each
    value exactly b^{min(w_j,m)} times; no common period."""
    p = W.make_random(seed, 2, m, s, 2, kind=W.KIND_NET_ROWS, wmode=wmode)
    X, _ = oracle.points(p)
    nonperiodic = 0
    for j in range(s):
        wj = min(int(p.w[j]), m)
        Mj = 2 ** (m - wj)
        k = X[:, j] * Mj
        assert np.array_equal(k, np.floor(k))
        counts = np.bincount(k.astype(np.int64), minlength=Mj)
        assert counts.shape == (Mj,) and (counts == 2 ** wj).all()
        if 0 < wj < m and not np.array_equal(X[:, j], np.tile(X[:Mj, j], 2 ** wj)):
            nonperiodic += 1
    assert nonperiodic > 0


def test_column_deleted_nets_coincide():
    """On a column-deleted matrix (reading C-7) the row-zeroed definition gives the same points as
    RQMC_DIGITAL_NET: zeroing rows of an upper-triangular matrix with columns >= m-w already zero
    changes nothing (P:671 vs P:601-605)."""
    p1 = W.make_random(7, 2, 9, 40, 3, kind=W.KIND_NET, shifted=True)
    import dataclasses
    p3 = dataclasses.replace(p1, kind=W.KIND_NET_ROWS)
    assert np.array_equal(oracle.points(p1)[1], oracle.points(p3)[1])


@pytest.mark.parametrize("seed,m,s,tau,wmode", [(11, 9, 37, 11, "rand"), (12, 10, 64, 5, "log"),
                                                  (13, 8, 90, 7, "rand")])
def test_alg4_equals_definition_exact(seed, m, s, tau, wmode):
    """Exact-arithmetic regime (integer A, |A| <= 8, dyadic points): Alg. 4's gathered table and the
    plain definition are bit-identical (includes w_j > m, i.e. j > s*)."""
    p = W.make_random(seed, 2, m, s, tau, kind=W.KIND_NET_ROWS, wmode=wmode, int_a=True, f=W.F_MEAN)
    assert np.array_equal(oracle.alg4_xa(p), oracle.xa(p))


def test_alg4_equals_definition_real():
    p = W.make_random(14, 2, 10, 70, 9, kind=W.KIND_NET_ROWS, wmode="log")
    Y2, Y4 = oracle.xa(p), oracle.alg4_xa(p)
    scale = np.abs(p.A).sum(axis=0)
    assert (np.abs(Y2 - Y4) <= 1e-14 * scale).all()


def test_alg4_rejects_shift_and_map():
    p = W.make_random(15, 2, 6, 8, 2, kind=W.KIND_NET_ROWS, shifted=True)
    with pytest.raises(ValueError):
        oracle.alg4_xa(p)
