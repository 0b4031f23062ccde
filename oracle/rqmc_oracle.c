/*
 * rqmc_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU oracle
 * for the reduced QMC matrix product of Dick, Ebert, Herrmann, Kritzer, Longo,
 * "The fast reduced QMC matrix-vector product" (arXiv 2305.11645; /root/reference/PAPER.md = P:n).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code, header, table or constant with the CUDA path
 * (paper_2305_11645_b200/csrc); the only common input is the seeded data from workloads/.
 *
 * What it computes: the PLAIN definition, never the reduced algorithm.
 *   O1 points  x_k materialised from the point-set definitions:
 *        lattice  x_{k,j} = { k z_j / N },  z_j = b^{w_j} z'_j          (first form P:307)
 *        shift    psi(x) = { x + Delta_j }
 *        net      vec y_{j,n} = Chat^(j) vec n, y = vec y . (b^-1..b^-m)    (Eq. def:digital)
 *                 Chat^(j): last min(w_j,m) rows of C^(j) set to zero      (Eq. reduced_genmat_net2)
 *        digital shift (reading C-9): V = (W << (53-m)) XOR sigma_j, x = V 2^-53
 *        reduced MC (Eq. randpts) x_{j,n} = y_{j, m_s N_{s+1} + ... + m_j N_{j+1}} from the
 *                 mixed-radix digits of n; the bank y_{j,r} is the counter-based stream of include/rqmc.h
 *        row-zeroed net (kind 3): the same definition with any C^(j) (no column deletion assumed)
 *        map      x = Phi^-1(u), zero rule reading C-5; or the tent
 *                 transformation phi(u) = 1 - |1 - 2u|
 *   O2 product Y[k,c] = sum_{j=1..s} x_{k,j} A[j,c], increasing j
 *   O3 f_k = F(tau^-1 sum_c g(Y[k,c])) (increasing c); sum_k f_k Neumaier-compensated
 *   O3' (g = id only) f_k = F(sum_j x_{k,j} abar_j), abar = tau^-1 A 1   -- algebraic identity, O(Ns)
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC (no FMA contraction).
 * Parity is pinned by tests/test_oracle_pins.py (paper example, SPEC examples, closed forms,
 * exact rational brute force, library Phi^-1); see DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int b, m, s;
  const int32_t* w;        /* s reduction indices, 0 = w_1 <= w_2 <= ... */
  int kind;                /* 0 lattice, 1 digital net (b = 2), 2 reduced MC, 3 row-zeroed net */
  const uint64_t* z;       /* lattice z'_j */
  const uint64_t* C;       /* net: column words, C[j*m+q] bit (m-1-p) = C^(j)_{p+1,q+1} */
  const double* shift;     /* lattice Delta_j in [0,1) or NULL */
  const uint64_t* dshift;  /* net sigma_j < 2^53 or NULL */
  int map;                 /* 0 identity, 1 Phi^-1, 2 tent */
  uint64_t seed;           /* kind 2 (reduced Monte Carlo): seed of the counter-based draws */
} orc_problem;

static uint64_t ipow(uint64_t b, int e) {
  uint64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

/* Standard normal CDF Phi(x) = erfc(-x/sqrt 2)/2 (libm erfc). */
static double orc_Phi(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

/* Phi^-1(u): the x with Phi(x) = u.  Start from Abramowitz-Stegun 26.2.23 and refine with
 * Halley steps on Phi(x) - q until the step stalls.  Works on q = min(u, 1-u) (x <= 0 side,
 * where erfc is accurate in relative terms) and restores the sign (Phi^-1(1-u) = -Phi^-1(u)). */
double orc_invnorm(double u) {
  if (!(u > 0.0 && u < 1.0)) return NAN;
  if (u == 0.5) return 0.0;
  double q = u < 0.5 ? u : 1.0 - u;
  double t = sqrt(-2.0 * log(q));
  double x = -(t - (2.515517 + 0.802853 * t + 0.010328 * t * t) /
                       (1.0 + 1.432788 * t + 0.189269 * t * t + 0.001308 * t * t * t));
  for (int it = 0; it < 100; ++it) {
    double e = orc_Phi(x) - q;
    double phi = exp(-0.5 * x * x) / sqrt(2.0 * M_PI);
    double dx = e / (phi + 0.5 * x * e);
    x -= dx;
    if (fabs(dx) <= 1e-17 * fmax(1.0, fabs(x))) break;
  }
  return u < 0.5 ? x : -x;
}

/* The tent transformation phi(x) = 1 - |1 - 2x| (the alternative to the random
 * shift), evaluated as written: 2x, 1 - 2x, |.|, 1 - |.| in fp64 (2x is exact). */
double orc_tent(double u) { return 1.0 - fabs(1.0 - 2.0 * u); }

/* u in [0,1) -> point coordinate: identity, Phi^-1 with the zero rule (reading C-5), or the tent map. */
static double orc_map(const orc_problem* p, double u, int shifted) {
  if (p->map == 0) return u;
  if (p->map == 2) return orc_tent(u);
  if (u == 0.0) u = shifted ? ldexp(1.0, -53) : 0.5 / (double)ipow((uint64_t)p->b, p->m);
  return orc_invnorm(u);
}

/* ---- reduced Monte Carlo (Sec. 5) ------------------------------------------------- */

/* Eq. randpts: with N_j = b^{m - w_j} (w_j clamped to m), N_{s+1} = 1, M_j = N_j / N_{j+1}, write
 * n = m_s N_{s+1} + m_{s-1} N_s + ... + m_1 N_2 with 0 <= m_i < M_i; coordinate j of
 * point n takes bank sample number m_s N_{s+1} + ... + m_j N_{j+1} (digits j..s only). */
uint64_t orc_mc_bank_index(const orc_problem* p, uint64_t n, int j) {
  uint64_t idx = 0, rem = n;
  for (int i = p->s - 1; i >= 0; --i) {                     /* i = s-1 .. 0 <-> paper's s .. 1 */
    const int wi = p->w[i] < p->m ? p->w[i] : p->m;
    const int wn = (i + 1 < p->s) ? (p->w[i + 1] < p->m ? p->w[i + 1] : p->m) : p->m;  /* w_{s+1} = m */
    const uint64_t Ni1 = ipow((uint64_t)p->b, p->m - wn);  /* N_{i+1} */
    const uint64_t Mi = ipow((uint64_t)p->b, wn - wi);     /* M_i = N_i / N_{i+1} */
    const uint64_t mi = rem % Mi;                          /* digit m_i (radix M_i, weight N_{i+1}) */
    rem /= Mi;
    if (i >= j) idx += mi * Ni1;
  }
  return idx;
}

/* All coordinates' bank indices of point n in one pass: the digits m_i of Eq. randpts do not depend
 * on j, so idx[j] = sum_{i >= j} m_i N_{i+1} is a suffix sum (same recurrence as orc_mc_bank_index). */
void orc_mc_bank_indices(const orc_problem* p, uint64_t n, uint64_t* idx) {
  uint64_t rem = n, acc = 0;
  for (int i = p->s - 1; i >= 0; --i) {
    const int wi = p->w[i] < p->m ? p->w[i] : p->m;
    const int wn = (i + 1 < p->s) ? (p->w[i + 1] < p->m ? p->w[i + 1] : p->m) : p->m;
    const uint64_t Ni1 = ipow((uint64_t)p->b, p->m - wn);
    const uint64_t Mi = ipow((uint64_t)p->b, wn - wi);
    acc += (rem % Mi) * Ni1;
    rem /= Mi;
    idx[i] = acc;
  }
}

/* the counter-based draw y_{j,r} (include/rqmc.h, rqmc_kind): 53-bit word and u = (word|1) 2^-53 */
static uint64_t orc_mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
uint64_t orc_mc_word(uint64_t seed, int j, uint64_t r) {
  const uint64_t G = 0x9E3779B97F4A7C15ull;
  const uint64_t key = orc_mix64(seed * G + (uint64_t)(j + 1));
  return orc_mix64(key + (r + 1) * G) >> 11;
}

/* Eq. randpts with an explicit bank: X[i][j] = bank[off[j] + index_j(k0 + i)] (the sample matrix of
 * SPEC's reduced-MC module; used with finite discrete banks by the exact-variance pin). */
int orc_mc_points_bank(const orc_problem* p, const double* bank, const int64_t* off, int64_t k0,
                       int64_t n, double* X) {
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < p->s; ++j)
      X[i * p->s + j] = bank[off[j] + (int64_t)orc_mc_bank_index(p, (uint64_t)(k0 + i), j)];
  return 0;
}

/* reduced MC: coordinate j's draw from bank index idx, mapped */
static double orc_mc_value(const orc_problem* p, int j, uint64_t idx, uint64_t* word_out) {
  const uint64_t word = orc_mc_word(p->seed, j, idx);
  if (word_out) *word_out = word;
  const double u = (double)(word | 1u) * ldexp(1.0, -53);    /* in (0,1): no zero rule needed */
  return p->map == 0 ? u : (p->map == 2 ? orc_tent(u) : orc_invnorm(u));
}

/* O1 for one entry: coordinate j of point k (value, and its integer word in *word). */
double orc_point(const orc_problem* p, uint64_t k, int j, uint64_t* word_out) {
  const uint64_t N = ipow((uint64_t)p->b, p->m);
  int wj = p->w[j];
  double u;
  uint64_t word;
  int shifted;
  if (p->kind == 2) return orc_mc_value(p, j, orc_mc_bank_index(p, k, j), word_out);
  if (p->kind == 0) {
    /* z_j = b^{w_j} z'_j; for w_j >= m, z_j is a multiple of N. */
    uint64_t zj = wj >= p->m ? 0 : (uint64_t)(((unsigned __int128)ipow((uint64_t)p->b, wj) * p->z[j]) % N);
    word = (uint64_t)(((unsigned __int128)k * zj) % N);     /* k z_j mod N */
    u = (double)word / (double)N;                            /* { k z_j / N } */
    shifted = p->shift != NULL;
    if (shifted) {                                           /* psi(x) = {x + Delta}, reading C-6 */
      u = u + p->shift[j];
      if (u >= 1.0) u = u - 1.0;
    }
  } else {
    /* digits of k, least significant first; Chat rows p > m - min(w_j,m) zeroed */
    int keep_rows = p->m - (wj < p->m ? wj : p->m);
    uint64_t W = 0;
    for (int pp = 1; pp <= p->m; ++pp) {            /* output digit p (weight b^-p) */
      if (pp > keep_rows) continue;                 /* row of Chat is zero */
      unsigned y = 0;
      for (int qq = 1; qq <= p->m; ++qq) {          /* input digit q */
        unsigned kappa = (unsigned)((k >> (qq - 1)) & 1u);
        unsigned c = (unsigned)((p->C[(size_t)j * p->m + (qq - 1)] >> (p->m - pp)) & 1u);
        y = (y + c * kappa) % 2u;
      }
      W += (uint64_t)y << (p->m - pp);              /* sum_p y_p 2^{m-p} */
    }
    shifted = p->dshift != NULL;
    if (shifted) {
      word = (W << (53 - p->m)) ^ p->dshift[j];
      u = (double)word * ldexp(1.0, -53);
    } else {
      word = W;
      u = (double)W * ldexp(1.0, -p->m);
    }
  }
  if (word_out) *word_out = word;
  return orc_map(p, u, shifted);
}

/* O1: rows k in [k0, k0+n) of X (row-major n x s); T gets the integer word of each entry:
 * lattice: (k z_j mod N) (numerator over N); net: W (unshifted m-digit word) or V (shifted 53-digit). */
int orc_points(const orc_problem* p, int64_t k0, int64_t n, double* X, uint64_t* T) {
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < p->s; ++j) {
      uint64_t word;
      double x = orc_point(p, (uint64_t)(k0 + i), j, &word);
      if (T) T[i * p->s + j] = word;
      if (X) X[i * p->s + j] = x;
    }
  return 0;
}

/* O1 on arbitrary rows ks[0..n): X (n x s). */
int orc_points_rows(const orc_problem* p, const int64_t* ks, int64_t n, double* X, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < p->s; ++j) X[i * p->s + j] = orc_point(p, (uint64_t)ks[i], j, NULL);
  return 0;
}

/* O2: naive product Y (n x tau) = X (n x s) A (s x tau), each Y[k,c] accumulated in increasing j. */
void orc_product(int64_t n, int s, int tau, const double* X, const double* A, double* Y) {
  for (int64_t k = 0; k < n; ++k) {
    double* y = Y + k * tau;
    for (int c = 0; c < tau; ++c) y[c] = 0.0;
    for (int j = 0; j < s; ++j) {
      double x = X[k * s + j];
      const double* a = A + (size_t)j * tau;
      for (int c = 0; c < tau; ++c) y[c] = y[c] + x * a[c];
    }
  }
}

/* O3: f_k = F(tau^-1 sum_c g(y_c)), c increasing (readings C-17). f ids as workloads.F_*. */
static double orc_f_row(const double* y, int tau, int f, const double* fp) {
  double acc = 0.0;
  switch (f) {
    case 0: for (int c = 0; c < tau; ++c) acc = acc + y[c]; return exp(acc / tau);
    case 1: for (int c = 0; c < tau; ++c) acc = acc + exp(fp[0] * y[c]);
            acc = acc / tau - fp[1]; return acc > 0.0 ? acc : 0.0;
    case 2: for (int c = 0; c < tau; ++c) acc = acc + y[c] * y[c]; return acc / tau;
    case 3: for (int c = 0; c < tau; ++c) acc = acc + y[c]; return acc / tau;
    default: return NAN;
  }
}

void orc_f(int64_t n, int tau, const double* Y, int f, const double* fp, double* fk) {
  for (int64_t k = 0; k < n; ++k) fk[k] = orc_f_row(Y + k * tau, tau, f, fp);
}

/* Neumaier-compensated sum in increasing index. */
double orc_neumaier(const double* v, int64_t n) {
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double t = s + v[i];
    if (fabs(s) >= fabs(v[i])) c += (s - t) + v[i];
    else c += (v[i] - t) + s;
    s = t;
  }
  return s + c;
}

/* f_k for arbitrary rows ks[0..n) via O1+O2+O3, OpenMP over rows (order within a row fixed). */
int orc_f_rows(const orc_problem* p, const double* A, int tau, int f, const double* fp,
               const int64_t* ks, int64_t n, double* fk, double* Yrows /* nullable n x tau */,
               int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  int err = 0;
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * p->s);
    double* y = (double*)malloc(sizeof(double) * tau);
    if (!x || !y) err = 1;
#pragma omp for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
      if (!x || !y) continue;
      orc_points(p, ks[i], 1, x, NULL);
      orc_product(1, p->s, tau, x, A, y);
      fk[i] = orc_f_row(y, tau, f, fp);
      if (Yrows) memcpy(Yrows + i * tau, y, sizeof(double) * tau);
    }
    free(x);
    free(y);
  }
  return err;
}

/* O3': for g = id (f in {0: exp(mean), 3: mean}): f_k = F(sum_j x_{k,j} abar_j), abar = tau^-1 A 1. */
int orc_f_rows_meanid(const orc_problem* p, const double* A, int tau, int f, const int64_t* ks,
                      int64_t n, double* fk, int nthreads) {
  if (f != 0 && f != 3) return 1;
  double* abar = (double*)malloc(sizeof(double) * p->s);
  for (int j = 0; j < p->s; ++j) {
    double acc = 0.0;
    for (int c = 0; c < tau; ++c) acc = acc + A[(size_t)j * tau + c];
    abar[j] = acc / tau;
  }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * p->s);
#pragma omp for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
      orc_points(p, ks[i], 1, x, NULL);
      double acc = 0.0;
      for (int j = 0; j < p->s; ++j) acc = acc + x[j] * abar[j];
      fk[i] = f == 0 ? exp(acc) : acc;
    }
    free(x);
  }
  free(abar);
  return 0;
}

/* O3' over ALL rows with the column tabulation SURVEY §8(c) allows: x_{k,j} depends only on
 * k mod M_j (pinned by the periodicity tests), so column j is tabulated from its plain
 * definition at k = 0..M_j-1 and f_k = F(sum_j tab_j[k mod M_j] abar_j) (increasing j). */
int orc_f_all_meanid_tab(const orc_problem* p, const double* A, int tau, int f, double* fk, int nthreads) {
  if (f != 0 && f != 3) return 1;
  if (p->kind == 3) return 3;   /* row-zeroed nets are not periodic in k */
  const uint64_t N = ipow((uint64_t)p->b, p->m);
  uint64_t* M = (uint64_t*)malloc(sizeof(uint64_t) * p->s);
  size_t* off = (size_t*)malloc(sizeof(size_t) * (p->s + 1));
  double* abar = (double*)malloc(sizeof(double) * p->s);
  off[0] = 0;
  for (int j = 0; j < p->s; ++j) {
    int wj = p->w[j] < p->m ? p->w[j] : p->m;
    M[j] = ipow((uint64_t)p->b, p->m - wj);
    off[j + 1] = off[j] + M[j];
    double acc = 0.0;
    for (int c = 0; c < tau; ++c) acc = acc + A[(size_t)j * tau + c];
    abar[j] = acc / tau;
  }
  double* tab = (double*)malloc(sizeof(double) * off[p->s]);
  if (!tab) { free(M); free(off); free(abar); return 2; }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  if (p->kind == 2) {
    /* reduced MC: entries r < M_j of every column j from one digit pass per r (orc_mc_bank_indices) */
    uint64_t Mmax = 0;
    for (int j = 0; j < p->s; ++j) Mmax = M[j] > Mmax ? M[j] : Mmax;
#pragma omp parallel
    {
      uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * p->s);
#pragma omp for schedule(static, 1024)
      for (int64_t r = 0; r < (int64_t)Mmax; ++r) {
        orc_mc_bank_indices(p, (uint64_t)r, idx);
        for (int j = 0; j < p->s; ++j)
          if ((uint64_t)r < M[j]) tab[off[j] + r] = orc_mc_value(p, j, idx[j], NULL);
      }
      free(idx);
    }
  } else {
#pragma omp parallel for schedule(dynamic, 1)
    for (int j = 0; j < p->s; ++j)
      for (uint64_t r = 0; r < M[j]; ++r) tab[off[j] + r] = orc_point(p, r, j, NULL);
  }
#pragma omp parallel for schedule(static, 4096)
  for (int64_t k = 0; k < (int64_t)N; ++k) {
    double acc = 0.0;
    for (int j = 0; j < p->s; ++j) acc = acc + tab[off[j] + (uint64_t)k % M[j]] * abar[j];
    fk[k] = f == 0 ? exp(acc) : acc;
  }
  free(tab); free(M); free(off); free(abar);
  return 0;
}

/* O1+O2+O3 over ALL N rows for any f, for periodic kinds (lattice, column-deleted net, reduced MC):
 * column j is tabulated from its plain definition at k = 0..M_j-1 (x_{k,j} depends only on k mod M_j,
 * the tabulation SURVEY §8(c) allows), then the naive product Y[k,c] = sum_j x_{k,j} A[j,c]
 * in increasing j (O2) on blocks of 32 rows x 64 columns (cache blocking only: every Y[k,c] is the
 * same increasing-j sum as orc_product), and f_k = F(tau^-1 sum_c g(Y[k,c])) with the column sum
 * carried across column blocks in increasing c (O3, as orc_f_row).  fk[k] for k = 0..N-1.
 * Returns 1 for row-zeroed nets (not periodic), 2 on allocation failure. */
int orc_f_all_tab(const orc_problem* p, const double* A, int tau, int f, const double* fp, double* fk,
                  int nthreads) {
  if (p->kind == 3) return 1;
  const uint64_t N = ipow((uint64_t)p->b, p->m);
  const int s = p->s;
  uint64_t* M = (uint64_t*)malloc(sizeof(uint64_t) * s);
  size_t* off = (size_t*)malloc(sizeof(size_t) * (s + 1));
  if (!M || !off) { free(M); free(off); return 2; }
  off[0] = 0;
  for (int j = 0; j < s; ++j) {
    int wj = p->w[j] < p->m ? p->w[j] : p->m;
    M[j] = ipow((uint64_t)p->b, p->m - wj);
    off[j + 1] = off[j] + M[j];
  }
  double* tab = (double*)malloc(sizeof(double) * off[s]);
  if (!tab) { free(M); free(off); return 2; }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int j = 0; j < s; ++j)
    for (uint64_t r = 0; r < M[j]; ++r) tab[off[j] + r] = orc_point(p, r, j, NULL);
  enum { RB = 32, CB = 64 };
  int err = 0;
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * RB * s);
    double* y = (double*)malloc(sizeof(double) * RB * CB);
    double* acc = (double*)malloc(sizeof(double) * RB);
    if (!x || !y || !acc) err = 2;
#pragma omp for schedule(dynamic, 1)
    for (int64_t k0 = 0; k0 < (int64_t)N; k0 += RB) {
      if (!x || !y || !acc) continue;
      const int nr = (int64_t)N - k0 < RB ? (int)((int64_t)N - k0) : RB;
      for (int i = 0; i < nr; ++i) {
        for (int j = 0; j < s; ++j) x[i * s + j] = tab[off[j] + (uint64_t)(k0 + i) % M[j]];
        acc[i] = 0.0;
      }
      for (int c0 = 0; c0 < tau; c0 += CB) {
        const int nc = tau - c0 < CB ? tau - c0 : CB;
        for (int i = 0; i < nr * CB; ++i) y[i] = 0.0;
        for (int j = 0; j < s; ++j) {
          const double* a = A + (size_t)j * tau + c0;
          for (int i = 0; i < nr; ++i) {
            const double xv = x[i * s + j];
            double* yr = y + i * CB;
#pragma omp simd
            for (int c = 0; c < nc; ++c) yr[c] = yr[c] + xv * a[c];   /* independent c: no reordering */
          }
        }
        for (int i = 0; i < nr; ++i)
          for (int c = 0; c < nc; ++c) {
            const double v = y[i * CB + c];
            switch (f) {
              case 1: acc[i] = acc[i] + exp(fp[0] * v); break;
              case 2: acc[i] = acc[i] + v * v; break;
              default: acc[i] = acc[i] + v; break;
            }
          }
      }
      for (int i = 0; i < nr; ++i) {
        double r;
        switch (f) {
          case 0: r = exp(acc[i] / tau); break;
          case 1: r = acc[i] / tau - fp[1]; r = r > 0.0 ? r : 0.0; break;
          default: r = acc[i] / tau; break;
        }
        fk[k0 + i] = r;
      }
    }
    free(x); free(y); free(acc);
  }
  free(tab); free(M); free(off);
  return err;
}

/* Alg. 4, "fast reduced matrix product for digital nets", step by step, for the
 * unshifted, unmapped row-zeroed net (kind 3).  The input point set is the FULL digital net y_n of
 * Eq. def:digital (C^(j) without row zeroing); coordinate j uses the table
 *   c_k = (k / b^{m-w_j}) a_j,  k = 0 .. b^{m-w_j}-1,
 * and P_j = P_{j+1} + (c_{floor(y_{n,j} b^{m-w_j})})_n, for j = s* down to 1, P_{s*+1} = 0.
 * Y (N x tau) = P_1.  Returns 1 for shifts / maps / other kinds (Alg. 4 does not define them). */
int orc_alg4_product(const orc_problem* p, const double* A, int tau, double* Y) {
  if (p->kind != 3 || p->b != 2 || p->dshift || p->map != 0) return 1;
  const uint64_t N = ipow(2u, p->m);
  int s_star = 0;
  for (int j = 0; j < p->s; ++j)
    if (p->w[j] < p->m) s_star = j + 1;                       /* s* */
  for (uint64_t i = 0; i < N * (uint64_t)tau; ++i) Y[i] = 0.0;  /* P_{s*+1} = 0 */
  double* c = (double*)malloc(sizeof(double) * N * (size_t)tau);
  if (!c) return 2;
  for (int j = s_star - 1; j >= 0; --j) {                     /* j = s* .. 1 (0-based) */
    const uint64_t Mj = ipow(2u, p->m - p->w[j]);               /* b^{m-w_j} */
    const double* a = A + (size_t)j * tau;
    for (uint64_t k = 0; k < Mj; ++k)
      for (int cc = 0; cc < tau; ++cc) c[k * tau + cc] = ((double)k / (double)Mj) * a[cc];
    for (uint64_t n = 0; n < N; ++n) {
      /* y_{n,j}: full C^(j) times the digits of n (Eq. def:digital), all m output digits */
      uint64_t W = 0;
      for (int pp = 1; pp <= p->m; ++pp) {
        unsigned y = 0;
        for (int qq = 1; qq <= p->m; ++qq)
          y ^= (unsigned)((p->C[(size_t)j * p->m + (qq - 1)] >> (p->m - pp)) & 1u) & (unsigned)((n >> (qq - 1)) & 1u);
        W |= (uint64_t)y << (p->m - pp);
      }
      const double yv = (double)W * ldexp(1.0, -p->m);
      const uint64_t k = (uint64_t)floor(yv * (double)Mj);     /* floor(y_{n,j} b^{m-w_j}) */
      double* row = Y + n * (size_t)tau;
      for (int cc = 0; cc < tau; ++cc) row[cc] = row[cc] + c[k * tau + cc];
    }
  }
  free(c);
  return 0;
}
