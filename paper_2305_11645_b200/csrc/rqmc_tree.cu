// k_fine_tree: compile-time fused fine levels for the paper's level shape w_j = floor(log_b j)
// (every BASELINE config).  Rows a3+a4+a5 of SURVEY §8(a): Alg. 2's recursion
// R_w[r] = P_w[r] + R_w'[r mod M_w'] walked depth-first below one bundle of checkpoint
// residues, fused with the leaf consumption (Y store and/or F(tau^-1 sum_c g(y_c))).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "rqmc_device.cuh"
#include "rqmc_exp2_table.h"

namespace rqmc {

// ------------------------------------------------------------------------------------------
// k_fine_tree<NF, B, G, STY, NFR, BUN, NH>.  Fine level i (coarse -> fine) is w = NF-1-i with
// K_i = (B-1) B^{NF-1-i} coordinates, every node has B children, and the fine coordinates are the
// prefix j < B^NF - 1 of A.  With the whole tree compile-time every loop is unrolled and every
// smem offset is a constant.
//
// CTA = one bundle of BUN checkpoint residues (16; 8 for b = 3) x one CW = 32 NH column tile at a
// time (NH = 2: two 32-column passes per barrier interval when the doubled A slab still allows two
// CTAs per SM), B warp groups (group h walks the subtree under the top level's run q = h) x 4/NFR
// column slices x BUN/8 row warps.  A warp owns 8 residues x 8 NFR columns = NFR DMMA.8x8x4
// accumulator fragments, so a tree node is 2 NFR doubles per lane and the DFS stack lives in
// registers.  NFR = 4 (255 registers, 2 CTAs of 4 warps per SM on C5) is the default; NFR = 2
// (128 registers, more LDS and shuffles per output) measured 2 % slower.
//
//   K >= 4 levels : DMMA.8x8x4 k-steps (mma.sync f64, C and D in distinct registers); the K = 4
//                   level's B fragments cached per tile
//   K = 2 level   : 2 DFMA per output on A values cached in registers per column tile
//   K = 1 leaves  : 1 DFMA per output, then Y store / g, lane-local sums of g (g = exp: exp_core)
//   row sums      : b = 2: one transpose-reduce over the 4 lanes of a row per 4 NQ leaves; each
//                   lane keeps complete column-slice sums of its leaf rows in registers across all
//                   column tiles (no shared-memory row accumulators); other shapes: smem rowacc.
// Shared memory: [A slab x2][root tile x2][X^red subtree][rowacc]; A / root pitch CW + 4, X^red
// t-stride 20 (BUN 16) / 12 (BUN 8) doubles: bank-conflict-free fragment loads.  Columns >= tau are
// zero in the A slab and the root tile.
// ------------------------------------------------------------------------------------------
// bottom-block instruction order (C5 fine kernel): both K = 2 tiles of a node before its leaves
// (S1_FIRST) 16.97 ms; both K = 4 nodes' DMMAs first (S2_FIRST) 17.02; both 17.32; neither 17.34;
// computing both children of the level above the bottom first: 17.29
#ifndef RQMC_S2_FIRST
#define RQMC_S2_FIRST 0
#endif
#ifndef RQMC_S1_FIRST
#define RQMC_S1_FIRST 1
#endif
#ifndef RQMC_CACHE_B4
#define RQMC_CACHE_B4 1
#endif
#ifndef RQMC_FAST_EXP
#define RQMC_FAST_EXP 1
#endif
#ifndef RQMC_TREE_WIDE
#define RQMC_TREE_WIDE 1
#endif
#ifndef RQMC_TREE_BUNDLE        // residues per CTA: 16 (2 CTAs per SM) or 32 (1 CTA per SM)
#define RQMC_TREE_BUNDLE 16
#endif
#ifndef RQMC_EXP_TB            // exp table bits for g = exp: 6 (64 entries, degree 5) or 11 (2048, degree 3)
#define RQMC_EXP_TB 6
#endif
#ifndef RQMC_TREE43
#define RQMC_TREE43 0
#endif
#ifndef RQMC_TREE_NFR
#define RQMC_TREE_NFR 4
#endif

template <int NF, int B, int NFR, int BUN, int NH>
struct Tree {
  __host__ __device__ static constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
  __host__ __device__ static constexpr int K(int i) { return (B - 1) * ipow(B, NF - 1 - i); }  // s_w, w = NF-1-i
  __host__ __device__ static constexpr int runs(int i) { return ipow(B, i + 1); }              // runs per bundle
  __host__ __device__ static constexpr int jlo(int i) { return ipow(B, NF - 1 - i) - 1; }      // first A row
  static constexpr int J = ipow(B, NF) - 1;                        // fine A rows
  static constexpr int CH = 4 / NFR;                               // column slices per group
  static constexpr int RWN = BUN / 8;                              // row warps (8 residues each)
  static constexpr int NGRP = B;                                   // warp groups: one per top-level run
  static constexpr int WARPS = NGRP * CH * RWN;
#ifdef RQMC_TREE_MINB
  static constexpr int MINB = RQMC_TREE_MINB;                      // A/B experiments: CTAs per SM
#else
  static constexpr int MINB = (8 + WARPS - 1) / WARPS;             // CTAs per SM for >= 8 warps
#endif
  static constexpr int XP = BUN == 8 ? 12 : (BUN == 16 ? 20 : kPad);  // X^red t-stride (conflict-free)
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int NV = 2 * NFR;                               // doubles per lane per node
  static constexpr int LEAVES = ipow(B, NF);
  static constexpr bool kRegAcc = (B == 2 && NF >= 3);             // register row sums (b = 2 bottom)
  static constexpr int CW = 32 * NH;                               // CTA column tile (NH passes of 32)
  static constexpr int AP = CW + 4;                                // A slab / root tile pitch
  static constexpr int ABUF = J * AP;                              // one A slab
  static constexpr int ROOT = 2 * ABUF;                            // root tiles
  static constexpr int XS = ROOT + 2 * BUN * AP;                   // X subtree
  static constexpr int XL = (B - 1) * ipow(B, NF) * XP;            // X per level
  static constexpr int ACC = XS + NF * XL;                         // rowacc [ch][leaf][t]
  static constexpr int ACCN = kRegAcc ? 0 : CH * LEAVES * BUN;
  static constexpr int SMEM = (ACC + ACCN) * 8;
};

struct TreeCtx {
  int grp, ch, wm, g, tg, t, cw, beff, c0;
  int64_t r0;
  int64_t ybase, ystride;  // Y row of this lane's residue (leaf run 0) and the step per leaf run
  const double* as;  // A slab of the current column tile
};

// S = Sp + X^red[run] A_w, compile-time K (DMMA k-steps of 4, DFMA remainder); xs, as: level bases.
template <int K, int NFR, int XP, int AP>
__device__ __forceinline__ void tree_step(const double* xs, const double* as, const TreeCtx& c,
                                          const double (&Sp)[2 * NFR], double (&S)[2 * NFR]) {
  static_assert(K >= 1, "");
  if constexpr (K >= 4) {
    constexpr int NS = K / 4;
    const double* ab = as + c.cw + c.g;
    double af = xs[c.tg * XP], bf[NFR];
#pragma unroll
    for (int cf = 0; cf < NFR; ++cf) bf[cf] = ab[c.tg * AP + cf * 8];
#pragma unroll
    for (int s = 0; s < NS; ++s) {  // fragments of step s+1 are loaded before step s's DMMAs issue
      double afn = 0.0, bfn[NFR];
#pragma unroll
      for (int cf = 0; cf < NFR; ++cf) bfn[cf] = 0.0;
      if (s + 1 < NS) {
        afn = xs[(4 * (s + 1) + c.tg) * XP];
#pragma unroll
        for (int cf = 0; cf < NFR; ++cf) bfn[cf] = ab[(4 * (s + 1) + c.tg) * AP + cf * 8];
      }
#pragma unroll
      for (int cf = 0; cf < NFR; ++cf) {
        if (s == 0) dmma_c(S[2 * cf], S[2 * cf + 1], af, bf[cf], Sp[2 * cf], Sp[2 * cf + 1]);
        else dmma_c(S[2 * cf], S[2 * cf + 1], af, bf[cf], S[2 * cf], S[2 * cf + 1]);
      }
      af = afn;
#pragma unroll
      for (int cf = 0; cf < NFR; ++cf) bf[cf] = bfn[cf];
    }
  }
#pragma unroll
  for (int kk = (K / 4) * 4; kk < K; ++kk) {
    const double x = xs[kk * XP];
#pragma unroll
    for (int cf = 0; cf < NFR; ++cf) {
      const double2 p = *reinterpret_cast<const double2*>(as + kk * AP + c.cw + cf * 8 + 2 * c.tg);
      if (K < 4 && kk == 0) {
        S[2 * cf] = fma(x, p.x, Sp[2 * cf]);
        S[2 * cf + 1] = fma(x, p.y, Sp[2 * cf + 1]);
      } else {
        S[2 * cf] = fma(x, p.x, S[2 * cf]);
        S[2 * cf + 1] = fma(x, p.y, S[2 * cf + 1]);
      }
    }
  }
}

// 2^(j/64), j = 0..63, correctly rounded (mpmath): the table of exp_t
__device__ __constant__ static const double kExp2Tab64[64] = {
1.0,
    1.0108892860517005,
    1.0218971486541166,
    1.0330248790212284,
    1.0442737824274138,
    1.0556451783605572,
    1.0671404006768237,
    1.0787607977571199,
    1.0905077326652577,
    1.102382583307841,
    1.1143867425958924,
    1.1265216186082418,
    1.1387886347566916,
    1.1511892299529827,
    1.1637248587775775,
    1.1763969916502812,
    1.189207115002721,
    1.202156731452703,
    1.215247359980469,
    1.22848053610687,
    1.241857812073484,
    1.255380757024691,
    1.2690509571917332,
    1.2828700160787783,
    1.2968395546510096,
    1.3109612115247644,
    1.3252366431597413,
    1.339667524053303,
    1.3542555469368927,
    1.3690024229745905,
    1.383909881963832,
    1.3989796725383112,
    1.4142135623730951,
    1.42961333839197,
    1.4451808069770467,
    1.460917794180647,
    1.4768261459394993,
    1.4929077282912648,
    1.5091644275934228,
    1.5255981507445384,
    1.5422108254079407,
    1.559004400237837,
    1.5759808451078865,
    1.593142151342267,
    1.6104903319492543,
    1.6280274218573478,
    1.645755478153965,
    1.6636765803267364,
    1.681792830507429,
    1.7001063537185235,
    1.718619298122478,
    1.7373338352737062,
    1.7562521603732995,
    1.7753764925265212,
    1.7947090750031072,
    1.8142521755003989,
    1.8340080864093424,
    1.8539791250833855,
    1.8741676341103,
    1.8945759815869656,
    1.9152065613971474,
    1.9360617934922943,
    1.9571441241754002,
    1.978456026387951
};

// exp(x) for the elementwise g = exp(p0 y) of C2, table-driven: x = (k / 2^TB) ln 2 + r with
// |r| <= ln 2 / 2^(TB+1), exp(x) = 2^(k >> TB) 2^((k & (2^TB - 1)) / 2^TB) e^r, the table in shared memory
// (etab), the power of two added to the exponent field of the high word.  k = rint(2^TB x / ln 2) by the
// 1.5 * 2^52 shifter (one DFMA + one DADD, k the low word); r by the two-part ln 2 (k ln2_hi exact:
// |k| < 2^21, ln2_hi has 32 significant bits).  TB = 11 (2048 entries, 16 KB; trees whose shared memory
// leaves room): |r| <= 1.7e-4, e^r by its degree-3 Taylor polynomial (truncation 3.4e-17): 8 fp64-pipe
// instructions; TB = 6 (64 entries): degree 5 (truncation < 4e-17), 10.  Both <= ~2 ulp.
// exp_core has no range handling (valid for |x| <= 700).
template <int TB>
__device__ __forceinline__ double exp_core(double x, const double* etab) {
  static_assert(TB == 6 || TB == 11, "");
  constexpr double kShift = 6755399441055744.0;                    // 1.5 * 2^52
  constexpr double kInv = TB == 11 ? 2954.639443740597 : 92.33248261689366;              // 2^TB / ln 2
  constexpr double kHi = TB == 11 ? 0.00033845077166461124 : 0.01083042469326756;        // ln2_hi / 2^TB
  constexpr double kLo = TB == 11 ? 9.317455709329042e-14 : 2.9815858269852933e-12;      // ln2_lo / 2^TB
  const double t = fma(x, kInv, kShift);
  const double kd = t - kShift;
  const int k = __double2loint(t);
  double r = fma(kd, -kHi, x);
  r = fma(kd, -kLo, r);
  double p;
  if constexpr (TB == 11) {
    p = fma(r, 1.0 / 6.0, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
  } else {
    p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
  }
  const double v = etab[k & ((1 << TB) - 1)] * p;
  return __hiloint2double(__double2hiint(v) + ((k >> TB) << 20), __double2loint(v));
}
// |x| > 700 or NaN, on the high word (the range exp_core does not handle)
__device__ __forceinline__ bool exp_out_of_range(double x) {
  return (unsigned)(__double2hiint(x) & 0x7fffffff) > 0x4085e000u;
}
// exp_core with the range handling: |x| > 700 is clamped (exp(+-700); the fused kernels' g = exp(p0 y)
// does not reproduce overflow to inf or underflow to 0 beyond that, include/rqmc.h), NaN propagates
// (integer selects on the bits of x, branch-free)
template <int TB>
__device__ __forceinline__ double exp_t(double x, const double* etab) {
  const long long e = __double_as_longlong(exp_core<TB>(x, etab));
  const long long xb = __double_as_longlong(x), ab = xb & 0x7fffffffffffffffLL;
  const long long sat = xb < 0 ? 0x00d14f2b0fb9307fLL : 0x7f0d945df4f8ec8eLL;   // exp(-700) / exp(700)
  const long long big = ab > 0x7ff0000000000000LL ? xb : sat;
  return __longlong_as_double(ab > 0x4085e00000000000LL ? big : e);
}

// lane-local sum of g over one leaf node's NV values (reading C-17: 1 identity, 2 exp(p0 y), 3 y^2)
// (g = exp: exp_core per value and one warp vote per node; a warp that saw |p0 y| > 700 or a NaN
// recomputes the node with exp_t's range handling -- identical bits for the in-range values.  Range
// selects on every value had cost 9 of C2's 36 instructions per output.)
template <int G, int NV, int TB>
__device__ __forceinline__ double gsum(const double (&S)[NV], double p0, const double* etab) {
  if constexpr (G == 2) {
#if RQMC_FAST_EXP
    double x = p0 * S[0];
    bool bad = exp_out_of_range(x);
    double v = exp_core<TB>(x, etab);
#pragma unroll
    for (int e = 1; e < NV; ++e) {
      x = p0 * S[e];
      bad |= exp_out_of_range(x);
      v += exp_core<TB>(x, etab);
    }
    if (__any_sync(0xffffffffu, bad)) {
      v = exp_t<TB>(p0 * S[0], etab);
#pragma unroll
      for (int e = 1; e < NV; ++e) v += exp_t<TB>(p0 * S[e], etab);
    }
#else
    double v = exp(p0 * S[0]);
#pragma unroll
    for (int e = 1; e < NV; ++e) v += exp(p0 * S[e]);
#endif
    return v;
  } else if constexpr (G == 3) {
    double v = S[0] * S[0];
#pragma unroll
    for (int e = 1; e < NV; ++e) v = fma(S[e], S[e], v);
    return v;
  } else if constexpr (NV == 8) {
    return ((S[0] + S[1]) + (S[2] + S[3])) + ((S[4] + S[5]) + (S[6] + S[7]));
  } else {
    static_assert(NV == 4, "");
    return (S[0] + S[1]) + (S[2] + S[3]);
  }
}

template <bool STY, int NFR>
__device__ __forceinline__ void tree_store(const FineArgs& a, const double (&S)[2 * NFR], int j, const TreeCtx& c) {
  if constexpr (STY) {
    if (c.t < c.beff) {
      double* yr = a.Y + (c.ybase + (int64_t)j * c.ystride) * a.ldy;
#pragma unroll
      for (int cf = 0; cf < NFR; ++cf) {
        const int col = c.c0 + c.cw + cf * 8 + 2 * c.tg;
        if (col < a.tau) RQMC_DCHECK(yr + col, col + 1 < a.tau ? 16 : 8);
        if (col + 1 < a.tau) {
          if (a.y_vec) *reinterpret_cast<double2*>(yr + col) = make_double2(S[2 * cf], S[2 * cf + 1]);
          else { yr[col] = S[2 * cf]; yr[col + 1] = S[2 * cf + 1]; }
        } else if (col < a.tau) {
          yr[col] = S[2 * cf];
        }
      }
    }
  }
}

template <int NF, int B, int G, bool STY, int NFR, int BUN, int NH>
struct TreeRun {
  using T = Tree<NF, B, NFR, BUN, NH>;
  static constexpr int NV = T::NV;
  static constexpr bool kB2 = (B == 2 && NF >= 3);
  static constexpr bool kRegAcc = T::kRegAcc && G > 0;
  static constexpr int I2 = NF - 3;                                // the K = 4 level of the b = 2 bottom
  static constexpr int NQ = (I2 <= 0) ? 1 : 2;                     // K = 4 nodes per bottom block
  static constexpr int NBAT = (I2 <= 0) ? 1 : T::ipow(2, I2 - 1);  // bottom blocks per warp and tile
  static constexpr int RW = NQ;                                    // leaf row sums a lane keeps per block
  static constexpr int NACC = kRegAcc ? NBAT * RW : 1;
  static constexpr int K1 = (B == 2 && NF >= 2) ? T::K(NF - 2) : 0;  // the K = 2 level (b = 2)
  // exp table bits (g = exp): 64 entries.  The 2048-entry table (16 KB, degree-3 polynomial: 8 instead of
  // 10 fp64 instructions) measured slower on C2 (fine 35.3 -> 38.0 us, C2 x 64 1.61 -> 1.69 ms): random
  // lookups into 16 KB hit more shared-memory bank conflicts than into 512 B (RQMC_EXP_TB=11 to A/B)
  static constexpr int TB = (RQMC_EXP_TB == 11 && G == 2 && T::SMEM + 2048 * 8 <= 112 * 1024) ? 11 : 6;

  const FineArgs& a;
  const TreeCtx& c;
  double a0[T::K(NF - 1) <= 2 ? T::K(NF - 1) : 1][NV];  // leaf A values (K <= 2: DFMA leaves)
  double a1[K1 == 2 ? 2 : 1][NV];                       // A values of the K = 2 level (DFMA)
  double b4[RQMC_CACHE_B4 && kB2 ? NFR : 1];            // B fragments of the K = 4 level (one DMMA k-step)
  double racc[NACC];                                    // row sums sum_c g(y_kc) of this lane's leaf rows
  const double* etab = nullptr;                         // g = exp: 2^(j/2^TB) table in shared memory

  __device__ __forceinline__ TreeRun(const FineArgs& a_, const TreeCtx& c_) : a(a_), c(c_) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) racc[i] = 0.0;
  }

  __device__ __forceinline__ const double* xs(int i, int j) const {
    return fsm + T::XS + i * T::XL + j * T::K(i) * T::XP + c.t;
  }
  __device__ __forceinline__ const double* as(int i) const { return c.as + T::jlo(i) * T::AP; }

  // S = Sp + X^red_w[run j] A_w for the K = 2 level (b = 2): cached A values, DFMA
  __device__ __forceinline__ void step_k2(const double (&Sp)[NV], int i, int j, double (&S)[NV]) const {
    const double x0 = xs(i, j)[0], x1 = xs(i, j)[T::XP];
#pragma unroll
    for (int e = 0; e < NV; ++e) S[e] = fma(x1, a1[1][e], fma(x0, a1[0][e], Sp[e]));
  }
  template <int I>
  __device__ __forceinline__ void step(const double (&Sp)[NV], int j, double (&S)[NV]) const {
    if constexpr (B == 2 && T::K(I) == 2) step_k2(Sp, I, j, S);
    else tree_step<T::K(I), NFR, T::XP, T::AP>(xs(I, j), as(I), c, Sp, S);
  }

  // leaves of parent run jp (level NF-1), generic shapes: Y store, g sums, smem rowacc[ch][leaf][t]
  __device__ __forceinline__ void leaves(const double (&Sp)[NV], int jp) {
    constexpr int I = NF - 1, KL = T::K(I), RP = T::runs(I) / B;
    double* acc = fsm + T::ACC + c.ch * (T::LEAVES * BUN) + c.t;
    double v[B], pre[B];
    if constexpr (G > 0) {
#pragma unroll
      for (int q = 0; q < B; ++q) pre[q] = acc[(jp + q * RP) * BUN];
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int j = jp + q * RP;
      double Y[NV];
      if constexpr (KL <= 2) {
        const double* x = xs(I, j);
        const double x0 = x[0];
#pragma unroll
        for (int e = 0; e < NV; ++e) Y[e] = fma(x0, a0[0][e], Sp[e]);
        if constexpr (KL == 2) {
          const double x1 = x[T::XP];
#pragma unroll
          for (int e = 0; e < NV; ++e) Y[e] = fma(x1, a0[KL - 1][e], Y[e]);
        }
      } else {
        tree_step<KL, NFR, T::XP, T::AP>(xs(I, j), as(I), c, Sp, Y);
      }
      tree_store<STY, NFR>(a, Y, j, c);
      if constexpr (G > 0) v[q] = gsum<G, NV, TB>(Y, a.fp0, etab);
    }
    if constexpr (G > 0) {
#pragma unroll
      for (int q = 0; q < B; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 1);
#pragma unroll
      for (int q = 0; q < B; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 2);
      if (c.tg == 0) {
#pragma unroll
        for (int q = 0; q < B; ++q) acc[(jp + q * RP) * BUN] = pre[q] + v[q];
      }
    }
  }

  // the K = 4 level of the b = 2 bottom: one DMMA k-step, B fragments cached per tile (RQMC_CACHE_B4)
  __device__ __forceinline__ void step4(const double* x, const double (&Sp)[NV], double (&S)[NV]) const {
    if constexpr (RQMC_CACHE_B4 && kB2) {
      const double af = x[c.tg * T::XP];
#pragma unroll
      for (int cf = 0; cf < NFR; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, b4[cf], Sp[2 * cf], Sp[2 * cf + 1]);
    } else {
      tree_step<4, NFR, T::XP, T::AP>(x, as(I2), c, Sp, S);
    }
  }

  // b = 2 bottom (levels K = 4, 2, 1 below the parent tile Sp, bottom block number P of this warp):
  // the NQ level-(NF-3) nodes, their level-(NF-2) tiles and all 4 NQ leaves are formed first; then one
  // transpose-reduce over the 4 lanes of each row leaves lane tg with the column-slice sums of the
  // leaves 2 tg, 2 tg + 1 (NQ = 2; leaf tg for NQ = 1), accumulated in registers.
  template <int P>
  __device__ __forceinline__ void bottom_b2(const double (&Sp)[NV], int jp) {
    bottom_nodes<P, 0, NQ>(Sp, jp);
  }

  // NN K = 4 nodes starting at node N0 of the bottom block; lane tg ends with the column-slice sums of
  // NN of the 4 NN leaves, accumulated into racc[P RW + N0 + i], i < NN
  template <int P, int N0, int NN>
  __device__ __forceinline__ void bottom_nodes(const double (&Sp)[NV], int jp) {
    constexpr int I1 = NF - 2, I0 = NF - 1;
    constexpr int RP2 = (I2 == 0) ? 1 : T::runs(I2) / 2, RP1 = T::runs(I1) / 2, RP0 = T::runs(I0) / 2;
    constexpr int NL = 4 * NN;
    int jl[NL];
    double v[NL];
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      const int q2 = (I2 == 0) ? c.grp : N0 + n;
      const int j2 = jp + q2 * RP2;
#pragma unroll
      for (int l = 0; l < 4; ++l) jl[4 * n + l] = j2 + (l >> 1) * RP1 + (l & 1) * RP0;
    }
#pragma unroll
#if RQMC_S2_FIRST
    // all K = 4 nodes' DMMAs issue first: node n+1's tensor work overlaps node n's DFMA work
    double S2a[NN][NV];
#pragma unroll
    for (int n = 0; n < NN; ++n) step4(xs(I2, jl[4 * n]), Sp, S2a[n]);
#endif
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      const int j2 = jl[4 * n];
#if RQMC_S2_FIRST
      const double (&S2)[NV] = S2a[n];
#else
      double S2[NV];
      step4(xs(I2, j2), Sp, S2);
#endif
#if RQMC_S1_FIRST
      double S1a[2][NV];
#pragma unroll
      for (int h = 0; h < 2; ++h) step_k2(S2, I1, j2 + h * RP1, S1a[h]);
#endif
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#if RQMC_S1_FIRST
        const double (&S1)[NV] = S1a[h];
#else
        double S1[NV];
        step_k2(S2, I1, j2 + h * RP1, S1);
#endif
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int l = 4 * n + 2 * h + q;
          const double x0 = xs(I0, jl[l])[0];
          double Y[NV];
#pragma unroll
          for (int e = 0; e < NV; ++e) Y[e] = fma(x0, a0[0][e], S1[e]);
          tree_store<STY, NFR>(a, Y, jl[l], c);
          if constexpr (G > 0) v[l] = gsum<G, NV, TB>(Y, a.fp0, etab);
        }
      }
    }
    if constexpr (G > 0) {
      // transpose-reduce: exchange halves with lane tg^2, then quarters with lane tg^1
      const bool hi1 = (c.tg & 2) != 0, hi0 = (c.tg & 1) != 0;
      double u[NL / 2];
#pragma unroll
      for (int i = 0; i < NL / 2; ++i) {
        const double keep = hi1 ? v[i + NL / 2] : v[i];
        const double send = hi1 ? v[i] : v[i + NL / 2];
        u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
#pragma unroll
      for (int i = 0; i < NL / 4; ++i) {
        const double keep = hi0 ? u[i + NL / 4] : u[i];
        const double send = hi0 ? u[i] : u[i + NL / 4];
        racc[P * RW + N0 + i] += keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
    }
  }

  // children at level I of the parent tile Sp (run jp); P = the parent's position among this warp's
  // level-(I-1) nodes (compile time, so register row sums are statically indexed)
  template <int I, int P>
  __device__ __forceinline__ void level(const double (&Sp)[NV], int jp) {
    if constexpr (kB2 && I == I2) {
      bottom_b2<P>(Sp, jp);
    } else if constexpr (I == NF - 1) {
      leaves(Sp, jp);
    } else if constexpr (I == 0) {
      for (int q = c.grp; q < B; q += T::NGRP) {  // top level: one run per warp group
        double S[NV];
        step<0>(Sp, q, S);
        level<1, 0>(S, q);
      }
    } else {
      level_children<I, P, 0>(Sp, jp);
    }
  }
  template <int I, int P, int Q>
  __device__ __forceinline__ void level_children(const double (&Sp)[NV], int jp) {
    if constexpr (Q < B) {
      const int j = jp + Q * (T::runs(I) / B);
      double S[NV];
      step<I>(Sp, j, S);
      level<I + 1, P * B + Q>(S, j);
      level_children<I, P, Q + 1>(Sp, jp);
    }
  }

  __device__ __forceinline__ void load_cache(double (&dst)[NV], const double* row) const {
#pragma unroll
    for (int cf = 0; cf < NFR; ++cf) {
      const double2 p = *reinterpret_cast<const double2*>(row + c.cw + cf * 8 + 2 * c.tg);
      dst[2 * cf] = p.x;
      dst[2 * cf + 1] = p.y;
    }
  }

  __device__ __forceinline__ void tile(const double (&Sroot)[NV]) {
    constexpr int KL = T::K(NF - 1);
    if constexpr (KL <= 2) {
#pragma unroll
      for (int q = 0; q < KL; ++q) load_cache(a0[q], as(NF - 1) + q * T::AP);
    }
    if constexpr (K1 == 2) {
#pragma unroll
      for (int q = 0; q < 2; ++q) load_cache(a1[q], as(NF - 2) + q * T::AP);
    }
    if constexpr (RQMC_CACHE_B4 && kB2) {
#pragma unroll
      for (int cf = 0; cf < NFR; ++cf) b4[cf] = as(I2)[c.tg * T::AP + c.cw + c.g + cf * 8];
    }
    level<0, 0>(Sroot, 0);
  }
};

// Phase clock (A/B builds with -DRQMC_TREE_CLOCK=1 only): thread 0 of CTA x records %globaltimer at
// entry, after the prologue, after each of the first 10 tiles and at the end into g_tree_clk[x][0..15]
// (tools/tree_clock.py reads it through rqmc_debug_tree_clock).
#ifndef RQMC_TREE_CLOCK
#define RQMC_TREE_CLOCK 0
#endif
#if RQMC_TREE_CLOCK
constexpr int kClkCtas = 8192, kClkSlots = 16;
__device__ unsigned long long g_tree_clk[kClkCtas * kClkSlots];
__device__ __forceinline__ void tree_clk(int slot) {
  if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < kClkCtas && slot < kClkSlots) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tree_clk[blockIdx.x * kClkSlots + slot] = t;
  }
}
#else
__device__ __forceinline__ void tree_clk(int) {}
#endif

// trees that end with finish_fsum (the a5 final reduction): the small b = 2 trees (C2's latency
// regime); the b = 3 trees (C4: one k_reduce launch is 3 us of 4.5 ms) keep their round-1 code
template <int NF, int B>
constexpr bool kFuseReduce = NF <= 4 && B == 2;
// programmatic launch with the early prologue (above): the same small trees (C2 / C1 regime); the
// larger trees keep plain stream order (parked CTAs measured slower on C4)
#ifndef RQMC_TREE_PDL
#define RQMC_TREE_PDL 1
#endif
template <int NF, int B>
constexpr bool kTreePdl = RQMC_TREE_PDL && kFuseReduce<NF, B>;

template <int NF, int B, int G, bool STY, int NFR, int BUN, int NH>
__global__ void __launch_bounds__(Tree<NF, B, NFR, BUN, NH>::THREADS, Tree<NF, B, NFR, BUN, NH>::MINB)
    k_fine_tree(const FineArgs a) {
  // Early prologue (the small b = 2 trees, launched programmatically after the checkpoint GEMM): the
  // X^red subtree is issued before the dependency wait -- k_gen wrote it before the GEMM chain, each of
  // whose kernels waits for its predecessor before it triggers, so k_gen has completed by the time this
  // grid launches; the root tile (the GEMM's R_c) is read after the wait.  No root (k_gen is the
  // predecessor itself): wait first.
  constexpr bool kEarly = kTreePdl<NF, B>;
  if constexpr (kEarly) {
    if (a.root == nullptr) pdl_wait();
  } else {
    pdl_enter();
  }
  tree_clk(0);
  using T = Tree<NF, B, NFR, BUN, NH>;
  using Run = TreeRun<NF, B, G, STY, NFR, BUN, NH>;
  constexpr int NT = T::THREADS, NW = T::WARPS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TreeCtx c;
  c.wm = warp % T::RWN;
  c.ch = (warp / T::RWN) % T::CH;
  c.grp = warp / (T::RWN * T::CH);
  c.g = lane >> 2;
  c.tg = lane & 3;
  c.t = c.wm * 8 + c.g;
  c.cw = c.ch * 8 * NFR;
  // tail split (b = 3 trees only, FineArgs::nsplit): CTAs past nfull take half a bundle's column tiles
  // (compile-time off for b = 2: the extra control flow measured 3.5 % slower on C5's fine kernel)
  constexpr bool kSplit = (B == 3) && (G > 0);
  int64_t bundle = blockIdx.x;
  int sidx = 0;
  bool split = false;
  if constexpr (kSplit) {
    split = a.nsplit > 1 && bundle >= a.nfull;
    if (split) {
      const int64_t k = bundle - a.nfull;
      bundle = a.nfull + (k >> 1);
      sidx = (int)(k & 1);
    }
  }
  c.r0 = bundle * BUN;
  c.beff = (int)((a.Mroot - c.r0) < BUN ? (a.Mroot - c.r0) : BUN);
  if constexpr (STY) {
    c.ybase = y_row(a, c.r0 + c.t);
    c.ystride = y_stride(a);
  }
  const int64_t rep = blockIdx.y;  // replica (batched randomisation): own X^red, root R and partials
  const double* __restrict__ root = a.root ? a.root + rep * a.rootrep : nullptr;

  // X^red of the subtree -> smem [level][run][q][t]: the bundle's rows of one run are 32 K contiguous
  // doubles in HBM, read coalesced by 8-byte cp.async and transposed on the way into smem
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    const int K = T::K(i), n = T::runs(i) * BUN * K;
    const double* src = a.lv[i].X + rep * a.xrep + c.r0 * (int64_t)K;
    double* dst = fsm + T::XS + i * T::XL;
    for (int e = tid; e < n; e += NT) {
      const int j = e / (BUN * K), r = e - j * (BUN * K), t = r / K, q = r - t * K;
      const bool ok = t < c.beff;
      cp_async8(dst + (j * K + q) * T::XP + t, ok ? src + (int64_t)j * a.Mroot * K + r : a.A, ok);
    }
  }
  cp_async_commit();
  if constexpr (kEarly) pdl_enter();   // the checkpoint GEMM's R_c is visible from here on
#if RQMC_TREE_CLOCK >= 2
  cp_async_wait<0>();   // phase split (clock builds only): X^red subtree landed
  tree_clk(12);
#endif
  if constexpr (G > 0 && !Run::kRegAcc)
    for (int e = tid; e < T::ACCN; e += NT) fsm[T::ACC + e] = 0.0;

  // column tile operands (cp.async, double buffer): A rows [0, J) x 32 columns and the root tile.
  // (One 256-byte cp.async.bulk per row completing on an mbarrier measured 2.1 ms slower on C5: the
  // 95 small bulk requests per tile serialise in the copy engine.)
  constexpr int CW = T::CW, AP = T::AP;
  const int ntiles = (a.tau + CW - 1) / CW;
  const int ct_lo = kSplit && split && sidx ? ntiles / 2 : 0, ct_hi = kSplit && split && !sidx ? ntiles / 2 : ntiles;
  // fast path (every full tile of a 16-byte-aligned A and root, full bundle): each thread's chunks are
  // fixed rows / columns, so addresses are base + compile-time multiples of a runtime stride
  constexpr int CPR = CW / 2;                               // 16-byte chunks per row
  constexpr int RPP = NT / CPR;                             // rows per pass of all threads
  constexpr int UA = (T::J + RPP - 1) / RPP, UR = (BUN + RPP - 1) / RPP;
  const bool fast = a.a_vec && root != nullptr && c.beff == BUN && (a.ldroot % 2) == 0 &&
                    ((uintptr_t)root % 16) == 0;
  const int fq = tid / CPR, fcc = (tid % CPR) * 2;
  const double* fa = a.A + (int64_t)fq * a.lda + fcc;
  const double* fr = root ? root + (c.r0 + fq) * a.ldroot + fcc : nullptr;
  const int fo = fq * AP + fcc;
  auto load_tile = [&](int buf, int c0) {
    double* as = fsm + buf * T::ABUF;
    double* rs = fsm + T::ROOT + buf * (BUN * AP);
    if (fast && c0 + CW <= a.tau) {
#pragma unroll
      for (int u = 0; u < UA; ++u)
        if (u + 1 < UA || fq + u * RPP < T::J)
          cp_async16(as + fo + u * RPP * AP, fa + (int64_t)u * RPP * a.lda + c0, true);
#pragma unroll
      for (int u = 0; u < UR; ++u)
        if (u + 1 < UR || fq + u * RPP < BUN)
          cp_async16(rs + fo + u * RPP * AP, fr + (int64_t)u * RPP * a.ldroot + c0, true);
      cp_async_commit();
      return;
    }
    if (a.a_vec) {
      for (int e = tid; e < T::J * CPR; e += NT) {
        const int q = e / CPR, cc = (e % CPR) * 2;
        const bool ok = c0 + cc < a.tau;
        cp_async16(as + q * AP + cc, ok ? a.A + (int64_t)q * a.lda + c0 + cc : a.A, ok);
      }
    } else {
      for (int e = tid; e < T::J * CW; e += NT) {
        const int q = e / CW, cc = e % CW;
        const bool ok = c0 + cc < a.tau;
        cp_async8(as + q * AP + cc, ok ? a.A + (int64_t)q * a.lda + c0 + cc : a.A, ok);
      }
    }
    for (int e = tid; e < BUN * CPR; e += NT) {
      const int t = e / CPR, cc = (e % CPR) * 2;
      const bool row_ok = root != nullptr && t < c.beff;
      const double* src = root + (c.r0 + t) * a.ldroot + c0 + cc;
      if (c0 + cc + 1 < a.tau || !row_ok) {
        cp_async16(rs + t * AP + cc, row_ok ? src : a.A, row_ok);
      } else {
        cp_async8(rs + t * AP + cc, row_ok && c0 + cc < a.tau ? src : a.A, row_ok && c0 + cc < a.tau);
        cp_async8(rs + t * AP + cc + 1, a.A, false);
      }
    }
    cp_async_commit();
  };

  Run run(a, c);
  if constexpr (G == 2) {   // exp's table, visible after the barrier below
    __shared__ double etab[1 << Run::TB];
    if constexpr (Run::TB == 11) {
      for (int i = tid; i < 2048; i += NT) etab[i] = kExp2Tab2048[i];
    } else {
      if (tid < 64) etab[tid] = kExp2Tab64[tid];
    }
    run.etab = etab;
  }
#if RQMC_TREE_CLOCK >= 2
  tree_clk(13);
#endif
  load_tile(ct_lo & 1, ct_lo * CW);
  cp_async_wait<0>();  // X^red subtree and the first tile resident
  __syncthreads();
  tree_clk(1);
  const int cw0 = c.cw;
  for (int ct = ct_lo; ct < ct_hi; ++ct) {
    c.c0 = ct * CW;
    c.as = fsm + (ct & 1) * T::ABUF;
    if (ct + 1 < ct_hi) load_tile((ct + 1) & 1, (ct + 1) * CW);  // buffer freed by the last barrier
#pragma unroll 1
    for (int h = 0; h < NH; ++h) {   // NH passes of 32 columns per barrier interval
      c.cw = cw0 + 32 * h;
      double Sroot[T::NV];
      run.load_cache(Sroot, fsm + T::ROOT + (ct & 1) * (BUN * AP) + c.t * AP);
      run.tile(Sroot);
    }
    cp_async_wait<0>();
    __syncthreads();  // tile ct + 1 landed and visible; buffers (ct & 1) free for tile ct + 2
    if (ct - ct_lo < 10) tree_clk(2 + ct - ct_lo);   // slots 2..11 (12, 13: CLOCK=2 sub-phases; 15: end)
  }

  if constexpr (G > 0) {
    // padded columns (>= tau) hold y = 0 exactly: g(0) = 0 except g = exp, which added exp(0) = 1
    const double pad = (G == 2) ? (double)(ntiles * CW - a.tau) : 0.0;
    double part = 0.0;
    // split halves park their complete-over-slices row sums in scratch (row slot idx, same mapping in
    // both halves); the second half to finish combines them in fixed order (half 0 + half 1)
    constexpr int SCR = T::LEAVES * BUN;
    double* scr = (kSplit && split) ? a.rscr + rep * a.partrep + (bundle - a.nfull) * 2 * SCR : nullptr;
    auto use = [&](int idx, double rs) {
      if (kSplit && split) { RQMC_DCHECK(scr + sidx * SCR + idx, 8); scr[sidx * SCR + idx] = rs; }
      else part += f_of_mean(a, (rs - pad) / a.tau);
    };
    if constexpr (Run::kRegAcc) {
      // column-slice partial row sums -> complete row sums: slices ch > 0 park theirs in smem (the
      // X region is free after the last tile's barrier), slice 0 adds them in fixed order
      constexpr int NA = Run::NACC;
      double* park = fsm + T::XS + ((c.grp * T::RWN + c.wm) * 32 + lane) * NA;
      constexpr int PS = T::NGRP * T::RWN * 32 * NA;   // one column slice's parked sums
      if (c.ch > 0) {
#pragma unroll
        for (int i = 0; i < NA; ++i) park[(c.ch - 1) * PS + i] = run.racc[i];
      }
      if constexpr (T::CH > 1) __syncthreads();
      if (c.ch == 0 && c.t < c.beff) {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
          double rs = run.racc[i];
#pragma unroll
          for (int h = 1; h < T::CH; ++h) rs += park[(h - 1) * PS + i];
          use(((c.grp * T::RWN + c.wm) * 32 + lane) * NA + i, rs);
        }
      }
    } else {
      for (int e = tid; e < T::LEAVES * BUN; e += NT) {
        const int t = e % BUN;
        if (t >= c.beff) continue;
        double rs = fsm[T::ACC + e];
#pragma unroll
        for (int h = 1; h < T::CH; ++h) rs += fsm[T::ACC + h * (T::LEAVES * BUN) + e];
        use(e, rs);
      }
    }
    if constexpr (kSplit) {
      if (split) {
        __shared__ int s_last;
        unsigned int* cnt = a.rcnt + rep * 2 * a.partrep + (bundle - a.nfull);
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(cnt, 1u) == 1u;
        __syncthreads();
        if (!s_last) return;          // the other half finishes the bundle
        __threadfence();
        for (int e = tid; e < T::LEAVES * BUN; e += NT)
          if (e % BUN < c.beff) {
            const double rs = __ldcg(scr + e) + __ldcg(scr + SCR + e);
            part += f_of_mean(a, (rs - pad) / a.tau);
          }
        if (tid == 0) *cnt = 0u;      // ready for the next call (k_gen zeroes the counters as well)
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __shared__ double red[NW];
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t += red[w];
      RQMC_DCHECK(a.partial + rep * a.partrep + bundle, 8);
      a.partial[rep * a.partrep + bundle] = t;
    }
    // (small trees only: in the NF >= 5 trees the extra code perturbs ptxas's allocation of the hot loop
    // -- C5 fine 16.9 -> 18.4 ms -- where one k_reduce launch is 0.01 % of the step)
    if constexpr (kFuseReduce<NF, B>) finish_fsum<NT>(a, rep, (a.Mroot + BUN - 1) / BUN);
  }
  tree_clk(15);
}

// residues per CTA: b = 3 trees run 3 warp groups (one per top-level run; 2 groups split the 3 runs
// 2:1) of one row warp each, 8-residue bundles, 3+ CTAs per SM
template <int NF, int B>
constexpr int tree_bundle() { return B == 3 ? 8 : RQMC_TREE_BUNDLE; }
// fragments per warp: b = 3 trees (C4: Y stored, HBM-bound) run 8 warps of 8 x 16 columns at <= 128
// registers (fine 3.49 -> 3.30 ms); b = 2 trees keep 4 fragments (NFR = 2 measured slower: C3 fine
// 0.576 -> 0.701 ms, C2 45 -> 49 us)
template <int NF, int B>
constexpr int tree_nfr() { return B == 3 ? 2 : RQMC_TREE_NFR; }
// 64-column CTA tiles (two 32-column passes per barrier interval) when the doubled A slab still allows
// two CTAs per SM: small trees (C4's b = 3, NF = 3) spend their time in per-tile barriers and loads
template <int NF, int B>
constexpr int tree_passes() {
  return (RQMC_TREE_WIDE && Tree<NF, B, tree_nfr<NF, B>(), RQMC_TREE_BUNDLE, 2>::SMEM <= 100 * 1024) ? 2 : 1;
}

// Tail split (b = 3 trees with f): when the fine grid's last wave would be at most half full, its
// bundles run as two CTAs over half the column tiles each.  Returns the first split bundle (nbt when
// nothing splits).  The decision depends only on the bundle count and on the kernel's occupancy on
// kSplitSMs = 148 SMs (a constant, not the device's SM count), so a given binary splits -- and sums --
// identically on every device it runs on, and a replica of a batch sums like a single run.
constexpr int kSplitSMs = 148;
template <int NF, int B, int G, bool STY>
static int64_t tree_split_first(const FineArgs& a, int64_t nbt) {
  constexpr int NFR = tree_nfr<NF, B>(), BUN = tree_bundle<NF, B>(), NH = tree_passes<NF, B>();
  using T = Tree<NF, B, NFR, BUN, NH>;
  if constexpr (B == 3 && G > 0 && T::SMEM <= 227 * 1024) {
    static const bool no_split = [] { const char* v = std::getenv("RQMC_NO_SPLIT"); return v && *v && *v != '0'; }();
    const int ntiles = (a.tau + T::CW - 1) / T::CW;
    if (no_split || !a.rscr || ntiles < 2) return nbt;
    static const int64_t slots = [] {
      int occ = 0;
      if (set_smem_once(k_fine_tree<NF, B, G, STY, NFR, BUN, NH>, T::SMEM) != cudaSuccess ||
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fine_tree<NF, B, G, STY, NFR, BUN, NH>, T::THREADS,
                                                        T::SMEM) != cudaSuccess) {
        cudaGetLastError();
        occ = 0;   // no device (host-only inspection): no split
      }
      return (int64_t)occ * kSplitSMs;
    }();
    // RQMC_FORCE_SPLIT=1 (tests): split every bundle, so small problems exercise the combine path
    const char* fv = std::getenv("RQMC_FORCE_SPLIT");
    const bool force = fv && *fv && *fv != '0';
    const int64_t tail = force ? nbt : (slots > 0 && nbt >= slots) ? nbt % slots : 0;
    if (tail > 0 && (force || 2 * tail <= slots) && tail <= a.ncnt && tail * 2 * (int64_t)T::LEAVES * BUN <= a.rscr_cap)
      return nbt - tail;
  }
  return nbt;
}

template <int NF, int B, int G, bool STY>
static cudaError_t launch_tree_t(const FineArgs& a, int64_t nb, int nrep, cudaStream_t st, int64_t* nparts) {
  constexpr int NFR = tree_nfr<NF, B>(), BUN = tree_bundle<NF, B>(), NH = tree_passes<NF, B>();
  using T = Tree<NF, B, NFR, BUN, NH>;
  if constexpr (T::SMEM > 227 * 1024) {
    return cudaErrorNotSupported;
  }
  // A/B experiments only: RQMC_FINE_SMEM_KB pads the dynamic shared memory (fewer fine CTAs per SM,
  // e.g. to leave room for concurrent GEMM CTAs of the residue-chunk pipeline)
  static const int pad_kb = [] { const char* v = std::getenv("RQMC_FINE_SMEM_KB"); return v && *v ? std::atoi(v) : 0; }();
  const int smem = std::max<int>(T::SMEM, pad_kb * 1024);
  cudaError_t e = set_smem_once(k_fine_tree<NF, B, G, STY, NFR, BUN, NH>, smem);
  if (e != cudaSuccess) return e;
  const int64_t nbt = (a.Mroot + BUN - 1) / BUN;   // bundles of BUN residues (partials written)
  if (nbt > 4 * nb) return cudaErrorInvalidValue;   // workspace holds 4 nb partials per replica
  *nparts = (kFuseReduce<NF, B> && a.fsum) ? 0 : nbt;   // 0: the kernel wrote the f-sum itself
  FineArgs b = a;
  b.nfull = tree_split_first<NF, B, G, STY>(a, nbt);
  b.nsplit = b.nfull < nbt ? 2 : 1;
  const int64_t grid = b.nfull + (nbt - b.nfull) * b.nsplit;
  return launch_k(k_fine_tree<NF, B, G, STY, NFR, BUN, NH>, dim3((unsigned)grid, (unsigned)nrep), dim3(T::THREADS),
                  (size_t)smem, st, kTreePdl<NF, B>, b);
}

// Does the fine level table have the compile-time shape Tree<NF, B> (X^red rows dense, ldx = K)?
template <int NF, int B>
static bool tree_matches(const FineArgs& a) {
  using T = Tree<NF, B, tree_nfr<NF, B>(), tree_bundle<NF, B>(), 1>;
  if (a.NF != NF) return false;
  for (int i = 0; i < NF; ++i) {
    const FineLevel& L = a.lv[i];
    if (L.K != T::K(i) || L.fan != B || L.runs != T::runs(i) || L.j_lo != T::jlo(i) || L.ldx != L.K) return false;
  }
  return true;
}

template <int NF, int B>
static cudaError_t launch_tree_g(const FineArgs& a, int64_t nb, int nrep, cudaStream_t st, int64_t* np) {
  const bool sty = a.Y != nullptr;
  switch (a.fk) {
    case -1: return launch_tree_t<NF, B, 0, true>(a, nb, nrep, st, np);
    case 1: return sty ? launch_tree_t<NF, B, 2, true>(a, nb, nrep, st, np) : launch_tree_t<NF, B, 2, false>(a, nb, nrep, st, np);
    case 2: return sty ? launch_tree_t<NF, B, 3, true>(a, nb, nrep, st, np) : launch_tree_t<NF, B, 3, false>(a, nb, nrep, st, np);
    default: return sty ? launch_tree_t<NF, B, 1, true>(a, nb, nrep, st, np) : launch_tree_t<NF, B, 1, false>(a, nb, nrep, st, np);
  }
}

// Which compile-time tree the fine level table matches: 10 NF + B, or 0 (none / nothing to consume).
// (No 7-level tree: the planner's shared-memory bound never fuses 7 levels of the log_2 shape.)
// Host only; the single source of the dispatch decision (launch_tree and describe_fine).
int tree_select(const FineArgs& a) {
  if (a.Y == nullptr && a.fk < 0) return 0;
  if (tree_matches<6, 2>(a)) return 62;
  if (tree_matches<5, 2>(a)) return 52;
  if (tree_matches<4, 2>(a)) return 42;
  if (tree_matches<3, 2>(a)) return 32;
  if (tree_matches<2, 2>(a)) return 22;
#if RQMC_TREE43   // A/B builds only: four fused b = 3 levels (C4 with its level-3 GEMM folded in)
  if (tree_matches<4, 3>(a)) return 43;
#endif
  if (tree_matches<3, 3>(a)) return 33;
  if (tree_matches<2, 3>(a)) return 23;
  return 0;
}

// First tail-split bundle of the tree launch (and the bundle count), for describe_fine; -1: no tree.
template <int NF, int B>
static int64_t tree_split_g(const FineArgs& a, int64_t* nbt) {
  constexpr int BUN = tree_bundle<NF, B>();
  *nbt = (a.Mroot + BUN - 1) / BUN;
  const bool sty = a.Y != nullptr;
  switch (a.fk) {
    case -1: return *nbt;
    case 1: return sty ? tree_split_first<NF, B, 2, true>(a, *nbt) : tree_split_first<NF, B, 2, false>(a, *nbt);
    case 2: return sty ? tree_split_first<NF, B, 3, true>(a, *nbt) : tree_split_first<NF, B, 3, false>(a, *nbt);
    default: return sty ? tree_split_first<NF, B, 1, true>(a, *nbt) : tree_split_first<NF, B, 1, false>(a, *nbt);
  }
}
int64_t tree_split(const FineArgs& a, int64_t* nbt) {
  switch (tree_select(a)) {
#if RQMC_TREE43
    case 43: return tree_split_g<4, 3>(a, nbt);
#endif
    case 33: return tree_split_g<3, 3>(a, nbt);
    case 23: return tree_split_g<2, 3>(a, nbt);
    default: *nbt = 0; return 0;   // b = 2 trees never split
  }
}

// returns cudaErrorNotSupported when no compile-time tree matches
cudaError_t launch_tree(const FineArgs& a, int64_t nb, int nrep, cudaStream_t st, int64_t* np) {
  switch (tree_select(a)) {
    case 62: return launch_tree_g<6, 2>(a, nb, nrep, st, np);
    case 52: return launch_tree_g<5, 2>(a, nb, nrep, st, np);
    case 42: return launch_tree_g<4, 2>(a, nb, nrep, st, np);
    case 32: return launch_tree_g<3, 2>(a, nb, nrep, st, np);
    case 22: return launch_tree_g<2, 2>(a, nb, nrep, st, np);
#if RQMC_TREE43
    case 43: return launch_tree_g<4, 3>(a, nb, nrep, st, np);
#endif
    case 33: return launch_tree_g<3, 3>(a, nb, nrep, st, np);
    case 23: return launch_tree_g<2, 3>(a, nb, nrep, st, np);
    default: return cudaErrorNotSupported;
  }
}

#if RQMC_TREE_CLOCK
}  // namespace rqmc
extern "C" int rqmc_debug_tree_clock(unsigned long long* out, int n) {   // A/B builds only
  if (n > rqmc::kClkCtas * rqmc::kClkSlots) n = rqmc::kClkCtas * rqmc::kClkSlots;
  return (int)cudaMemcpyFromSymbol(out, rqmc::g_tree_clk, (size_t)n * sizeof(unsigned long long));
}
extern "C" int rqmc_debug_tree_clock_reset() {
  static unsigned long long z[rqmc::kClkCtas * rqmc::kClkSlots];
  return (int)cudaMemcpyToSymbol(rqmc::g_tree_clk, z, sizeof(z));
}
namespace rqmc {
#endif

#if RQMC_DEBUG
cudaError_t dbg_set_tree(const DbgRanges& r, cudaStream_t st) { return dbg_set_tu(r, st); }
#else
cudaError_t dbg_set_tree(const DbgRanges&, cudaStream_t) { return cudaSuccess; }
#endif

}  // namespace rqmc
