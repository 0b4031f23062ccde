// sm_100a kernels of the reduced QMC matrix product (PAPER.md P:n).
//
//   k_gen        a2  reduced points X^red_w of every level (lattice P:304-313 / net P:590-597,
//                    shift P:562, Phi^-1), written once per call; X (N x s) is never formed.
//   k_level_gemm a3+a4 coarse levels: R_w = tile(R_w') + X^red_w A_w (Alg. 2) as a
//                    DMMA.8x8x4 (mma.sync f64) GEMM, cp.async double-buffered smem tiles, the
//                    accumulator initialised from the parent rows r mod M_w' (the "tile").
//   k_fine<NF>   a3+a4+a5 the NF finest levels fused: one CTA owns a bundle of residues of the
//                    checkpoint level and walks its subtree depth-first (Alg. 2's recursion
//                    restricted to k = r (mod M_ckpt)); the partial sums of the path live in
//                    registers, X^red of the subtree in shared memory, A_w slabs double-buffered;
//                    the leaf rows x_k^T A are stored (Y) and/or reduced by f in the same pass.
//   k_reduce     a5  fixed-order reduction of the per-bundle f sums.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "rqmc_device.cuh"

namespace rqmc {

// S = Sp + X^red_w[run] A_w for one level with compile-time K (<= 0: runtime L.K)
// (paper Alg. 2 "tile(P_{I+1}) + X_I A_I").  xs: X^red of the run at this lane's row.
template <int KC>
__device__ __forceinline__ void level_step(const double* xs, const double* as, int Krt, const FineCtx& c,
                                           const double (&Sp)[8], double (&S)[8]) {
  const int K = KC > 0 ? KC : Krt;
  int kk = 0;
  if (K >= 4) {
    {
      const double af = xs[c.tg * kPad];
      const double* aq = as + c.tg * kPad + c.g;
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, aq[cf * 8], Sp[2 * cf], Sp[2 * cf + 1]);
    }
    kk = 4;
    if (kk + 4 <= K) {  // fragments of step k+4 are loaded before the DMMAs of step k issue
      double af = xs[(kk + c.tg) * kPad], bf[4];
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) bf[cf] = as[(kk + c.tg) * kPad + c.g + cf * 8];
      for (; kk + 8 <= K; kk += 4) {
        const double afn = xs[(kk + 4 + c.tg) * kPad];
        double bfn[4];
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) bfn[cf] = as[(kk + 4 + c.tg) * kPad + c.g + cf * 8];
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, bf[cf], S[2 * cf], S[2 * cf + 1]);
        af = afn;
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) bf[cf] = bfn[cf];
      }
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, bf[cf], S[2 * cf], S[2 * cf + 1]);
      kk += 4;
    }
  } else {
    const double x = xs[0];
#pragma unroll
    for (int cf = 0; cf < 4; ++cf) {
      const double2 p = *reinterpret_cast<const double2*>(as + cf * 8 + 2 * c.tg);
      S[2 * cf] = fma(x, p.x, Sp[2 * cf]);
      S[2 * cf + 1] = fma(x, p.y, Sp[2 * cf + 1]);
    }
    kk = 1;
  }
#pragma unroll
  for (; kk < K; ++kk) {  // K mod 4 remainder on the DFMA pipe, same fragment layout
    const double x = xs[kk * kPad];
#pragma unroll
    for (int cf = 0; cf < 4; ++cf) {
      const double2 p = *reinterpret_cast<const double2*>(as + kk * kPad + cf * 8 + 2 * c.tg);
      S[2 * cf] = fma(x, p.x, S[2 * cf]);
      S[2 * cf + 1] = fma(x, p.y, S[2 * cf + 1]);
    }
  }
}

// Compile-time description of the bottom NB fine levels (index 0 = coarsest of them).
template <int NB_, int F0, int K0, int F1, int K1, int F2, int K2>
struct Bot {
  static constexpr int NB = NB_;
  __host__ __device__ static constexpr int fan(int i) { return i == 0 ? F0 : (i == 1 ? F1 : F2); }
  __host__ __device__ static constexpr int k(int i) { return i == 0 ? K0 : (i == 1 ? K1 : K2); }
  __host__ __device__ static constexpr int kleaf() { return k(NB_ - 1); }
};
using BotNone = Bot<0, 0, 0, 0, 0, 0, 0>;
using BotB2 = Bot<3, 2, 4, 2, 2, 2, 1>;   // b = 2, w_j = floor(log2 j): K = 4, 2, 1, fans 2
using BotB2s = Bot<2, 2, 2, 2, 1, 0, 0>;  // b = 2, only two fine levels below: K = 2, 1
using BotB3 = Bot<2, 3, 6, 3, 2, 0, 0>;   // b = 3, w_j = floor(log3 j): K = 6, 2, fans 3

// Per-column-tile register cache of the bottom block: the leaf level's A values (K <= 2, used by
// DFMA), the B fragments of a K = 4 bottom level (one DMMA step), and the parent run counts.
template <class BT>
struct LeafCache {
  static constexpr int KL = BT::kleaf();
  static constexpr bool CL = BT::NB > 0 && KL <= 2;
  // non-leaf bottom levels with K <= 4 run as ONE DMMA k-step (zero-padded to 4 when K < 4):
  // their B fragments B[tg][g] = (tg < K ? A_w[tg][cf*8+g] : 0) are cached here
  __host__ __device__ static constexpr bool cached(int bl) { return bl < BT::NB - 1 && BT::k(bl) <= 4; }
  double v[CL ? KL : 1][8];
  double bk[BT::NB > 1 ? BT::NB - 1 : 1][4];
  int runs[3];
};


// Leaf level of the bottom block: F children of the parent tile Sp; Y store + g, batched row sums.
template <int NF, class BT, int G, bool STY>
__device__ __forceinline__ void bot_leaves(const FineArgs& a, const double (&Sp)[8], int jp, const FineCtx& c,
                                           const LeafCache<BT>& lc) {
  constexpr int BL = BT::NB - 1, I = NF - 1, F = BT::fan(BL), K = BT::k(BL);
  const FineLevel& L = a.lv[I];
  const int runs_parent = lc.runs[BL];
  double v[F], pre[F];
  if constexpr (G > 0 && I > 0) {  // prefetch this lane's row sums of the F leaves (hides LDS latency)
#pragma unroll
    for (int q = 0; q < F; ++q) pre[q] = fsm[a.acc_off + (jp + q * runs_parent) * kBundle + c.t];
  }
  auto leaf = [&](int q) {
    const int j = jp + q * runs_parent;
    const double* xs = fsm + L.xs_off + j * K * kPad + c.t;
    double S[8];
    if constexpr (K <= 2) {
      const double x0 = xs[0];
#pragma unroll
      for (int e = 0; e < 8; ++e) S[e] = fma(x0, lc.v[0][e], Sp[e]);
      if constexpr (K == 2) {
        const double x1 = xs[kPad];
#pragma unroll
        for (int e = 0; e < 8; ++e) S[e] = fma(x1, lc.v[1][e], S[e]);
      }
    } else {
      level_step<K>(xs, c.as + L.as_off, K, c, Sp, S);
    }
    store_leaf<STY>(a, S, j, c);
    if constexpr (G > 0) v[q] = gsum8<G>(S, a.fp0);
  };
  if constexpr (I == 0) {
    for (int q = c.grp; q < F; q += 2) leaf(q);
  } else {
#pragma unroll
    for (int q = 0; q < F; ++q) leaf(q);
  }
  if constexpr (G > 0) {
    if constexpr (I == 0) {  // (degenerate: leaf level is the top level) one leaf at a time
      for (int q = c.grp; q < F; q += 2) {
        double s = v[q];
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (c.tg == 0) fsm[a.acc_off + q * kBundle + c.t] += s;
      }
    } else {
#pragma unroll
      for (int q = 0; q < F; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 1);
#pragma unroll
      for (int q = 0; q < F; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 2);
      if (c.tg == 0) {
#pragma unroll
        for (int q = 0; q < F; ++q) fsm[a.acc_off + (jp + q * runs_parent) * kBundle + c.t] = pre[q] + v[q];
      }
    }
  }
}

template <int NF, int BL, class BT, int G, bool STY>
__device__ __forceinline__ void bot_level(const FineArgs& a, const double (&Sp)[8], int jp, const FineCtx& c,
                                          const LeafCache<BT>& lc) {
  if constexpr (BL == BT::NB - 1) {
    bot_leaves<NF, BT, G, STY>(a, Sp, jp, c, lc);
  } else {
    constexpr int I = NF - BT::NB + BL, F = BT::fan(BL), K = BT::k(BL);
    const FineLevel& L = a.lv[I];
    const int runs_parent = lc.runs[BL];
    auto child = [&](int q) {
      const int j = jp + q * runs_parent;
      double S[8];
      if constexpr (LeafCache<BT>::cached(BL)) {  // K <= 4: one DMMA step, B fragments cached
        const double af = (K == 4 || c.tg < K) ? fsm[L.xs_off + (j * K + c.tg) * kPad + c.t] : 0.0;
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, lc.bk[BL][cf], Sp[2 * cf], Sp[2 * cf + 1]);
      } else {
        level_step<K>(fsm + L.xs_off + j * K * kPad + c.t, c.as + L.as_off, K, c, Sp, S);
      }
      bot_level<NF, BL + 1, BT, G, STY>(a, S, j, c, lc);
    };
    if constexpr (I == 0) {
      for (int q = c.grp; q < F; q += 2) child(q);
    } else {
#pragma unroll
      for (int q = 0; q < F; ++q) child(q);
    }
  }
}

// Hand-scheduled bottom block for the hot shape BotB2 (levels K = 4, 2, 1 with fans 2, i.e. b = 2 and
// w_j = floor(log2 j)): one level-2 node -> 2 level-1 tiles -> 4 leaves.  All operand loads of the
// node are issued first, then the DMMAs (level 2, both level-1 tiles), then the 4 leaves' DFMA +
// g sums, then the interleaved row-sum shuffles -- so smem, DMMA, DFMA and SHFL latencies overlap
// inside one warp.  Same arithmetic (and rounding) as the generic template path.
template <int NF, int G, bool STY>
__device__ __forceinline__ void bot_b2(const FineArgs& a, const double (&S3)[8], int j3, const FineCtx& c,
                                       const LeafCache<BotB2>& lc) {
  const FineLevel& L2 = a.lv[NF - 3];
  const FineLevel& L1 = a.lv[NF - 2];
  const FineLevel& L0 = a.lv[NF - 1];
  const int r2 = lc.runs[0], r1 = lc.runs[1], r0 = lc.runs[2];
  // one level-2 node: loads, DMMAs (level 2 and both level-1 tiles), leaves -> per-leaf g sums v[]
  auto node = [&](int q2, int (&jl)[4], double (&v)[4], double (&pre)[4]) {
    const int j2 = j3 + q2 * r2;
    const int j1[2] = {j2, j2 + r1};
    jl[0] = j1[0]; jl[1] = j1[0] + r0; jl[2] = j1[1]; jl[3] = j1[1] + r0;
    const double x2 = fsm[L2.xs_off + (j2 * 4 + c.tg) * kPad + c.t];
    double x1[2], x0[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) x1[h] = c.tg < 2 ? fsm[L1.xs_off + (j1[h] * 2 + c.tg) * kPad + c.t] : 0.0;
#pragma unroll
    for (int l = 0; l < 4; ++l) x0[l] = fsm[L0.xs_off + jl[l] * kPad + c.t];
    if constexpr (G > 0) {
#pragma unroll
      for (int l = 0; l < 4; ++l) pre[l] = fsm[a.acc_off + jl[l] * kBundle + c.t];
    }
    double S2[8], S1[2][8];
#pragma unroll
    for (int cf = 0; cf < 4; ++cf) dmma_c(S2[2 * cf], S2[2 * cf + 1], x2, lc.bk[0][cf], S3[2 * cf], S3[2 * cf + 1]);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int cf = 0; cf < 4; ++cf)
        dmma_c(S1[h][2 * cf], S1[h][2 * cf + 1], x1[h], lc.bk[1][cf], S2[2 * cf], S2[2 * cf + 1]);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      double Y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) Y[e] = fma(x0[l], lc.v[0][e], S1[l >> 1][e]);
      store_leaf<STY>(a, Y, jl[l], c);
      if constexpr (G > 0) v[l] = gsum8<G>(Y, a.fp0);
    }
  };
  // row sums of a node's 4 leaves: butterfly over the 4 lanes of a row, then one store per row
  auto finish = [&](const int (&jl)[4], double (&v)[4], const double (&pre)[4]) {
    if constexpr (G > 0) {
#pragma unroll
      for (int l = 0; l < 4; ++l) v[l] += __shfl_xor_sync(0xffffffffu, v[l], 1);
#pragma unroll
      for (int l = 0; l < 4; ++l) v[l] += __shfl_xor_sync(0xffffffffu, v[l], 2);
      if (c.tg == 0) {
#pragma unroll
        for (int l = 0; l < 4; ++l) fsm[a.acc_off + jl[l] * kBundle + c.t] = pre[l] + v[l];
      }
    }
  };
  int jla[4], jlb[4];
  double va[4], vb[4], pa[4], pb[4];
  if (NF - 3 == 0) {  // the node level is the top fine level: one node per group
    node(c.grp, jla, va, pa);
    finish(jla, va, pa);
  } else {            // two sibling nodes, the first node's shuffles overlap the second's math
    node(0, jla, va, pa);
    node(1, jlb, vb, pb);
    finish(jla, va, pa);
    finish(jlb, vb, pb);
  }
}

template <int NF, class BT>
__device__ __forceinline__ void bot_dispatch(const FineArgs& a, const double (&Sp)[8], int jp, const FineCtx& c,
                                             const LeafCache<BT>& lc) {
  const bool sty = a.Y != nullptr;
  if constexpr (std::is_same<BT, BotB2>::value) {
    switch (a.fk) {
      case -1: sty ? bot_b2<NF, 0, true>(a, Sp, jp, c, lc) : bot_b2<NF, 0, false>(a, Sp, jp, c, lc); return;
      case 1: sty ? bot_b2<NF, 2, true>(a, Sp, jp, c, lc) : bot_b2<NF, 2, false>(a, Sp, jp, c, lc); return;
      case 2: sty ? bot_b2<NF, 3, true>(a, Sp, jp, c, lc) : bot_b2<NF, 3, false>(a, Sp, jp, c, lc); return;
      default: sty ? bot_b2<NF, 1, true>(a, Sp, jp, c, lc) : bot_b2<NF, 1, false>(a, Sp, jp, c, lc); return;
    }
  }
  switch (a.fk) {
    case -1: sty ? bot_level<NF, 0, BT, 0, true>(a, Sp, jp, c, lc) : bot_level<NF, 0, BT, 0, false>(a, Sp, jp, c, lc); break;
    case 1: sty ? bot_level<NF, 0, BT, 2, true>(a, Sp, jp, c, lc) : bot_level<NF, 0, BT, 2, false>(a, Sp, jp, c, lc); break;
    case 2: sty ? bot_level<NF, 0, BT, 3, true>(a, Sp, jp, c, lc) : bot_level<NF, 0, BT, 3, false>(a, Sp, jp, c, lc); break;
    default: sty ? bot_level<NF, 0, BT, 1, true>(a, Sp, jp, c, lc) : bot_level<NF, 0, BT, 1, false>(a, Sp, jp, c, lc); break;
  }
}

// Generic leaf consumption (runtime g / Y), used when the bottom shape is not specialised.
__device__ __forceinline__ void fine_consume(const FineArgs& a, const double (&S)[8], int j, const FineCtx& c) {
  if (a.Y) store_leaf<true>(a, S, j, c);
  if (a.fk >= 0) {
    double v = a.fk == 1 ? gsum8<2>(S, a.fp0) : (a.fk == 2 ? gsum8<3>(S, a.fp0) : gsum8<1>(S, a.fp0));
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (c.tg == 0) fsm[a.acc_off + j * kBundle + c.t] += v;
  }
}

// Upper fine levels: runtime fans / K, register stack; hands over to the bottom block.
template <int I, int NF, class BT>
__device__ __forceinline__ void fine_level(const FineArgs& a, const double (&Sp)[8], int jp, const FineCtx& c,
                                           const LeafCache<BT>& lc) {
  if constexpr (BT::NB > 0 && I == NF - BT::NB) {
    bot_dispatch<NF, BT>(a, Sp, jp, c, lc);
  } else if constexpr (I >= NF) {
    fine_consume(a, Sp, jp, c);
  } else {
    const FineLevel& L = a.lv[I];
    const int runs_parent = (I == 0) ? 1 : a.lv[I > 0 ? I - 1 : 0].runs;
    const int q0 = (I == 0) ? c.grp : 0, qs = (I == 0) ? 2 : 1;  // top level split over the 2 groups
    for (int qf = q0; qf < L.fan; qf += qs) {
      const int j = jp + qf * runs_parent;
      double S[8];
      level_step<0>(fsm + L.xs_off + j * L.K * kPad + c.t, c.as + L.as_off, L.K, c, Sp, S);
      fine_level<I + 1, NF, BT>(a, S, j, c, lc);
    }
  }
}

template <int NF, class BT>
__global__ void __launch_bounds__(kFineThreads, 1) k_fine(const FineArgs a) {
  pdl_enter();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  FineCtx c;
  c.grp = warp >> 2;
  c.wm = warp & 3;
  c.g = lane >> 2;
  c.tg = lane & 3;
  c.t = c.wm * 8 + c.g;
  c.r0 = (int64_t)blockIdx.x * kBundle;
  const int64_t rep = blockIdx.y;  // replica (batched randomisation): own X^red, root R and partials
  const double* __restrict__ root = a.root ? a.root + rep * a.rootrep : nullptr;
  c.beff = (int)((a.Mroot - c.r0) < kBundle ? (a.Mroot - c.r0) : kBundle);
  c.ybase = y_row(a, c.r0 + c.t);
  c.ystride = y_stride(a);

  // X^red of the subtree -> smem [run][q][t] (t stride kPad); global rows r0 + t + j Mroot, read
  // row-contiguously, written transposed.
  for (int i = 0; i < NF; ++i) {
    const FineLevel& L = a.lv[i];
    double* xs = fsm + L.xs_off;
    // lane = t (conflict-free smem stores), loop over (run, q) rows, 4 loads in flight per thread
    const int nrow = L.runs * L.K;
    const int t = tid & (kBundle - 1);
    const double* src = L.X + rep * a.xrep + (c.r0 + t) * L.ldx;
    for (int r = tid >> 5; r < nrow; r += 4 * (kFineThreads >> 5)) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = r + u * (kFineThreads >> 5);
        const int j = rr / L.K, q = rr - j * L.K;
        if (rr < nrow && t < c.beff) RQMC_DCHECK(src + (int64_t)j * a.Mroot * L.ldx + q, 8);
        v[u] = (rr < nrow && t < c.beff) ? src[(int64_t)j * a.Mroot * L.ldx + q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = r + u * (kFineThreads >> 5);
        if (rr < nrow) xs[rr * kPad + t] = v[u];
      }
    }
  }
  if (a.fk >= 0)
    for (int e = tid; e < a.leafruns * kBundle; e += kFineThreads) fsm[a.acc_off + e] = 0.0;

  // One column tile's operands, cp.async double buffer: the A slab of all fine levels [q][c] and the
  // root tile R_ckpt[t][c] (c stride kPad); zero-filled beyond tau / the bundle.
  auto load_tile = [&](int buf, int c0) {
    double* as = fsm + buf * a.as_stride;
    double* rs = fsm + a.root_off + buf * (kBundle * kPad);
    if (a.a_vec) {
      for (int i = 0; i < NF; ++i) {
        const FineLevel& L = a.lv[i];
        for (int e = tid; e < L.K * (kFineBN / 2); e += kFineThreads) {
          const int q = e / (kFineBN / 2), cc = (e % (kFineBN / 2)) * 2;
          const bool ok = c0 + cc < a.tau;
          const double* src = ok ? a.A + (int64_t)(L.j_lo + q) * a.lda + c0 + cc : a.A;
          cp_async16(as + L.as_off + q * kPad + cc, src, ok);
        }
      }
    } else {
      for (int i = 0; i < NF; ++i) {
        const FineLevel& L = a.lv[i];
        for (int e = tid; e < L.K * kFineBN; e += kFineThreads) {
          const int q = e / kFineBN, cc = e % kFineBN;
          const bool ok = c0 + cc < a.tau;
          const double* src = ok ? a.A + (int64_t)(L.j_lo + q) * a.lda + c0 + cc : a.A;
          cp_async8(as + L.as_off + q * kPad + cc, src, ok);
        }
      }
    }
    // root rows: ldroot even and c0 even -> 16B chunks; a chunk is valid iff its first column is
    // (tau may be odd: the second element of the last chunk is then masked by a scalar copy)
    for (int e = tid; e < kBundle * (kFineBN / 2); e += kFineThreads) {
      const int t = e / (kFineBN / 2), cc = (e % (kFineBN / 2)) * 2;
      const bool row_ok = root != nullptr && t < c.beff;
      const double* src = root + (c.r0 + t) * a.ldroot + c0 + cc;
      if (c0 + cc + 1 < a.tau || !row_ok) {
        cp_async16(rs + t * kPad + cc, row_ok ? src : a.A, row_ok);
      } else {  // last, odd column: copy one element, zero the other
        cp_async8(rs + t * kPad + cc, row_ok && c0 + cc < a.tau ? src : a.A, row_ok && c0 + cc < a.tau);
        cp_async8(rs + t * kPad + cc + 1, a.A, false);
      }
    }
    cp_async_commit();
  };

  const int ntiles = (a.tau + kFineBN - 1) / kFineBN;
  load_tile(0, 0);
  for (int ct = 0; ct < ntiles; ++ct) {
    c.c0 = ct * kFineBN;
    c.as = fsm + (ct & 1) * a.as_stride;
    if (ct + 1 < ntiles) {
      load_tile((ct + 1) & 1, (ct + 1) * kFineBN);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // operands of this tile (and X, rowacc on the first pass) visible
    double Sroot[8];
    {
      const double* rs = fsm + a.root_off + (ct & 1) * (kBundle * kPad) + c.t * kPad + 2 * c.tg;
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) {
        const double2 p = *reinterpret_cast<const double2*>(rs + cf * 8);
        Sroot[2 * cf] = p.x;
        Sroot[2 * cf + 1] = p.y;
      }
    }
    LeafCache<BT> lc;
#pragma unroll
    for (int bl = 0; bl < 3; ++bl) {
      const int I = NF - BT::NB + bl;
      lc.runs[bl] = (I <= 0 || bl >= BT::NB) ? 1 : a.lv[I - 1].runs;
    }
#pragma unroll
    for (int bl = 0; bl + 1 < BT::NB; ++bl) {
      if (LeafCache<BT>::cached(bl)) {
        const FineLevel& L = a.lv[NF - BT::NB + bl];
#pragma unroll
        for (int cf = 0; cf < 4; ++cf)
          lc.bk[bl][cf] = c.tg < BT::k(bl) ? c.as[L.as_off + c.tg * kPad + cf * 8 + c.g] : 0.0;
      }
    }
    if constexpr (BT::NB > 0 && BT::kleaf() <= 2) {
      const FineLevel& L = a.lv[NF - 1];
#pragma unroll
      for (int q = 0; q < BT::kleaf(); ++q)
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) {
          const double2 p = *reinterpret_cast<const double2*>(c.as + L.as_off + q * kPad + cf * 8 + 2 * c.tg);
          lc.v[q][2 * cf] = p.x;
          lc.v[q][2 * cf + 1] = p.y;
        }
    }
    if (NF > 0 || c.grp == 0) fine_level<0, NF, BT>(a, Sroot, 0, c, lc);
    __syncthreads();  // buffers (ct & 1) are refilled at iteration ct + 1
  }

  if (a.fk >= 0) {
    // F(tau^-1 sum_c g) per leaf row, then a fixed-order CTA reduction -> partial[bundle].
    // Padded columns (>= tau) hold y = 0 exactly: g(0) = 0 except g = exp, which added exp(0) = 1.
    const double pad = a.fk == 1 ? (double)(ntiles * kFineBN - a.tau) : 0.0;
    double part = 0.0;
    for (int e = tid; e < a.leafruns * kBundle; e += kFineThreads) {
      const int t = e % kBundle;
      if (t >= c.beff) continue;
      const double rs = fsm[a.acc_off + e] - pad;
      const double mean = rs / a.tau;
      double fv;
      switch (a.fk) {
        case 0: fv = exp(mean); break;
        case 1: fv = mean - a.fp1; fv = fv > 0.0 ? fv : 0.0; break;
        default: fv = mean; break;
      }
      part += fv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __shared__ double red[kFineThreads / 32];
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kFineThreads / 32; ++w) t += red[w];
      RQMC_DCHECK(a.partial + rep * a.partrep + blockIdx.x, 8);
      a.partial[rep * a.partrep + blockIdx.x] = t;
    }
    finish_fsum<kFineThreads>(a, rep, gridDim.x);
  }
}

template <int NF, class BT>
static cudaError_t launch_fine_t(const FineArgs& a, int64_t nb, int nrep, cudaStream_t st) {
  cudaError_t e = set_smem_once(k_fine<NF, BT>, a.smem_bytes);
  if (e != cudaSuccess) return e;
  return launch_k(k_fine<NF, BT>, dim3((unsigned)nb, (unsigned)nrep), dim3(kFineThreads), a.smem_bytes, st, true, a);
}

// Does the bottom of the fine level table match the compile-time shape BT?
template <class BT>
static bool bottom_matches(const FineArgs& a) {
  if (a.NF < BT::NB) return false;
  for (int i = 0; i < BT::NB; ++i) {
    const FineLevel& L = a.lv[a.NF - BT::NB + i];
    if (L.fan != BT::fan(i) || L.K != BT::k(i)) return false;
  }
  return true;
}

// bottom block of the general kernel: 0 BotNone, 1 BotB2, 2 BotB2s, 3 BotB3 (host; the dispatch decision)
static int bottom_select(const FineArgs& a) {
  if (a.NF >= 3 && bottom_matches<BotB2>(a)) return 1;
  if (a.NF >= 2 && bottom_matches<BotB2s>(a)) return 2;
  if (a.NF >= 2 && bottom_matches<BotB3>(a)) return 3;
  return 0;
}

template <int NF>
static cudaError_t launch_fine_n(const FineArgs& a, int64_t nb, int nrep, cudaStream_t st) {
  const int bs = bottom_select(a);
  if constexpr (NF >= 3)
    if (bs == 1) return launch_fine_t<NF, BotB2>(a, nb, nrep, st);
  if constexpr (NF >= 2) {
    if (bs == 2) return launch_fine_t<NF, BotB2s>(a, nb, nrep, st);
    if (bs == 3) return launch_fine_t<NF, BotB3>(a, nb, nrep, st);
  }
  return launch_fine_t<NF, BotNone>(a, nb, nrep, st);
}

cudaError_t launch_tree(const FineArgs& a, int64_t nb, int nrep, cudaStream_t st, int64_t* nparts);
int tree_select(const FineArgs& a);
int64_t tree_split(const FineArgs& a, int64_t* nbt);

static bool no_tree() { const char* e = std::getenv("RQMC_NO_TREE"); return e != nullptr && *e && *e != '0'; }

// The kernel template launch_fine picks for these arguments, e.g. "k_fine_tree<6,2,g=1,Y=0>" or
// "k_fine<4,BotB2>" (g: 0 none, 1 identity, 2 exp, 3 square; tests assert which branch they reach).
int describe_fine(const FineArgs& a, char* buf, size_t n) {
  const int g = a.fk < 0 ? 0 : (a.fk == 1 ? 2 : (a.fk == 2 ? 3 : 1));
  const int ts = no_tree() ? 0 : tree_select(a);
  if (ts) {
    int64_t nbt = 0;
    const int64_t first = tree_split(a, &nbt);
    if (first < nbt)   // tail split active (b = 3 with f, a device present): bundles [first, nbt) split
      return snprintf(buf, n, "k_fine_tree<%d,%d,g=%d,Y=%d>split=%lld/%lld", ts / 10, ts % 10, g,
                      a.Y != nullptr ? 1 : 0, (long long)first, (long long)nbt);
    return snprintf(buf, n, "k_fine_tree<%d,%d,g=%d,Y=%d>", ts / 10, ts % 10, g, a.Y != nullptr ? 1 : 0);
  }
  static const char* bots[4] = {"BotNone", "BotB2", "BotB2s", "BotB3"};
  return snprintf(buf, n, "k_fine<%d,%s>", a.NF, bots[a.NF == 0 ? 0 : bottom_select(a)]);
}

cudaError_t launch_fine(const FineArgs& a, int64_t nb, int nrep, cudaStream_t st, int64_t* nparts) {
  *nparts = a.fsum ? 0 : nb;   // k_fine ends with finish_fsum (the a5 final reduction) when fsum is set
  if (!no_tree()) {
    const cudaError_t e = launch_tree(a, nb, nrep, st, nparts);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (a.NF) {
    case 0: return launch_fine_t<0, BotNone>(a, nb, nrep, st);
    case 1: return launch_fine_n<1>(a, nb, nrep, st);
    case 2: return launch_fine_n<2>(a, nb, nrep, st);
    case 3: return launch_fine_n<3>(a, nb, nrep, st);
    case 4: return launch_fine_n<4>(a, nb, nrep, st);
    case 5: return launch_fine_n<5>(a, nb, nrep, st);
    case 6: return launch_fine_n<6>(a, nb, nrep, st);
    case 7: return launch_fine_n<7>(a, nb, nrep, st);
    default: return cudaErrorInvalidValue;
  }
}

#if RQMC_DEBUG
cudaError_t dbg_set_fine(const DbgRanges& r, cudaStream_t st) { return dbg_set_tu(r, st); }
#else
cudaError_t dbg_set_fine(const DbgRanges&, cudaStream_t) { return cudaSuccess; }
#endif

}  // namespace rqmc
