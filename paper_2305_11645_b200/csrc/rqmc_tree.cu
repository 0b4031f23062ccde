// k_fine_tree: compile-time fused fine levels for the paper's level shape w_j = floor(log_b j).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstdlib>
#include <type_traits>

#include "rqmc_device.cuh"

namespace rqmc {

// ------------------------------------------------------------------------------------------
// k_fine_tree<NF, B, G, STY>: the fused fine levels for the paper's own level shape
// w_j = floor(log_B j) (every BASELINE config): fine level i (coarse -> fine) is
// w = NF-1-i with K_i = (B-1) B^{NF-1-i} coordinates, every node has B children, and the fine
// coordinates are the prefix j < B^NF - 1 of A.  With the whole tree compile-time, every loop is
// unrolled and every smem offset is a constant; the lane/warp/CTA mapping, the smem layout and the
// arithmetic are exactly those of k_fine (same fragments, same summation order).
// ------------------------------------------------------------------------------------------
// K = 2 non-leaf level of the b = 2 tree: 2 DFMA steps on cached A values (default) or, with
// -DRQMC_K2_PAD=1, one zero-padded DMMA step (twice the fp64-pipe time, fewer issue slots)
#ifndef RQMC_K2_PAD
#define RQMC_K2_PAD 0
#endif
#ifndef RQMC_K2_CACHE          // DFMA K = 2 level: A values cached in registers per column tile (1) or read from smem
#define RQMC_K2_CACHE 1
#endif

template <int NF, int B>
struct Tree {
  __host__ __device__ static constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
  __host__ __device__ static constexpr int K(int i) { return (B - 1) * ipow(B, NF - 1 - i); }          // s_w, w = NF-1-i
  __host__ __device__ static constexpr int runs(int i) { return ipow(B, i + 1); }                      // runs per bundle
  static constexpr int J = ipow(B, NF) - 1;                                        // fine A rows
  __host__ __device__ static constexpr int jlo(int i) { return ipow(B, NF - 1 - i) - 1; }              // first A row
  static constexpr int ABUF = J * kPad;                                            // one A slab
  static constexpr int ROOT = 2 * ABUF;                                            // root tiles
  static constexpr int XS = ROOT + 2 * kBundle * kPad;                             // X subtree
  static constexpr int XL = (B - 1) * ipow(B, NF) * kPad;                          // X per level
  static constexpr int ACC = XS + NF * XL;                                         // rowacc
  static constexpr int LEAVES = ipow(B, NF);
  static constexpr int SMEM = (ACC + LEAVES * kBundle) * 8;
};

// S = Sp + X^red[run j] A_w, compile-time K (DMMA k-steps of 4, DFMA remainder); xs, as: level bases.
template <int K>
__device__ __forceinline__ void tree_step(const double* xs, const double* as, const FineCtx& c, const double (&Sp)[8],
                                          double (&S)[8]) {
  static_assert(K >= 1, "");
  if constexpr (K >= 4) {
    constexpr int NS = K / 4;
    double af = xs[c.tg * kPad], bf[4];
#pragma unroll
    for (int cf = 0; cf < 4; ++cf) bf[cf] = as[c.tg * kPad + c.g + cf * 8];
#pragma unroll
    for (int s = 0; s < NS; ++s) {  // fragments of step s+1 are loaded before step s's DMMAs issue
      double afn = 0.0, bfn[4] = {0.0, 0.0, 0.0, 0.0};
      if (s + 1 < NS) {
        afn = xs[(4 * (s + 1) + c.tg) * kPad];
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) bfn[cf] = as[(4 * (s + 1) + c.tg) * kPad + c.g + cf * 8];
      }
      if (s == 0) {
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, bf[cf], Sp[2 * cf], Sp[2 * cf + 1]);
      } else {
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, bf[cf], S[2 * cf], S[2 * cf + 1]);
      }
      af = afn;
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) bf[cf] = bfn[cf];
    }
  }
#pragma unroll
  for (int kk = (K / 4) * 4; kk < K; ++kk) {
    const double x = xs[kk * kPad];
#pragma unroll
    for (int cf = 0; cf < 4; ++cf) {
      const double2 p = *reinterpret_cast<const double2*>(as + kk * kPad + cf * 8 + 2 * c.tg);
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

template <int NF, int B, int G, bool STY>
struct TreeRun {
  using T = Tree<NF, B>;
  // b = 2 trees with >= 3 fine levels: the bottom three levels run as one block (bottom_b2) and the
  // row sums of g live in registers across all column tiles (kRegAcc); otherwise in smem (rowacc).
  static constexpr bool kB2 = (B == 2 && NF >= 3);
  static constexpr bool kRegAcc = kB2 && G > 0;
  static constexpr int I2 = NF - 3;                                // the K = 4 level of the b = 2 bottom
  static constexpr int NQ = (I2 <= 0) ? 1 : 2;                     // K = 4 nodes per bottom block
  static constexpr int NBAT = (I2 <= 0) ? 1 : T::ipow(2, I2 - 1);  // bottom blocks per warp and tile
  static constexpr int RW = NQ;                                    // leaf row sums a lane keeps per block
  static constexpr int K1 = (B == 2 && NF >= 2) ? T::K(NF - 2) : 0;  // the K = 2 level (b = 2)

  const FineArgs& a;
  const FineCtx& c;
  double a0[T::K(NF - 1) <= 2 ? T::K(NF - 1) : 1][8];  // leaf A values (K <= 2: DFMA leaves)
#if RQMC_K2_PAD
  double bk[4];                                         // B fragments of the zero-padded K = 2 DMMA step
#else
  double a1[K1 == 2 && RQMC_K2_CACHE ? 2 : 1][8];       // A values of the K = 2 level (DFMA, no padding)
#endif
  double racc[kRegAcc ? NBAT * RW : 1];                 // row sums sum_c g(y_kc) of this lane's leaf rows

  __device__ __forceinline__ TreeRun(const FineArgs& a_, const FineCtx& c_) : a(a_), c(c_) {
#pragma unroll
    for (int i = 0; i < (kRegAcc ? NBAT * RW : 1); ++i) racc[i] = 0.0;
  }

  __device__ __forceinline__ const double* xs(int i, int j) const {
    return fsm + T::XS + i * T::XL + j * T::K(i) * kPad + c.t;
  }
  __device__ __forceinline__ const double* as(int i) const { return c.as + T::jlo(i) * kPad; }

  // S = Sp + X^red[run j] A_w for the K = 2 level (b = 2): cached A values, DFMA (or one padded DMMA)
  __device__ __forceinline__ void step_k2(const double (&Sp)[8], int i, int j, double (&S)[8]) const {
#if RQMC_K2_PAD
    const double af = c.tg < 2 ? xs(i, j)[c.tg * kPad] : 0.0;
#pragma unroll
    for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, bk[cf], Sp[2 * cf], Sp[2 * cf + 1]);
#elif RQMC_K2_CACHE
    const double x0 = xs(i, j)[0], x1 = xs(i, j)[kPad];
#pragma unroll
    for (int e = 0; e < 8; ++e) S[e] = fma(x1, a1[1][e], fma(x0, a1[0][e], Sp[e]));
#else
    tree_step<2>(xs(i, j), as(i), c, Sp, S);
#endif
  }

  // leaves of parent run jp (level NF-1): values, Y store, g sums, row-sum shuffles, rowacc update
  __device__ __forceinline__ void leaves(const double (&Sp)[8], int jp) {
    constexpr int I = NF - 1, KL = T::K(I), RP = T::runs(I) / B;
    double v[B], pre[B];
    if constexpr (G > 0) {
#pragma unroll
      for (int q = 0; q < B; ++q) pre[q] = fsm[T::ACC + (jp + q * RP) * kBundle + c.t];
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int j = jp + q * RP;
      double Y[8];
      if constexpr (KL <= 2) {
        const double* x = xs(I, j);
        const double x0 = x[0];
#pragma unroll
        for (int e = 0; e < 8; ++e) Y[e] = fma(x0, a0[0][e], Sp[e]);
        if constexpr (KL == 2) {
          const double x1 = x[kPad];
#pragma unroll
          for (int e = 0; e < 8; ++e) Y[e] = fma(x1, a0[KL - 1][e], Y[e]);
        }
      } else {
        tree_step<KL>(xs(I, j), as(I), c, Sp, Y);
      }
      store_leaf<STY>(a, Y, j, c);
      if constexpr (G > 0) v[q] = gsum8<G>(Y, a.fp0);
    }
    if constexpr (G > 0) {
#pragma unroll
      for (int q = 0; q < B; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 1);
#pragma unroll
      for (int q = 0; q < B; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 2);
      if (c.tg == 0) {
#pragma unroll
        for (int q = 0; q < B; ++q) fsm[T::ACC + (jp + q * RP) * kBundle + c.t] = pre[q] + v[q];
      }
    }
  }

  // b = 2 bottom (levels K = 4, 2, 1 below the parent tile Sp, bottom block number P of this warp):
  // the NQ level-(NF-3) nodes, their level-(NF-2) tiles and all 4 NQ leaves are formed first; then one
  // transpose-reduce over the 4 lanes of each row leaves lane tg with the complete 32-column sums of
  // the leaves 2 tg, 2 tg + 1 (NQ = 2; leaf tg for NQ = 1), accumulated in registers.
  template <int P>
  __device__ __forceinline__ void bottom_b2(const double (&Sp)[8], int jp) {
    constexpr int I1 = NF - 2, I0 = NF - 1;
    constexpr int RP2 = (I2 == 0) ? 1 : T::runs(I2) / 2, RP1 = T::runs(I1) / 2, RP0 = T::runs(I0) / 2;
    constexpr int NL = 4 * NQ;
    int jl[NL];
    double v[NL];
#pragma unroll
    for (int n = 0; n < NQ; ++n) {
      const int q2 = (I2 == 0) ? c.grp : n;
      const int j2 = jp + q2 * RP2;
#pragma unroll
      for (int l = 0; l < 4; ++l) jl[4 * n + l] = j2 + (l >> 1) * RP1 + (l & 1) * RP0;
    }
#pragma unroll
    for (int n = 0; n < NQ; ++n) {
      const int j2 = jl[4 * n];
      double S2[8];
      tree_step<4>(xs(I2, j2), as(I2), c, Sp, S2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double S1[8];
        step_k2(S2, I1, j2 + h * RP1, S1);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int l = 4 * n + 2 * h + q;
          const double x0 = xs(I0, jl[l])[0];
          double Y[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) Y[e] = fma(x0, a0[0][e], S1[e]);
          store_leaf<STY>(a, Y, jl[l], c);
          if constexpr (G > 0) v[l] = gsum8<G>(Y, a.fp0);
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
        racc[P * RW + i] += keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
    }
  }

  // children at level I of the parent tile Sp (run jp); P = the parent's position among this warp's
  // level-(I-1) nodes (compile time, so register row sums are statically indexed)
  template <int I, int P>
  __device__ __forceinline__ void level(const double (&Sp)[8], int jp) {
    if constexpr (kB2 && I == I2) {
      bottom_b2<P>(Sp, jp);
    } else if constexpr (I == NF - 1) {
      leaves(Sp, jp);
    } else {
      constexpr int RP = (I == 0) ? 1 : T::runs(I) / B;
      if constexpr (I == 0) {
        for (int q = c.grp; q < B; q += 2) {  // top level split over the two warp groups
          double S[8];
          if constexpr (B == 2 && T::K(I) == 2) step_k2(Sp, I, q, S);
          else tree_step<T::K(I)>(xs(I, q), as(I), c, Sp, S);
          level<I + 1, 0>(S, q);
        }
      } else {
        level_children<I, P, 0>(Sp, jp);
      }
    }
  }
  template <int I, int P, int Q>
  __device__ __forceinline__ void level_children(const double (&Sp)[8], int jp) {
    if constexpr (Q < B) {
      constexpr int RP = T::runs(I) / B;
      const int j = jp + Q * RP;
      double S[8];
      if constexpr (B == 2 && T::K(I) == 2) step_k2(Sp, I, j, S);
      else tree_step<T::K(I)>(xs(I, j), as(I), c, Sp, S);
      level<I + 1, P * B + Q>(S, j);
      level_children<I, P, Q + 1>(Sp, jp);
    }
  }

  __device__ __forceinline__ void tile(const double (&Sroot)[8]) {
    constexpr int KL = T::K(NF - 1);
    if constexpr (KL <= 2) {
#pragma unroll
      for (int q = 0; q < KL; ++q)
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) {
          const double2 p = *reinterpret_cast<const double2*>(as(NF - 1) + q * kPad + cf * 8 + 2 * c.tg);
          a0[q][2 * cf] = p.x;
          a0[q][2 * cf + 1] = p.y;
        }
    }
    if constexpr (K1 == 2) {
#if RQMC_K2_PAD
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) bk[cf] = c.tg < 2 ? as(NF - 2)[c.tg * kPad + cf * 8 + c.g] : 0.0;
#elif RQMC_K2_CACHE
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) {
          const double2 p = *reinterpret_cast<const double2*>(as(NF - 2) + q * kPad + cf * 8 + 2 * c.tg);
          a1[q][2 * cf] = p.x;
          a1[q][2 * cf + 1] = p.y;
        }
#endif
    }
    level<0, 0>(Sroot, 0);
  }

  // sum over this lane's complete leaf rows of F(tau^-1 sum_c g), fixed order (kRegAcc only)
  __device__ __forceinline__ double fsum_regs(double pad) const {
    double part = 0.0;
    if (c.t < c.beff) {
#pragma unroll
      for (int i = 0; i < (kRegAcc ? NBAT * RW : 1); ++i) part += f_of_mean(a, (racc[i] - pad) / a.tau);
    }
    return part;
  }
};

template <int NF, int B, int G, bool STY>
__global__ void __launch_bounds__(kFineThreads, 1) k_fine_tree(const FineArgs a) {
  using T = Tree<NF, B>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  FineCtx c;
  c.grp = warp >> 2;
  c.wm = warp & 3;
  c.g = lane >> 2;
  c.tg = lane & 3;
  c.t = c.wm * 8 + c.g;
  c.r0 = (int64_t)blockIdx.x * kBundle;
  c.beff = (int)((a.Mroot - c.r0) < kBundle ? (a.Mroot - c.r0) : kBundle);

  // X^red of the subtree -> smem [level][run][q][t]; lane = t, rows (run, q) strided over warps
  {
    const int t = tid & (kBundle - 1);
#pragma unroll
    for (int i = 0; i < NF; ++i) {
      const int K = T::K(i), nrow = T::runs(i) * K;
      const double* src = a.lv[i].X + (c.r0 + t) * (int64_t)K;
      double* dst = fsm + T::XS + i * T::XL + t;
      for (int r = tid >> 5; r < nrow; r += 4 * (kFineThreads >> 5)) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = r + u * (kFineThreads >> 5);
          const int j = rr / K, q = rr - j * K;
          v[u] = (rr < nrow && t < c.beff) ? src[(int64_t)j * a.Mroot * K + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = r + u * (kFineThreads >> 5);
          if (rr < nrow) dst[rr * kPad] = v[u];
        }
      }
    }
  }
  using Run = TreeRun<NF, B, G, STY>;
  if constexpr (G > 0 && !Run::kRegAcc)
    for (int e = tid; e < T::LEAVES * kBundle; e += kFineThreads) fsm[T::ACC + e] = 0.0;

  // column tile operands (cp.async, double buffer): A rows [0, J) x 32 columns and the root tile
  const int ntiles = (a.tau + kFineBN - 1) / kFineBN;
  auto load_tile = [&](int buf, int c0) {
    double* as = fsm + buf * T::ABUF;
    if (a.a_vec) {
      for (int e = tid; e < T::J * (kFineBN / 2); e += kFineThreads) {
        const int q = e >> 4, cc = (e & 15) * 2;
        const bool ok = c0 + cc < a.tau;
        cp_async16(as + q * kPad + cc, ok ? a.A + (int64_t)q * a.lda + c0 + cc : a.A, ok);
      }
    } else {
      for (int e = tid; e < T::J * kFineBN; e += kFineThreads) {
        const int q = e >> 5, cc = e & 31;
        const bool ok = c0 + cc < a.tau;
        cp_async8(as + q * kPad + cc, ok ? a.A + (int64_t)q * a.lda + c0 + cc : a.A, ok);
      }
    }
    double* rs = fsm + T::ROOT + buf * (kBundle * kPad);
    for (int e = tid; e < kBundle * (kFineBN / 2); e += kFineThreads) {
      const int t = e >> 4, cc = (e & 15) * 2;
      const bool row_ok = a.root != nullptr && t < c.beff;
      const double* src = a.root + (c.r0 + t) * a.ldroot + c0 + cc;
      if (c0 + cc + 1 < a.tau || !row_ok) {
        cp_async16(rs + t * kPad + cc, row_ok ? src : a.A, row_ok);
      } else {
        cp_async8(rs + t * kPad + cc, row_ok && c0 + cc < a.tau ? src : a.A, row_ok && c0 + cc < a.tau);
        cp_async8(rs + t * kPad + cc + 1, a.A, false);
      }
    }
    cp_async_commit();
  };

  Run run(a, c);
  load_tile(0, 0);
  for (int ct = 0; ct < ntiles; ++ct) {
    c.c0 = ct * kFineBN;
    c.as = fsm + (ct & 1) * T::ABUF;
    if (ct + 1 < ntiles) {
      load_tile((ct + 1) & 1, (ct + 1) * kFineBN);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    double Sroot[8];
    {
      const double* rs = fsm + T::ROOT + (ct & 1) * (kBundle * kPad) + c.t * kPad + 2 * c.tg;
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) {
        const double2 p = *reinterpret_cast<const double2*>(rs + cf * 8);
        Sroot[2 * cf] = p.x;
        Sroot[2 * cf + 1] = p.y;
      }
    }
    run.tile(Sroot);
    __syncthreads();
  }

  if constexpr (G > 0) {
    // padded columns (>= tau) hold y = 0 exactly: g(0) = 0 except g = exp, which added exp(0) = 1
    const double pad = (G == 2) ? (double)(ntiles * kFineBN - a.tau) : 0.0;
    double part = 0.0;
    if constexpr (Run::kRegAcc) {
      part = run.fsum_regs(pad);
    } else {
      for (int e = tid; e < T::LEAVES * kBundle; e += kFineThreads) {
        const int t = e % kBundle;
        if (t >= c.beff) continue;
        part += f_of_mean(a, (fsm[T::ACC + e] - pad) / a.tau);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __shared__ double red[kFineThreads / 32];
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kFineThreads / 32; ++w) t += red[w];
      a.partial[blockIdx.x] = t;
    }
  }
}

template <int NF, int B, int G, bool STY>
static cudaError_t launch_tree_t(const FineArgs& a, int64_t nb, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_fine_tree<NF, B, G, STY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Tree<NF, B>::SMEM);
  if (e != cudaSuccess) return e;
  k_fine_tree<NF, B, G, STY><<<(unsigned)nb, kFineThreads, Tree<NF, B>::SMEM, st>>>(a);
  return cudaGetLastError();
}

// Does the fine level table have the compile-time shape Tree<NF, B> (and the same smem layout)?
template <int NF, int B>
static bool tree_matches(const FineArgs& a) {
  using T = Tree<NF, B>;
  if (a.NF != NF || a.smem_bytes != T::SMEM || a.acc_off != T::ACC || a.leafruns != T::LEAVES) return false;
  for (int i = 0; i < NF; ++i) {
    const FineLevel& L = a.lv[i];
    if (L.K != T::K(i) || L.fan != B || L.runs != T::runs(i) || L.j_lo != T::jlo(i) || L.ldx != L.K ||
        L.xs_off != T::XS + i * T::XL)
      return false;
  }
  return true;
}

template <int NF, int B>
static cudaError_t launch_tree_g(const FineArgs& a, int64_t nb, cudaStream_t st) {
  const bool sty = a.Y != nullptr;
  switch (a.fk) {
    case -1: return launch_tree_t<NF, B, 0, true>(a, nb, st);
    case 1: return sty ? launch_tree_t<NF, B, 2, true>(a, nb, st) : launch_tree_t<NF, B, 2, false>(a, nb, st);
    case 2: return sty ? launch_tree_t<NF, B, 3, true>(a, nb, st) : launch_tree_t<NF, B, 3, false>(a, nb, st);
    default: return sty ? launch_tree_t<NF, B, 1, true>(a, nb, st) : launch_tree_t<NF, B, 1, false>(a, nb, st);
  }
}

// returns cudaErrorNotSupported when no compile-time tree matches
cudaError_t launch_tree(const FineArgs& a, int64_t nb, cudaStream_t st) {
  if (a.Y == nullptr && a.fk < 0) return cudaErrorNotSupported;
  if (tree_matches<6, 2>(a)) return launch_tree_g<6, 2>(a, nb, st);
  if (tree_matches<5, 2>(a)) return launch_tree_g<5, 2>(a, nb, st);
  if (tree_matches<4, 2>(a)) return launch_tree_g<4, 2>(a, nb, st);
  if (tree_matches<3, 2>(a)) return launch_tree_g<3, 2>(a, nb, st);
  if (tree_matches<2, 2>(a)) return launch_tree_g<2, 2>(a, nb, st);
  if (tree_matches<7, 2>(a)) return launch_tree_g<7, 2>(a, nb, st);
  if (tree_matches<3, 3>(a)) return launch_tree_g<3, 3>(a, nb, st);
  if (tree_matches<2, 3>(a)) return launch_tree_g<2, 3>(a, nb, st);
  return cudaErrorNotSupported;
}

}  // namespace rqmc
