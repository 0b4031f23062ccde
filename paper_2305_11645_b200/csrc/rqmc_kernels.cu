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

#include <cstdlib>
#include <type_traits>

#include "rqmc_internal.h"

namespace rqmc {

// ------------------------------------------------------------------------------------------
// a2: point generator
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ int64_t global_residue(const GenArgs& a, const GenLevel& L, int64_t rl) {
  // residue-class partition: local row rl of rank g is global residue (g + G rl) mod M
  return L.M >= a.world ? (int64_t)a.rank + (int64_t)a.world * rl : (int64_t)a.rank % L.M;
}

__device__ __forceinline__ double point_value(const GenArgs& a, const GenLevel& L, int64_t r, int j,
                                              uint64_t* word_out) {
  double u;
  if (a.kind == 0) {
    // x = (r z'_j mod M) / M, r < M <= 2^32 and z' < M: the product fits in 64 bits
    const uint64_t M = (uint64_t)L.M;
    const uint64_t prod = (uint64_t)r * a.z[j];
    const uint64_t t = (a.b == 2) ? (prod & (M - 1)) : (prod % M);
    *word_out = t;
    u = __ddiv_rn((double)t, (double)M);
    if (a.shifted) {                       // psi(x) = {x + Delta_j}, reading C-6
      u = __dadd_rn(u, a.shift[j]);
      if (u >= 1.0) u = __dadd_rn(u, -1.0);
    }
  } else {
    // digital net: W = XOR of the (row-zeroed) column words over the set bits of r
    uint64_t W = 0;
    uint64_t rr = (uint64_t)r;
    const uint64_t* col = a.C + (size_t)j * a.m;
    for (int q = 0; rr; ++q, rr >>= 1)
      if (rr & 1u) W ^= col[q];
    if (a.shifted) {
      const uint64_t V = (W << (53 - a.m)) ^ a.dshift[j];
      *word_out = V;
      u = (double)V * 0x1p-53;
    } else {
      *word_out = W;
      u = ldexp((double)W, -a.m);
    }
  }
  if (a.map == 1) {
    if (u == 0.0) u = a.zero_u;            // zero rule, reading C-5
    u = normcdfinv(u);
  }
  return u;
}

__global__ void __launch_bounds__(256) k_gen(const GenArgs a) {
  const GenLevel& L = a.lv[blockIdx.y];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L.Ml * L.ldx) return;
  const int64_t rl = e / L.ldx;
  const int q = (int)(e - rl * L.ldx);
  double v = 0.0;
  if (q < L.s_w) {
    uint64_t wd;
    v = point_value(a, L, global_residue(a, L, rl), L.j_lo + q, &wd);
  }
  a.X[L.xoff + e] = v;
}

__global__ void k_points(const GenArgs a, int lev, int64_t r0, int64_t count, uint64_t* words, double* vals) {
  const GenLevel& L = a.lv[lev];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count * L.s_w) return;
  const int64_t rl = r0 + e / L.s_w;
  const int q = (int)(e % L.s_w);
  uint64_t wd = 0;
  const double v = point_value(a, L, global_residue(a, L, rl), L.j_lo + q, &wd);
  if (words) words[e] = wd;
  if (vals) vals[e] = v;
}

cudaError_t launch_gen(const GenArgs& a, int64_t max_entries, cudaStream_t st) {
  if (a.nlev == 0 || max_entries == 0) return cudaSuccess;
  dim3 grid((unsigned)((max_entries + 255) / 256), (unsigned)a.nlev);
  k_gen<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_points(const GenArgs& a, int lev, int64_t r0, int64_t count, uint64_t* words,
                          double* vals, cudaStream_t st) {
  const int64_t n = count * a.lv[lev].s_w;
  if (n == 0) return cudaSuccess;
  k_points<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, lev, r0, count, words, vals);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// async copy helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// DMMA.8x8x4: D(8x8) += A(8x4, row) B(4x8, col); lane l: a = A[l/4][l%4], b = B[l%4][l/4],
// d = {D[l/4][2(l%4)], D[l/4][2(l%4)+1]}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------------------------------
// a3+a4: coarse level GEMM  R[r, c] = Rp[r mod Mp, c] + sum_q X[r, q] A[q, c]
// CTA tile BM x 64, K step 16, warps (BM/32) x 2 each 32 x 32 (4 x 4 DMMA fragments).
// ------------------------------------------------------------------------------------------
template <int BM, int CH>
__global__ void __launch_bounds__(BM * 2) k_level_gemm(const GemmArgs a) {
  constexpr int BN = 64, BK = 16, XS = BK + 4, AS = BN + 4, NT = BM * 2;
  extern __shared__ __align__(16) double gsm[];
  double (*Xs)[BM][XS] = reinterpret_cast<double (*)[BM][XS]>(gsm);
  double (*As)[BK][AS] = reinterpret_cast<double (*)[BK][AS]>(gsm + 2 * BM * XS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, tg = lane & 3;
  const int64_t r0 = (int64_t)blockIdx.y * BM;
  const int c0 = blockIdx.x * BN;

  auto load_stage = [&](int buf, int k0) {
    // X tile: BM rows x BK cols (ldx even: 16B chunks stay inside the zero-padded row)
    for (int c = tid; c < BM * (BK / 2); c += NT) {
      const int row = c / (BK / 2), kc = (c % (BK / 2)) * 2;
      const int64_t gr = r0 + row;
      const bool ok = gr < a.M && (k0 + kc) < a.ldx;
      const double* src = ok ? a.X + gr * a.ldx + k0 + kc : a.X;
      cp_async16(&Xs[buf][row][kc], src, ok);
    }
    // A tile: BK rows x BN cols
    for (int c = tid; c < BK * (BN / CH); c += NT) {
      const int row = c / (BN / CH), cc = (c % (BN / CH)) * CH;
      const bool ok = (k0 + row) < a.K && (c0 + cc) < a.tau;
      const double* src = ok ? a.A + (int64_t)(k0 + row) * a.lda + c0 + cc : a.A;
      if (CH == 2) cp_async16(&As[buf][row][cc], src, ok);
      else cp_async8(&As[buf][row][cc], src, ok);
    }
    cp_async_commit();
  };

  const int nk = (a.K + BK - 1) / BK;
  load_stage(0, 0);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = r0 + wm * 32 + i * 8 + g;
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      const int col = c0 + wn * 32 + jn * 8 + 2 * tg;
      acc[i][jn][0] = 0.0;
      acc[i][jn][1] = 0.0;
      if (a.Rp && row < a.M) {  // tile(R_w'): row r reads parent row r mod M_w'
        const double* p = a.Rp + (row % a.Mp) * a.ldp + col;
        if (col < a.tau) acc[i][jn][0] = p[0];
        if (col + 1 < a.tau) acc[i][jn][1] = p[1];
      }
    }
  }

  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      load_stage(buf ^ 1, (kt + 1) * BK);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Xs[buf][wm * 32 + i * 8 + g][kk + tg];
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) bf[jn] = As[buf][kk + tg][wn * 32 + jn * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) dmma(acc[i][jn], af[i], bf[jn]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = r0 + wm * 32 + i * 8 + g;
    if (row >= a.M) continue;
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      const int col = c0 + wn * 32 + jn * 8 + 2 * tg;
      double* p = a.R + row * a.ldr + col;
      if (col + 1 < a.tau) {
        *reinterpret_cast<double2*>(p) = make_double2(acc[i][jn][0], acc[i][jn][1]);
      } else if (col < a.tau) {
        p[0] = acc[i][jn][0];
      }
    }
  }
}

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t st) {
  const bool vec = ((uintptr_t)a.A % 16 == 0) && (a.lda % 2 == 0) && (a.tau % 2 == 0);
  const int BM = a.M >= 64 * 148 ? 128 : 64;
  dim3 grid((unsigned)((a.tau + 63) / 64), (unsigned)((a.M + BM - 1) / BM));
  const int sm = (int)sizeof(double) * 2 * (BM * 20 + 16 * 68);
  auto go = [&](auto kern, int nt) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e != cudaSuccess) return e;
    kern<<<grid, nt, sm, st>>>(a);
    return cudaGetLastError();
  };
  if (BM == 128) return vec ? go(k_level_gemm<128, 2>, 256) : go(k_level_gemm<128, 1>, 256);
  return vec ? go(k_level_gemm<64, 2>, 128) : go(k_level_gemm<64, 1>, 128);
}

// ------------------------------------------------------------------------------------------
// a3+a4+a5: fused fine levels.  CTA = bundle of kBundle (32) residues of the checkpoint level x a
// kFineBN (32)-column tile, 8 warps in two groups; group h walks the subtrees under the top fine
// level's runs q = h (mod 2), so the two groups never touch the same leaf row.  In a group, warp
// wm owns rows 8 wm .. 8 wm + 7 of every run and all 32 columns = 1 x 4 DMMA.8x8x4 fragments, so a
// path tile is 8 doubles per lane and one lane's 8 leaf values share ONE row (cheap row sums).
// The DFS stack (one tile per fine level) lives in registers.  K >= 4 steps run on the fp64 tensor
// pipe (mma.sync f64 with C and D in different registers: no stack copies), K mod 4 remainders and
// K < 4 levels as DFMA on the same fragment registers (no zero padding).
// The bottom NB levels of common shapes (BT) are compile-time: fans and K known, loops unrolled,
// leaf consumption (Y store, g) templated, so the per-leaf control overhead disappears.
// Shared memory: [A slab x2][root tile x2][X^red subtree][rowacc], t / c strides padded to 36 doubles
// (bank-conflict-free fragment loads).  Columns >= tau are zero in the A slab and the root tile, so
// leaf values there are exactly 0 and need no mask (g = exp is corrected in the finalisation).
// ------------------------------------------------------------------------------------------
constexpr int kPad = kFinePad;

struct FineCtx {
  int grp, wm, g, tg, t, beff, c0;
  int64_t r0;
  const double* as;      // A slab of the current column tile
};

// D = A B + C with C and D in distinct registers (DMMA.8x8x4)
__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

extern __shared__ __align__(16) double fsm[];

// ---- g kinds (f(y) = F(tau^-1 sum_c g(y_c)), reading C-17): 0 none, 1 identity, 2 exp(p0 y), 3 y^2
template <int G>
__device__ __forceinline__ double gsum8(const double (&S)[8], double p0) {
  if constexpr (G == 2) {
    double v = exp(p0 * S[0]);
#pragma unroll
    for (int e = 1; e < 8; ++e) v += exp(p0 * S[e]);
    return v;
  } else if constexpr (G == 3) {
    double v = S[0] * S[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) v = fma(S[e], S[e], v);
    return v;
  } else {
    return ((S[0] + S[1]) + (S[2] + S[3])) + ((S[4] + S[5]) + (S[6] + S[7]));
  }
}

template <bool STY>
__device__ __forceinline__ void store_leaf(const FineArgs& a, const double (&S)[8], int j, const FineCtx& c) {
  if constexpr (STY) {
    if (c.t < c.beff) {
      double* yr = a.Y + (c.r0 + c.t + (int64_t)j * a.Mroot) * a.ldy;
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) {
        const int col = c.c0 + cf * 8 + 2 * c.tg;
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
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  FineCtx c;
  c.grp = warp >> 2;
  c.wm = warp & 3;
  c.g = lane >> 2;
  c.tg = lane & 3;
  c.t = c.wm * 8 + c.g;
  c.r0 = (int64_t)blockIdx.x * kBundle;
  c.beff = (int)((a.Mroot - c.r0) < kBundle ? (a.Mroot - c.r0) : kBundle);

  // X^red of the subtree -> smem [run][q][t] (t stride kPad); global rows r0 + t + j Mroot, read
  // row-contiguously, written transposed.
  for (int i = 0; i < NF; ++i) {
    const FineLevel& L = a.lv[i];
    double* xs = fsm + L.xs_off;
    // lane = t (conflict-free smem stores), loop over (run, q) rows, 4 loads in flight per thread
    const int nrow = L.runs * L.K;
    const int t = tid & (kBundle - 1);
    const double* src = L.X + (c.r0 + t) * L.ldx;
    for (int r = tid >> 5; r < nrow; r += 4 * (kFineThreads >> 5)) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = r + u * (kFineThreads >> 5);
        const int j = rr / L.K, q = rr - j * L.K;
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
      const bool row_ok = a.root != nullptr && t < c.beff;
      const double* src = a.root + (c.r0 + t) * a.ldroot + c0 + cc;
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
      a.partial[blockIdx.x] = t;
    }
  }
}

template <int NF, class BT>
static cudaError_t launch_fine_t(const FineArgs& a, int64_t nb, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_fine<NF, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
  if (e != cudaSuccess) return e;
  k_fine<NF, BT><<<(unsigned)nb, kFineThreads, a.smem_bytes, st>>>(a);
  return cudaGetLastError();
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

template <int NF>
static cudaError_t launch_fine_n(const FineArgs& a, int64_t nb, cudaStream_t st) {
  if constexpr (NF >= 3)
    if (bottom_matches<BotB2>(a)) return launch_fine_t<NF, BotB2>(a, nb, st);
  if constexpr (NF >= 2) {
    if (bottom_matches<BotB2s>(a)) return launch_fine_t<NF, BotB2s>(a, nb, st);
    if (bottom_matches<BotB3>(a)) return launch_fine_t<NF, BotB3>(a, nb, st);
  }
  return launch_fine_t<NF, BotNone>(a, nb, st);
}

// ------------------------------------------------------------------------------------------
// k_fine_tree<NF, B, G, STY>: the fused fine levels for the paper's own level shape
// w_j = floor(log_B j) (every BASELINE config): fine level i (coarse -> fine) is
// w = NF-1-i with K_i = (B-1) B^{NF-1-i} coordinates, every node has B children, and the fine
// coordinates are the prefix j < B^NF - 1 of A.  With the whole tree compile-time, every loop is
// unrolled and every smem offset is a constant; the lane/warp/CTA mapping, the smem layout and the
// arithmetic are exactly those of k_fine (same fragments, same summation order).
// ------------------------------------------------------------------------------------------
// K = 2 non-leaf level of the b = 2 tree: one zero-padded DMMA step (true) or 2 DFMA steps (false)
constexpr bool kTreePadK2 = true;

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
  const FineArgs& a;
  const FineCtx& c;
  double a0[T::K(NF - 1) <= 2 ? T::K(NF - 1) : 1][8];  // leaf A values (K <= 2: DFMA leaves)
  double bk[4];                                         // B fragments of a K < 4 non-leaf level (B = 2)

  __device__ __forceinline__ TreeRun(const FineArgs& a_, const FineCtx& c_) : a(a_), c(c_) {}

  __device__ __forceinline__ const double* xs(int i, int j) const {
    return fsm + T::XS + i * T::XL + j * T::K(i) * kPad + c.t;
  }
  __device__ __forceinline__ const double* as(int i) const { return c.as + T::jlo(i) * kPad; }

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

  // b = 2 bottom (levels K = 4, 2, 1 below the parent tile Sp): both level-2 nodes (or the group's
  // one, at the top), their level-1 tiles and all leaves are formed first, then the 8 (4) row-sum
  // shuffle chains run together and the prefetched rowacc slots are updated once.
  __device__ __forceinline__ void bottom_b2(const double (&Sp)[8], int jp) {
    constexpr int I2 = NF - 3, I1 = NF - 2, I0 = NF - 1;
    constexpr int RP2 = (I2 == 0) ? 1 : T::runs(I2) / 2, RP1 = T::runs(I1) / 2, RP0 = T::runs(I0) / 2;
    constexpr int NQ = (I2 == 0) ? 1 : 2;  // level-2 nodes handled by this warp
    int jl[4 * NQ];
    double v[4 * NQ], pre[4 * NQ];
#pragma unroll
    for (int n = 0; n < NQ; ++n) {
      const int q2 = (I2 == 0) ? c.grp : n;
      const int j2 = jp + q2 * RP2;
#pragma unroll
      for (int l = 0; l < 4; ++l) jl[4 * n + l] = j2 + (l >> 1) * RP1 + (l & 1) * RP0;
    }
    if constexpr (G > 0) {
#pragma unroll
      for (int l = 0; l < 4 * NQ; ++l) pre[l] = fsm[T::ACC + jl[l] * kBundle + c.t];
    }
#pragma unroll
    for (int n = 0; n < NQ; ++n) {
      const int j2 = jl[4 * n];
      double S2[8];
      tree_step<4>(xs(I2, j2), as(I2), c, Sp, S2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j1 = j2 + h * RP1;
        double S1[8];
        if constexpr (kTreePadK2) {
          const double af = c.tg < 2 ? xs(I1, j1)[c.tg * kPad] : 0.0;
#pragma unroll
          for (int cf = 0; cf < 4; ++cf) dmma_c(S1[2 * cf], S1[2 * cf + 1], af, bk[cf], S2[2 * cf], S2[2 * cf + 1]);
        } else {
          tree_step<2>(xs(I1, j1), as(I1), c, S2, S1);
        }
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
#pragma unroll
      for (int l = 0; l < 4 * NQ; ++l) v[l] += __shfl_xor_sync(0xffffffffu, v[l], 1);
#pragma unroll
      for (int l = 0; l < 4 * NQ; ++l) v[l] += __shfl_xor_sync(0xffffffffu, v[l], 2);
      if (c.tg == 0) {
#pragma unroll
        for (int l = 0; l < 4 * NQ; ++l) fsm[T::ACC + jl[l] * kBundle + c.t] = pre[l] + v[l];
      }
    }
  }

  template <int I>
  __device__ __forceinline__ void level(const double (&Sp)[8], int jp) {
    if constexpr (B == 2 && NF >= 3 && I == NF - 3) {
      bottom_b2(Sp, jp);
    } else if constexpr (I == NF - 1) {
      leaves(Sp, jp);
    } else {
      constexpr int RP = (I == 0) ? 1 : T::runs(I) / B;
      auto child = [&](int q) {
        const int j = jp + q * RP;
        double S[8];
        if constexpr (B == 2 && T::K(I) < 4) {  // K = 2 non-leaf level: one zero-padded DMMA step
          const double af = c.tg < T::K(I) ? xs(I, j)[c.tg * kPad] : 0.0;
#pragma unroll
          for (int cf = 0; cf < 4; ++cf) dmma_c(S[2 * cf], S[2 * cf + 1], af, bk[cf], Sp[2 * cf], Sp[2 * cf + 1]);
        } else {
          tree_step<T::K(I)>(xs(I, j), as(I), c, Sp, S);
        }
        level<I + 1>(S, j);
      };
      if constexpr (I == 0) {
        for (int q = c.grp; q < B; q += 2) child(q);  // top level split over the two warp groups
      } else {
#pragma unroll
        for (int q = 0; q < B; ++q) child(q);
      }
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
    if constexpr (B == 2 && NF >= 2) {
      constexpr int I1 = NF - 2;  // the K = 2 level
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) bk[cf] = c.tg < T::K(I1) ? as(I1)[c.tg * kPad + cf * 8 + c.g] : 0.0;
    }
    level<0>(Sroot, 0);
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
  if constexpr (G > 0)
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
    TreeRun<NF, B, G, STY> run(a, c);
    run.tile(Sroot);
    __syncthreads();
  }

  if constexpr (G > 0) {
    const double pad = (G == 2) ? (double)(ntiles * kFineBN - a.tau) : 0.0;
    double part = 0.0;
    for (int e = tid; e < T::LEAVES * kBundle; e += kFineThreads) {
      const int t = e % kBundle;
      if (t >= c.beff) continue;
      const double mean = (fsm[T::ACC + e] - pad) / a.tau;
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
static cudaError_t launch_tree(const FineArgs& a, int64_t nb, cudaStream_t st) {
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

cudaError_t launch_fine(const FineArgs& a, int64_t nb, cudaStream_t st) {
  if (std::getenv("RQMC_NO_TREE") == nullptr) {
    const cudaError_t e = launch_tree(a, nb, st);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (a.NF) {
    case 0: return launch_fine_t<0, BotNone>(a, nb, st);
    case 1: return launch_fine_n<1>(a, nb, st);
    case 2: return launch_fine_n<2>(a, nb, st);
    case 3: return launch_fine_n<3>(a, nb, st);
    case 4: return launch_fine_n<4>(a, nb, st);
    case 5: return launch_fine_n<5>(a, nb, st);
    case 6: return launch_fine_n<6>(a, nb, st);
    case 7: return launch_fine_n<7>(a, nb, st);
    case 8: return launch_fine_n<8>(a, nb, st);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------------------
// a5: fixed-order reduction of per-bundle partial sums
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_reduce(const double* __restrict__ p, int64_t n, double* out) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) s += p[i];
  __shared__ double red[1024];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

cudaError_t launch_reduce(const double* partial, int64_t n, double* out, cudaStream_t st) {
  k_reduce<<<1, 1024, 0, st>>>(partial, n, out);
  return cudaGetLastError();
}

}  // namespace rqmc
