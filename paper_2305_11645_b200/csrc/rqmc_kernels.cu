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
// level's runs q = h (mod 2), so the two groups never touch the same leaf row.  Inside a group the
// 4 warps tile the 32 x 32 block as 2 x 2 warp tiles of 16 x 16 = 2 x 2 DMMA.8x8x4 fragments;
// a path tile is 8 doubles per lane, so the whole DFS stack (one tile per fine level) lives in
// registers.  K >= 4 steps run on the fp64 tensor pipe (mma.sync f64), K mod 4 remainders (and the
// K = 1, 2 finest levels) as DFMA on the same accumulator registers -- no zero padding.
// Shared memory: [A slab buf 0][A slab buf 1][X^red subtree][rowacc], t / c strides padded to 36
// doubles so fragment loads are bank-conflict free.
// ------------------------------------------------------------------------------------------
constexpr int kPad = kFinePad;

struct FineCtx {
  int grp, wm, wn, g, tg, beff, c0;
  int64_t r0;
  double* smem;
  const double* as;      // A slab of the current column tile
};

__device__ __forceinline__ double g_of(int fk, double y, double p0) {
  return fk == 1 ? exp(p0 * y) : (fk == 2 ? y * y : y);
}

// Leaf (level 0 rows of run j): store Y and / or accumulate g into rowacc[wn][j][t].
__device__ __forceinline__ void fine_consume(const FineArgs& a, const double (&S)[8], int j, const FineCtx& c) {
  if (a.Y) {
#pragma unroll
    for (int rf = 0; rf < 2; ++rf) {
      const int t = c.wm * 16 + rf * 8 + c.g;
      if (t >= c.beff) continue;
      double* yr = a.Y + (c.r0 + t + (int64_t)j * a.Mroot) * a.ldy;
#pragma unroll
      for (int cf = 0; cf < 2; ++cf) {
        const int col = c.c0 + c.wn * 16 + cf * 8 + 2 * c.tg;
        const double v0 = S[rf * 4 + cf * 2], v1 = S[rf * 4 + cf * 2 + 1];
        if (col + 1 < a.tau) {
          if (a.y_vec) *reinterpret_cast<double2*>(yr + col) = make_double2(v0, v1);
          else { yr[col] = v0; yr[col + 1] = v1; }
        } else if (col < a.tau) {
          yr[col] = v0;
        }
      }
    }
  }
  if (a.fk >= 0) {
    double s[2];
#pragma unroll
    for (int rf = 0; rf < 2; ++rf) {
      double acc = 0.0;
#pragma unroll
      for (int cf = 0; cf < 2; ++cf) {
        const int col = c.c0 + c.wn * 16 + cf * 8 + 2 * c.tg;
        if (col < a.tau) acc += g_of(a.fk, S[rf * 4 + cf * 2], a.fp0);
        if (col + 1 < a.tau) acc += g_of(a.fk, S[rf * 4 + cf * 2 + 1], a.fp0);
      }
      s[rf] = acc;
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      s[0] += __shfl_xor_sync(0xffffffffu, s[0], o);
      s[1] += __shfl_xor_sync(0xffffffffu, s[1], o);
    }
    if (c.tg == 0) {
      double* acc = c.smem + a.acc_off + ((size_t)c.wn * a.leafruns + j) * kBundle + c.wm * 16 + c.g;
      acc[0] += s[0];
      acc[8] += s[1];
    }
  }
}

// S += X^red_w[run j] A_w for one fine level (paper Alg. 2 "+ X_I A_I").
__device__ __forceinline__ void fine_product(const FineLevel& L, int j, const FineCtx& c, double (&S)[8]) {
  const double* xs = c.smem + L.xs_off + (size_t)j * L.K * kPad + c.wm * 16 + c.g;
  const double* as = c.as + L.as_off + c.wn * 16;
  int kk = 0;
#pragma unroll 2
  for (; kk + 4 <= L.K; kk += 4) {
    const double* xq = xs + (kk + c.tg) * kPad;
    const double* aq = as + (kk + c.tg) * kPad + c.g;
    const double a0 = xq[0], a1 = xq[8];
    const double b0 = aq[0], b1 = aq[8];
    double d[2];
#define RQMC_MMA(IDX, AF, BF) d[0] = S[IDX]; d[1] = S[IDX + 1]; dmma(d, AF, BF); S[IDX] = d[0]; S[IDX + 1] = d[1];
    RQMC_MMA(0, a0, b0)
    RQMC_MMA(2, a0, b1)
    RQMC_MMA(4, a1, b0)
    RQMC_MMA(6, a1, b1)
#undef RQMC_MMA
  }
  for (; kk < L.K; ++kk) {  // K mod 4 remainder on the DFMA pipe, same fragment layout
    const double x0 = xs[kk * kPad], x1 = xs[kk * kPad + 8];
    const double2 p0 = *reinterpret_cast<const double2*>(as + kk * kPad + 2 * c.tg);
    const double2 p1 = *reinterpret_cast<const double2*>(as + kk * kPad + 8 + 2 * c.tg);
    S[0] = fma(x0, p0.x, S[0]); S[1] = fma(x0, p0.y, S[1]);
    S[2] = fma(x0, p1.x, S[2]); S[3] = fma(x0, p1.y, S[3]);
    S[4] = fma(x1, p0.x, S[4]); S[5] = fma(x1, p0.y, S[5]);
    S[6] = fma(x1, p1.x, S[6]); S[7] = fma(x1, p1.y, S[7]);
  }
}

template <int I, int NF>
__device__ __forceinline__ void fine_level(const FineArgs& a, const double (&Sp)[8], int jp, const FineCtx& c) {
  if constexpr (I >= NF) {
    fine_consume(a, Sp, jp, c);
  } else {
    const FineLevel& L = a.lv[I];
    const int runs_parent = (I == 0) ? 1 : a.lv[I > 0 ? I - 1 : 0].runs;
    const int q0 = (I == 0) ? c.grp : 0, qs = (I == 0) ? 2 : 1;  // top level split over the 2 groups
    for (int qf = q0; qf < L.fan; qf += qs) {
      const int j = jp + qf * runs_parent;
      double S[8];
      if (I == NF - 1 && L.K == 1) {  // finest level, K = 1: leaf = parent + x a (no copy)
        const double* xs = c.smem + L.xs_off + (size_t)j * kPad + c.wm * 16 + c.g;
        const double* as = c.as + L.as_off + c.wn * 16 + 2 * c.tg;
        const double x0 = xs[0], x1 = xs[8];
        const double2 p0 = *reinterpret_cast<const double2*>(as);
        const double2 p1 = *reinterpret_cast<const double2*>(as + 8);
        S[0] = fma(x0, p0.x, Sp[0]); S[1] = fma(x0, p0.y, Sp[1]);
        S[2] = fma(x0, p1.x, Sp[2]); S[3] = fma(x0, p1.y, Sp[3]);
        S[4] = fma(x1, p0.x, Sp[4]); S[5] = fma(x1, p0.y, Sp[5]);
        S[6] = fma(x1, p1.x, Sp[6]); S[7] = fma(x1, p1.y, Sp[7]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) S[e] = Sp[e];
        fine_product(L, j, c, S);
      }
      fine_level<I + 1, NF>(a, S, j, c);
    }
  }
}

template <int NF>
__global__ void __launch_bounds__(kFineThreads, 1) k_fine(const FineArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  FineCtx c;
  c.smem = smem;
  c.grp = warp >> 2;
  c.wm = (warp >> 1) & 1;
  c.wn = warp & 1;
  c.g = lane >> 2;
  c.tg = lane & 3;
  c.r0 = (int64_t)blockIdx.x * kBundle;
  c.beff = (int)((a.Mroot - c.r0) < kBundle ? (a.Mroot - c.r0) : kBundle);

  // X^red of the subtree -> smem [run][q][t] (t stride kPad); global rows r0 + t + j Mroot, read
  // row-contiguously (t-major), written transposed.
  for (int i = 0; i < NF; ++i) {
    const FineLevel& L = a.lv[i];
    double* xs = smem + L.xs_off;
    const int per_run = kBundle * L.K;
    for (int e = tid; e < L.runs * per_run; e += kFineThreads) {
      const int j = e / per_run, rem = e - j * per_run, t = rem / L.K, q = rem - t * L.K;
      double v = 0.0;
      if (t < c.beff) v = L.X[(c.r0 + t + (int64_t)j * a.Mroot) * L.ldx + q];
      xs[((size_t)j * L.K + q) * kPad + t] = v;
    }
  }
  if (a.fk >= 0)
    for (int e = tid; e < 2 * a.leafruns * kBundle; e += kFineThreads) smem[a.acc_off + e] = 0.0;

  // A slab of all fine levels for one column tile: [q][c] (c stride kPad), cp.async double buffer
  auto load_a = [&](int buf, int c0) {
    double* as = smem + buf * a.as_stride;
    for (int i = 0; i < NF; ++i) {
      const FineLevel& L = a.lv[i];
      if (a.a_vec) {
        for (int e = tid; e < L.K * (kFineBN / 2); e += kFineThreads) {
          const int q = e / (kFineBN / 2), cc = (e % (kFineBN / 2)) * 2;
          const bool ok = c0 + cc < a.tau;
          const double* src = ok ? a.A + (int64_t)(L.j_lo + q) * a.lda + c0 + cc : a.A;
          cp_async16(as + L.as_off + q * kPad + cc, src, ok);
        }
      } else {
        for (int e = tid; e < L.K * kFineBN; e += kFineThreads) {
          const int q = e / kFineBN, cc = e % kFineBN;
          const bool ok = c0 + cc < a.tau;
          const double* src = ok ? a.A + (int64_t)(L.j_lo + q) * a.lda + c0 + cc : a.A;
          cp_async8(as + L.as_off + q * kPad + cc, src, ok);
        }
      }
    }
    cp_async_commit();
  };

  const int ntiles = (a.tau + kFineBN - 1) / kFineBN;
  auto load_root = [&](double (&R)[8], int c0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) R[e] = 0.0;
    if (!a.root) return;
#pragma unroll
    for (int rf = 0; rf < 2; ++rf) {
      const int t = c.wm * 16 + rf * 8 + c.g;
      if (t >= c.beff) continue;
      const double* p = a.root + (c.r0 + t) * a.ldroot + c0;
#pragma unroll
      for (int cf = 0; cf < 2; ++cf) {
        const int col = c.wn * 16 + cf * 8 + 2 * c.tg;
        if (c0 + col < a.tau) R[rf * 4 + cf * 2] = p[col];
        if (c0 + col + 1 < a.tau) R[rf * 4 + cf * 2 + 1] = p[col + 1];
      }
    }
  };

  if (NF > 0) load_a(0, 0);
  double Rnext[8];
  load_root(Rnext, 0);
  for (int ct = 0; ct < ntiles; ++ct) {
    c.c0 = ct * kFineBN;
    c.as = smem + (ct & 1) * a.as_stride;
    double Sroot[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) Sroot[e] = Rnext[e];
    if (NF > 0) {
      if (ct + 1 < ntiles) {
        load_a((ct + 1) & 1, (ct + 1) * kFineBN);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    }
    __syncthreads();  // A slab of this tile (and X, rowacc on the first pass) visible
    if (ct + 1 < ntiles) load_root(Rnext, (ct + 1) * kFineBN);
    if (NF > 0 || c.grp == 0) fine_level<0, NF>(a, Sroot, 0, c);
    __syncthreads();  // buffer (ct & 1) is refilled at iteration ct + 1
  }

  if (a.fk >= 0) {
    // F(tau^-1 sum_c g) per leaf row, then a fixed-order CTA reduction -> partial[bundle]
    double part = 0.0;
    for (int e = tid; e < a.leafruns * kBundle; e += kFineThreads) {
      const int t = e % kBundle;
      if (t >= c.beff) continue;
      const double rs = smem[a.acc_off + e] + smem[a.acc_off + a.leafruns * kBundle + e];
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

template <int NF>
static cudaError_t launch_fine_t(const FineArgs& a, int64_t nb, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_fine<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
  if (e != cudaSuccess) return e;
  k_fine<NF><<<(unsigned)nb, kFineThreads, a.smem_bytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fine(const FineArgs& a, int64_t nb, cudaStream_t st) {
  switch (a.NF) {
    case 0: return launch_fine_t<0>(a, nb, st);
    case 1: return launch_fine_t<1>(a, nb, st);
    case 2: return launch_fine_t<2>(a, nb, st);
    case 3: return launch_fine_t<3>(a, nb, st);
    case 4: return launch_fine_t<4>(a, nb, st);
    case 5: return launch_fine_t<5>(a, nb, st);
    case 6: return launch_fine_t<6>(a, nb, st);
    case 7: return launch_fine_t<7>(a, nb, st);
    case 8: return launch_fine_t<8>(a, nb, st);
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
