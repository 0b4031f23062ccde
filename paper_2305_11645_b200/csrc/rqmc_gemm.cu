// a3+a4 coarse level GEMM (k_level_gemm): one level of paper Alg. 2,
// R_w = tile(R_w') + X^red_w A_w, as a DMMA.8x8x4 (fp64 tensor core) GEMM -- optionally fused with
// the next finer level (R_c = tile(R_w) + X^red_c A_c) so that R_w never goes to HBM.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "rqmc_device.cuh"

namespace rqmc {

// ------------------------------------------------------------------------------------------
// R[r, c] = Rp[r mod Mp, c] + sum_q X[r, q] A[q, c]   (the accumulator starts from the parent row)
//
// CTA tile BM x 64, k-tile 16, 2-stage cp.async ring with one barrier per k-tile, warps
// (BM / 8 WMF) x 2 each (8 WMF) x 32 = WMF x 4 DMMA fragments.  Measured on C5 (ncu, per level):
// BM = 64 (4 CTAs per SM) beats 128 (2 per SM) on every level (13.5 vs 14.1 ms) and 32; 3 stages
// equal, 4 stages and BK = 32 slower; WMF = 8 (64 x 32 warp tiles) slower.
// Row blocks are ordered sibling-first: CTA y = pb * nu + u covers rows u Mp + pb BM + [0, BM), so the
// nu = M / Mp child blocks of one parent block run back to back and all but the first read the
// parent tile from L2 (the parent R is read from HBM once instead of nu times).
//
// Pair mode (a.Xc != nullptr): the tile of R_w stays in registers and seeds the GEMMs of the next
// finer level c (parent w, M_c = ncu * M_w): for u < ncu, R_c[u M_w + r] = R_w[r] + X_c[u M_w + r] A_c.
// The arithmetic (accumulator initialised with the parent value, DMMA k-steps in increasing k) is
// exactly that of two separate launches, so the result is bit-identical; R_w's HBM write and
// re-read disappear.
// ------------------------------------------------------------------------------------------
#ifndef RQMC_GEMM_STAGES
#define RQMC_GEMM_STAGES 2
#endif
#ifndef RQMC_GEMM_SIBLING
#define RQMC_GEMM_SIBLING 1
#endif
#ifndef RQMC_GEMM_BK
#define RQMC_GEMM_BK 16
#endif
#ifndef RQMC_GEMM_WMF
#define RQMC_GEMM_WMF 4
#endif
#ifndef RQMC_GEMM_BN
#define RQMC_GEMM_BN 64
#endif
constexpr int kGemmBN = RQMC_GEMM_BN, kGemmBK = RQMC_GEMM_BK, kGemmStages = RQMC_GEMM_STAGES;
constexpr int kGemmWN = kGemmBN / 32;   // warps along N

template <int BM>
constexpr int gemm_smem_bytes() {
  return (int)sizeof(double) * kGemmStages * (BM * (kGemmBK + 4) + kGemmBK * (kGemmBN + 4));
}

template <int BM, int CH, int WMF, bool PAIR, bool RAG>
__global__ void __launch_bounds__(BM / (8 * WMF) * 32 * kGemmWN) k_level_gemm(const GemmArgs a, int64_t mp_blk, int64_t nu,
                                                                   int64_t y0) {
  pdl_enter();
  constexpr int BN = kGemmBN, BK = kGemmBK, NST = kGemmStages, XS = BK + 4, AS = BN + 4;
  constexpr int NT = BM / (8 * WMF) * 32 * kGemmWN, WR = 8 * WMF;
  extern __shared__ __align__(16) double gsm[];
  double (*Xs)[BM][XS] = reinterpret_cast<double (*)[BM][XS]>(gsm);
  double (*As)[BK][AS] = reinterpret_cast<double (*)[BK][AS]>(gsm + NST * BM * XS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / kGemmWN, wn = warp % kGemmWN, g = lane >> 2, tg = lane & 3;  // warp grid (BM / WR) x WN
  // sibling-first row blocks: rows [rb, rb + BM) of slice u, valid while inside the slice and < M
  const int64_t yb = y0 + blockIdx.y;  // grid.y <= 65535: long levels launch in chunks
  const int64_t pb = (int64_t)((uint32_t)yb / (uint32_t)nu), u = yb - pb * nu;  // 32-bit: yb < 2^31, nu small
  const int64_t in0 = pb * BM;                       // offset inside the slice
  const int64_t r0 = u * mp_blk + in0;               // first row of the tile
  const int64_t rlim = min(a.M, u * mp_blk + mp_blk);  // rows >= rlim belong to another tile
  const int c0 = blockIdx.x * BN;
  // replica blockIdx.z (batched randomisation): its own X^red and R buffers, shared A
  const int64_t zr = blockIdx.z;
  const double* __restrict__ Rpg = a.Rp ? a.Rp + zr * a.rrep : nullptr;

  // one GEMM into acc: rows rbase + [0, BM) (valid below rl) of X (ldx, K columns) times A (K rows)
  auto gemm = [&](const double* X, int64_t ldx, int K, const double* A, int64_t rbase, int64_t rl,
                  double (&acc)[WMF][4][2]) {
    // each thread's chunks are fixed (row, column) pairs: rows xr + u XRP of X, rows ar + u ARP of A
    constexpr int XCPR = BK / 2, XRP = NT / XCPR, ACPR = BN / CH, ARP = NT / ACPR;
    static_assert(NT % XCPR == 0 && NT % ACPR == 0, "loader shape");
    const int xr = tid / XCPR, xk = (tid % XCPR) * 2, ar = tid / ACPR, ac = (tid % ACPR) * CH;
    const double* Xt = X + (rbase + xr) * ldx + xk;
    const double* At = A + (int64_t)ar * a.lda + c0 + ac;
    const bool acol = c0 + ac < a.tau;
    auto load_stage = [&](int buf, int k0) {
      // X tile: BM rows x BK cols (ldx even: 16B chunks stay inside the zero-padded row)
      const bool kok = k0 + xk < ldx;
#pragma unroll
      for (int u = 0; u < BM / XRP; ++u) {
        const bool ok = kok && rbase + xr + u * XRP < rl;
        cp_async16(&Xs[buf][xr + u * XRP][xk], ok ? Xt + (int64_t)u * XRP * ldx + k0 : X, ok);
      }
      // A tile: BK rows x BN cols
#pragma unroll
      for (int u = 0; u < BK / ARP; ++u) {
        const bool ok = acol && k0 + ar + u * ARP < K;
        const double* src = ok ? At + (int64_t)(k0 + u * ARP) * a.lda : A;
        if (CH == 2) cp_async16(&As[buf][ar + u * ARP][ac], src, ok);
        else cp_async8(&As[buf][ar + u * ARP][ac], src, ok);
      }
    };
    const int nk = (K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
      if (s < nk) load_stage(s, s * BK);
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<NST - 2>();
      __syncthreads();  // stage kt landed for all threads; stage kt-1's buffer is free
      if (kt + NST - 1 < nk) load_stage((kt + NST - 1) % NST, (kt + NST - 1) * BK);
      cp_async_commit();
      const int buf = kt % NST;
      auto kstep = [&](int kk) {
        double af[WMF], bf[4];
#pragma unroll
        for (int i = 0; i < WMF; ++i) af[i] = Xs[buf][wm * WR + i * 8 + g][kk + tg];
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) bf[jn] = As[buf][kk + tg][wn * 32 + jn * 8 + g];
#pragma unroll
        for (int i = 0; i < WMF; ++i)
#pragma unroll
          for (int jn = 0; jn < 4; ++jn) dmma(acc[i][jn], af[i], bf[jn]);
      };
      // RAG (K % BK != 0): a ragged last tile runs ceil(kl/4) k-steps -- its zero padding would only
      // add exact zeros (C4's K = 54, 162: 12 %, 7 % of the MACs); compile-time so that the K % BK == 0
      // levels keep the branch-free loop (C5 coarse 12.35 vs 12.47 ms)
      const int kl = RAG ? K - kt * BK : BK;
      if (kl >= BK) {
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) kstep(kk);
      } else {
#pragma unroll 1
        for (int kk = 0; kk < kl; kk += 4) kstep(kk);
      }
    }
    cp_async_wait<0>();
    if constexpr (PAIR) __syncthreads();  // the stage buffers are refilled by the next gemm() of this CTA
  };
  auto store = [&](double* R, int64_t ldr, int64_t rbase, int64_t rl, const double (&acc)[WMF][4][2]) {
#pragma unroll
    for (int i = 0; i < WMF; ++i) {
      const int64_t row = rbase + wm * WR + i * 8 + g;
      if (row >= rl) continue;
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {
        const int col = c0 + wn * 32 + jn * 8 + 2 * tg;
        double* p = R + row * ldr + col;
        if (col < a.tau) RQMC_DCHECK(p, col + 1 < a.tau ? 16 : 8);
        if (col + 1 < a.tau) {
          *reinterpret_cast<double2*>(p) = make_double2(acc[i][jn][0], acc[i][jn][1]);
        } else if (col < a.tau) {
          p[0] = acc[i][jn][0];
        }
      }
    }
  };

  double acc[WMF][4][2];
#pragma unroll
  for (int i = 0; i < WMF; ++i) {
    const int64_t row = r0 + wm * WR + i * 8 + g;
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      const int col = c0 + wn * 32 + jn * 8 + 2 * tg;
      acc[i][jn][0] = 0.0;
      acc[i][jn][1] = 0.0;
      if (Rpg && row < rlim) {  // tile(R_w'): row r reads parent row r mod M_w'
        // sibling-first tiles (mp_blk = Mp) lie inside one period: r mod Mp = in0 + (r - r0)
        const int64_t prow = (mp_blk == a.Mp) ? in0 + (row - r0) : row % a.Mp;
        const double* p = Rpg + prow * a.ldp + col;
        if (col < a.tau) RQMC_DCHECK(p, col + 1 < a.tau ? 16 : 8);
        if (CH == 2 && col + 1 < a.tau) {
          const double2 v = *reinterpret_cast<const double2*>(p);
          acc[i][jn][0] = v.x;
          acc[i][jn][1] = v.y;
        } else {
          if (col < a.tau) acc[i][jn][0] = p[0];
          if (col + 1 < a.tau) acc[i][jn][1] = p[1];
        }
      }
    }
  }
  gemm(a.X + zr * a.xrep, a.ldx, a.K, a.A, r0, rlim, acc);
  if constexpr (!PAIR) {
    store(a.R + zr * a.rrep, a.ldr, r0, rlim, acc);
  } else {
    // children of this tile's rows in level c: rows uc M + r, uc < ncu (tile(R_w) for level c)
    for (int uc = 0; uc < a.ncu; ++uc) {
      double acc2[WMF][4][2];
#pragma unroll
      for (int i = 0; i < WMF; ++i)
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) {
          acc2[i][jn][0] = acc[i][jn][0];
          acc2[i][jn][1] = acc[i][jn][1];
        }
      const int64_t cb = (int64_t)uc * a.M + r0, cl = (int64_t)uc * a.M + rlim;
      gemm(a.Xc + zr * a.xrep, a.ldxc, a.Kc, a.Ac, cb, cl, acc2);
      store(a.Rc + zr * a.rrep, a.ldr, cb, cl, acc2);
    }
  }
}

// ------------------------------------------------------------------------------------------
// TMA variant (levels with K >= 128; north_star "tiles of A staged through TMA and shared memory"): the
// X^red tile (64 rows x 16 k) and the A tile (16 k x 64 columns, four 16 x 16 boxes) of each k-tile are
// brought in by cp.async.bulk.tensor with 128-byte swizzle, completing on one mbarrier per stage
// (3-stage ring, thread 0 issues); the 4 warps read the DMMA fragments through the swizzle.  Same
// arithmetic and k order as k_level_gemm (bit-identical R; a ragged last k-tile multiplies the
// zero fill).  Single replica, 16-byte aligned A / lda even, 64-row slices.
// ------------------------------------------------------------------------------------------
constexpr int kTmaStages = 3;
constexpr int kTmaStageBytes = 64 * 16 * 8 + 4 * 16 * 16 * 8;   // X tile + 4 A boxes = 16 KB

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

template <int WMF>
__global__ void __launch_bounds__(128) k_level_gemm_tma(const GemmArgs a, const __grid_constant__ CUtensorMap tmX,
                                                         const __grid_constant__ CUtensorMap tmA, int64_t mp_blk,
                                                         int64_t nu, int64_t y0) {
  pdl_enter();
  constexpr int BM = 64, BN = 64, BK = 16, NST = kTmaStages, WR = 8 * WMF;
  extern __shared__ __align__(1024) unsigned char tsm[];
  __shared__ __align__(8) uint64_t bar[NST];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / 2, wn = warp % 2, g = lane >> 2, tg = lane & 3;
  const int64_t yb = y0 + blockIdx.y;
  const int64_t pb = (int64_t)((uint32_t)yb / (uint32_t)nu), u = yb - pb * nu;
  const int64_t in0 = pb * BM, r0 = u * mp_blk + in0;
  const int64_t rlim = min(a.M, u * mp_blk + mp_blk);
  const int c0 = blockIdx.x * BN;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm) + 1023) & ~uintptr_t(1023));
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nk = (a.K + BK - 1) / BK;   // a ragged last tile: TMA zero-fills rows >= K of A and
                                        // columns >= ldx of X^red (k_gen zeroes [s_w, ldx))
  auto issue = [&](int kt) {   // thread 0: stage kt's X tile and A boxes
    unsigned char* sb = base + (kt % NST) * kTmaStageBytes;
    uint64_t* b = &bar[kt % NST];
    mbar_expect_tx(b, kTmaStageBytes);
    tma_load_2d(sb, &tmX, kt * BK, (int)r0, b);
#pragma unroll
    for (int q = 0; q < 4; ++q) tma_load_2d(sb + 8192 + q * 2048, &tmA, c0 + 16 * q, kt * BK, b);
  };
  if (tid == 0)
    for (int s = 0; s < NST - 1 && s < nk; ++s) issue(s);

  double acc[WMF][4][2];
#pragma unroll
  for (int i = 0; i < WMF; ++i) {
    const int64_t row = r0 + wm * WR + i * 8 + g;
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      const int col = c0 + wn * 32 + jn * 8 + 2 * tg;
      acc[i][jn][0] = 0.0;
      acc[i][jn][1] = 0.0;
      if (a.Rp && row < rlim) {
        const int64_t prow = (mp_blk == a.Mp) ? in0 + (row - r0) : row % a.Mp;
        const double* p = a.Rp + prow * a.ldp + col;
        if (col < a.tau) RQMC_DCHECK(p, col + 1 < a.tau ? 16 : 8);
        if (col + 1 < a.tau) {
          const double2 v = *reinterpret_cast<const double2*>(p);
          acc[i][jn][0] = v.x;
          acc[i][jn][1] = v.y;
        } else if (col < a.tau) {
          acc[i][jn][0] = p[0];
        }
      }
    }
  }
  for (int kt = 0; kt < nk; ++kt) {
    mbar_wait(&bar[kt % NST], (unsigned)((kt / NST) & 1));
    __syncthreads();   // every warp is past stage kt-1: its buffer may be refilled
    if (tid == 0 && kt + NST - 1 < nk) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(kt + NST - 1);
    }
    const unsigned char* sx = base + (kt % NST) * kTmaStageBytes;
    const unsigned char* sa = sx + 8192;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int k = kk + tg;
      double af[WMF], bf[4];
#pragma unroll
      for (int i = 0; i < WMF; ++i) {   // X[row][k], row & 7 = g: 128-byte swizzle XORs the 16-byte chunk
        const int row = wm * WR + i * 8 + g;
        const int off = row * 128 + ((((k >> 1) ^ g) & 7) << 4) + ((k & 1) << 3);
        af[i] = *reinterpret_cast<const double*>(sx + off);
      }
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {  // A[k][col] in box col / 16, row k
        const int col = wn * 32 + jn * 8 + g, c16 = col & 15;
        const int off = (col >> 4) * 2048 + k * 128 + ((((c16 >> 1) ^ k) & 7) << 4) + ((c16 & 1) << 3);
        bf[jn] = *reinterpret_cast<const double*>(sa + off);
      }
#pragma unroll
      for (int i = 0; i < WMF; ++i)
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) dmma(acc[i][jn], af[i], bf[jn]);
    }
  }
#pragma unroll
  for (int i = 0; i < WMF; ++i) {
    const int64_t row = r0 + wm * WR + i * 8 + g;
    if (row >= rlim) continue;
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      const int col = c0 + wn * 32 + jn * 8 + 2 * tg;
      double* p = a.R + row * a.ldr + col;
      if (col < a.tau) RQMC_DCHECK(p, col + 1 < a.tau ? 16 : 8);
      if (col + 1 < a.tau) {
        *reinterpret_cast<double2*>(p) = make_double2(acc[i][jn][0], acc[i][jn][1]);
      } else if (col < a.tau) {
        p[0] = acc[i][jn][0];
      }
    }
  }
}

// 2-D tensor map of a row-major fp64 matrix (rows x cols, leading dimension ld), box bc x br, 128-byte
// swizzle, out-of-bounds elements read as zero
static bool make_tmap(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld, int bc, int br) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static cudaError_t launch_gemm_tma(const GemmArgs& a, int64_t mp_blk, int64_t nu, int64_t nrb, cudaStream_t st) {
  CUtensorMap tx, ta;
  if (!make_tmap(&tx, a.X, a.M, a.ldx, a.ldx, 16, 64) || !make_tmap(&ta, a.A, a.K, a.tau, a.lda, 16, 16))
    return cudaErrorNotSupported;
  constexpr int WMF = 4;
  const int sm = kTmaStages * kTmaStageBytes + 1024;
  cudaError_t e = set_smem_once(k_level_gemm_tma<WMF>, sm);
  if (e != cudaSuccess) return e;
  for (int64_t y0 = 0; y0 < nrb; y0 += 65535) {
    dim3 grid((unsigned)((a.tau + 63) / 64), (unsigned)std::min<int64_t>(65535, nrb - y0), 1);
    if ((e = launch_k(k_level_gemm_tma<WMF>, grid, dim3(128), sm, st, true, a, tx, ta, mp_blk, nu, y0)) != cudaSuccess)
      return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------------------------------
// Latency-regime variant (levels under one wave of 64 x 64 tiles with <= kLatMacs multiply-adds: C2's
// coarse chain, C1): a level that small is its launch, load and store latency plus the DMMA chain of
// one warp (C2's K = 128 level: 32 CTAs of 64 x 64, 512 DMMAs per warp, 9 us).  32 x 32 CTA tiles of
// 4 warps (2 x 2 warps of 16 x 16 = 2 x 2 DMMA fragments) spread it over 4x the SMs with 4x fewer
// DMMAs per warp; k-tile 16 on a deep cp.async ring (launch_lat_t).  GATHER: the X operand of merged coarse levels
// is read from each level's own X^red (GemmArgs::nseg) -- k_gen generates no extra points.  Same
// accumulation as k_level_gemm (parent row first, k-steps in increasing k).
// ------------------------------------------------------------------------------------------
constexpr double kLatMacs = 67108864.0;   // 2^26 multiply-adds (~3.6 us at the fp64 peak)

constexpr int kLatStage = 32 * 20 + 16 * 36;   // doubles per stage: X tile (pitch 20) + A tile (pitch 36)

template <bool GATHER, int CH, int NST>
__global__ void __launch_bounds__(128) k_level_gemm_lat(const GemmArgs a) {
  pdl_enter();
  constexpr int BM = 32, BN = 32, BK = 16, XS = BK + 4, AS = BN + 4;   // pitches: conflict-free
  extern __shared__ __align__(16) double lsm[];
  double (*Xs)[BM][XS] = reinterpret_cast<double (*)[BM][XS]>(lsm);
  double (*As)[BK][AS] = reinterpret_cast<double (*)[BK][AS]>(lsm + NST * BM * XS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, tg = lane & 3;
  const int64_t r0 = (int64_t)blockIdx.y * BM;
  const int c0 = blockIdx.x * BN;
  const int64_t zr = blockIdx.z;   // replica: its own X^red and R buffers, shared A
  const double* __restrict__ Rpg = a.Rp ? a.Rp + zr * a.rrep : nullptr;
  // loader: X tile 32 x 16 = 256 16-byte chunks, two per thread (rows xr, xr + 16; columns xk, xk + 1);
  // A tile 16 x 32: CH = 2 two 16-byte chunks per thread (rows ar, ar + 8), CH = 1 four 8-byte elements
  const int xr = tid >> 3, xk = (tid & 7) * 2;
  const double* Xb = a.X + zr * a.xrep;
  // gather: the thread's column q = k0 + xk only moves forward, so its segment and the two row offsets
  // (row mod M_i) ld_i are recomputed only when q enters the next segment (nseg modulos per thread)
  int seg = -1;
  int64_t soff[2] = {0, 0};
  auto load_stage = [&](int buf, int k0) {
    const int q = k0 + xk;
    if constexpr (GATHER) {
      if (seg < 0 || (seg + 1 < a.nseg && q >= a.segq[seg + 1])) {
        do { ++seg; } while (seg + 1 < a.nseg && q >= a.segq[seg + 1]);
        const uint32_t sm = (uint32_t)a.segM[seg];
#pragma unroll
        for (int u = 0; u < 2; ++u) soff[u] = (int64_t)((uint32_t)(r0 + xr + 16 * u) % sm) * a.segld[seg];
      }
      const double* sx = a.segX[seg] + zr * a.xrep + (q - a.segq[seg]);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const bool ok = r0 + xr + 16 * u < a.M && q < a.segq[a.nseg];
        cp_async16(&Xs[buf][xr + 16 * u][xk], ok ? sx + soff[u] : a.X, ok);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t xrow = r0 + xr + 16 * u;
        const bool ok = xrow < a.M && q < a.ldx;
        cp_async16(&Xs[buf][xr + 16 * u][xk], ok ? Xb + xrow * a.ldx + q : a.X, ok);
      }
    }
    if constexpr (CH == 2) {
      const int ar = tid >> 4, ac = (tid & 15) * 2;
      const bool cok = c0 + ac < a.tau;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + ar + 8 * u;
        const bool ok = cok && k < a.K;
        cp_async16(&As[buf][ar + 8 * u][ac], ok ? a.A + (int64_t)k * a.lda + c0 + ac : a.A, ok);
      }
    } else {
      const int ar = tid >> 5, ac = tid & 31;
      const bool cok = c0 + ac < a.tau;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + ar + 4 * u;
        const bool ok = cok && k < a.K;
        cp_async8(&As[buf][ar + 4 * u][ac], ok ? a.A + (int64_t)k * a.lda + c0 + ac : a.A, ok);
      }
    }
  };
  const int nk = (a.K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < NST - 1; ++s) {
    if (s < nk) load_stage(s, s * BK);
    cp_async_commit();
  }
  // accumulators start from the parent rows (tile(R_w')) -- loaded while the stages fly
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t row = r0 + wm * 16 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = c0 + wn * 16 + j * 8 + 2 * tg;
      acc[i][j][0] = 0.0;
      acc[i][j][1] = 0.0;
      if (Rpg && row < a.M) {
        const double* p = Rpg + (int64_t)((uint32_t)row % (uint32_t)a.Mp) * a.ldp + col;   // M < 2^21 here
        if (col < a.tau) RQMC_DCHECK(p, col + 1 < a.tau ? 16 : 8);
        if (CH == 2 && col + 1 < a.tau) {
          const double2 v = *reinterpret_cast<const double2*>(p);
          acc[i][j][0] = v.x;
          acc[i][j][1] = v.y;
        } else {
          if (col < a.tau) acc[i][j][0] = p[0];
          if (col + 1 < a.tau) acc[i][j][1] = p[1];
        }
      }
    }
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<NST - 2>();
    __syncthreads();   // stage kt landed for all threads; stage kt-1's buffer is free
    if (kt + NST - 1 < nk) load_stage((kt + NST - 1) % NST, (kt + NST - 1) * BK);
    cp_async_commit();
    const int buf = kt % NST, kl = a.K - kt * BK;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if (kk < kl) {   // a ragged last tile runs only its valid k-steps
        double af[2], bf[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) af[i] = Xs[buf][wm * 16 + i * 8 + g][kk + tg];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = As[buf][kk + tg][wn * 16 + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    }
  }
  cp_async_wait<0>();
  double* R = a.R + zr * a.rrep;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t row = r0 + wm * 16 + i * 8 + g;
    if (row >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = c0 + wn * 16 + j * 8 + 2 * tg;
      double* p = R + row * a.ldr + col;
      if (col < a.tau) RQMC_DCHECK(p, col + 1 < a.tau ? 16 : 8);
      if (CH == 2 && col + 1 < a.tau) {
        *reinterpret_cast<double2*>(p) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (col < a.tau) p[0] = acc[i][j][0];
        if (col + 1 < a.tau) p[1] = acc[i][j][1];
      }
    }
  }
}

// stages: up to 10 k-tiles in flight (K <= 176 resident at once; 107 KB, 2 CTAs per SM) when the level
// has more than 4 k-tiles -- each k-tile is only 16 DMMAs per warp, so a shallow ring waits one load
// latency per k-tile (C2's merged K = 193 level: 25 us with 3 stages); 5 stages (48 KB) for K <= 64
template <bool GATHER, int CH>
static cudaError_t launch_lat_t(const GemmArgs& a, dim3 grid, cudaStream_t st) {
  const int nk = (a.K + 15) / 16;
  auto go = [&](auto kern, int nst) -> cudaError_t {
    const int sm = nst * kLatStage * (int)sizeof(double);
    cudaError_t e = set_smem_once(kern, sm);
    if (e != cudaSuccess) return e;
    return launch_k(kern, grid, dim3(128), (size_t)sm, st, true, a);
  };
  if (nk <= 4) return go(k_level_gemm_lat<GATHER, CH, 5>, 5);
  return go(k_level_gemm_lat<GATHER, CH, 11>, 11);
}

static cudaError_t launch_gemm_lat(const GemmArgs& a, int nrep, bool vec, cudaStream_t st) {
  const dim3 grid((unsigned)((a.tau + 31) / 32), (unsigned)((a.M + 31) / 32), (unsigned)nrep);
  if (grid.y > 65535) return cudaErrorInvalidValue;
  if (a.nseg > 0) return vec ? launch_lat_t<true, 2>(a, grid, st) : launch_lat_t<true, 1>(a, grid, st);
  return vec ? launch_lat_t<false, 2>(a, grid, st) : launch_lat_t<false, 1>(a, grid, st);
}

template <int BM>
static cudaError_t launch_gemm_bm(const GemmArgs& a, int nrep, cudaStream_t st);

cudaError_t launch_gemm(const GemmArgs& a, int nrep, cudaStream_t st) {
  if (a.M == 0 || nrep == 0) return cudaSuccess;
  // 64-row tiles (4 CTAs per SM) everywhere: 32-row tiles for levels under 2 waves (one rank's share
  // of C5 on 8 GPUs) measured slower (per-rank 4.08 vs 4.04 ms)
#ifdef RQMC_GEMM_BM
  return launch_gemm_bm<RQMC_GEMM_BM>(a, nrep, st);
#else
  return launch_gemm_bm<64>(a, nrep, st);
#endif
}

template <int BM>
static cudaError_t launch_gemm_bm(const GemmArgs& a, int nrep, cudaStream_t st) {
  const bool pair = a.Xc != nullptr;
  if (pair && a.nseg > 0) return cudaErrorNotSupported;   // only k_level_gemm_lat gathers
  const bool vec = ((uintptr_t)a.A % 16 == 0) && (a.lda % 2 == 0) && (a.tau % 2 == 0) &&
                   (!pair || ((uintptr_t)a.Ac % 16 == 0)) &&
                   (a.Rp == nullptr || (((uintptr_t)a.Rp % 16 == 0) && a.ldp % 2 == 0));
  constexpr int WMF = RQMC_GEMM_WMF, NT = BM / (8 * WMF) * 32 * kGemmWN;
  // sibling-first ordering when the parent has at least one full row block; else plain row blocks
  int64_t mp_blk = a.M, nu = 1;
  if (RQMC_GEMM_SIBLING && a.Rp && a.Mp >= BM && a.Mp < a.M) {
    mp_blk = a.Mp;
    nu = (a.M + a.Mp - 1) / a.Mp;
  }
  const int64_t nrb = (mp_blk + BM - 1) / BM * nu;
  // latency regime (k_level_gemm_lat): under one wave of 64 x 64 tiles and <= kLatMacs, or a gathered
  // GEMM of merged coarse levels (only that kernel gathers).  RQMC_GEMM_LAT=0 disables (gathered
  // GEMMs still use it), =1 forces every single-level GEMM onto it.
  const char* le = std::getenv("RQMC_GEMM_LAT");   // read per launch (tests switch it; graphs capture once)
  const int lat_mode = le && *le ? std::atoi(le) : -1;
  const int64_t ncta64 = nrb * ((a.tau + 63) / 64) * nrep;
  const double macs = (double)a.M * a.tau * a.K * nrep;
  if (!pair && (a.nseg > 0 || lat_mode == 1 || (lat_mode < 0 && ncta64 < 592 && macs <= kLatMacs)))
    return launch_gemm_lat(a, nrep, vec, st);
  // TMA tiles for K >= 128 (C5 levels 7..11: 2.01-2.07 vs 2.07-2.10 ms, tensor pipe 93.5-94.7 % vs
  // 91.2-91.8 %: the 128-byte swizzle leaves 2-way bank conflicts on the 8-byte fragment loads
  // (l1tex wavefronts x2), but the loader's address arithmetic disappears (-18 % instructions)); the
  // K = 64 level (4 k-tiles, R-traffic bound) is faster on cp.async (2.18 vs 2.28 ms;
  // profiles/r02_gemm_tma_C5.txt).  RQMC_GEMM_TMA=0 disables, =1 forces every eligible level.
  static const int tma_mode = [] { const char* e = std::getenv("RQMC_GEMM_TMA"); return e && *e ? std::atoi(e) : -1; }();
  // (and at least one full wave of 592 CTAs: on small grids the 3-stage TMA prologue is exposed, C2's
  // K = 128 level 12.6 us vs ~9 us)
  const int64_t ncta = nrb * ((a.tau + 63) / 64);
  const bool use_tma = tma_mode == 1 || (tma_mode < 0 && a.K >= 128 && ncta >= 592);
  if (use_tma && BM == 64 && !pair && vec && nrep == 1 && mp_blk % 64 == 0 && a.ldx % 2 == 0 &&
      a.M < (int64_t(1) << 31) &&
      (uintptr_t)a.X % 16 == 0) {
    const cudaError_t e = launch_gemm_tma(a, mp_blk, nu, nrb, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const int sm = gemm_smem_bytes<BM>();
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = set_smem_once(kern, sm);
    if (e != cudaSuccess) return e;
    // grid.x = column blocks (fastest: the CTAs of one row block share its X^red rows in L2)
    for (int64_t y0 = 0; y0 < nrb; y0 += 65535) {
      dim3 grid((unsigned)((a.tau + kGemmBN - 1) / kGemmBN), (unsigned)std::min<int64_t>(65535, nrb - y0),
                (unsigned)nrep);
      if (cudaError_t e = launch_k(kern, grid, dim3(NT), sm, st, true, a, mp_blk, nu, y0)) return e;
    }
    return cudaGetLastError();
  };
  if (pair) return vec ? go(k_level_gemm<BM, 2, WMF, true, false>) : go(k_level_gemm<BM, 1, WMF, true, false>);
  if (a.K % kGemmBK != 0)
    return vec ? go(k_level_gemm<BM, 2, WMF, false, true>) : go(k_level_gemm<BM, 1, WMF, false, true>);
  return vec ? go(k_level_gemm<BM, 2, WMF, false, false>) : go(k_level_gemm<BM, 1, WMF, false, false>);
}

#if RQMC_DEBUG
cudaError_t dbg_set_gemm(const DbgRanges& r, cudaStream_t st) { return dbg_set_tu(r, st); }
#else
cudaError_t dbg_set_gemm(const DbgRanges&, cudaStream_t) { return cudaSuccess; }
#endif

}  // namespace rqmc
