// a3+a4 coarse level GEMM (k_level_gemm); PAPER.md P:n.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstdlib>
#include <type_traits>

#include "rqmc_device.cuh"

namespace rqmc {

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

}  // namespace rqmc
