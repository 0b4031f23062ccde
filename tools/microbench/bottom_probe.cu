// Probe: achievable fp64-pipe rate of the fine kernel's b = 2 bottom block instruction mix on B200.
// One iteration = one bottom block of k_fine_tree (NQ = 2): 2 K = 4 nodes (4 DMMA.8x8x4 each from
// the parent tile), 4 K = 2 nodes (16 DFMA each, cached A), 8 leaves (8 DFMA + 7 DADD each), the
// transpose-reduce (6 SHFL + 6 DADD) and the register row-sum update; x values come from smem.
// Variants isolate the parts.  Pipe cycles per iteration per warp: 8*16 + (64+64+62)*2 = 508.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bottom_probe bottom_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// V: 0 full, 1 no DMMA (K=4 nodes as a copy), 2 no sums (leaves consumed by one DADD chain per leaf pair),
//    3 DMMA K=4 nodes + DMMA-padded K=2 (no DFMA K=2)
template <int V>
__global__ void __launch_bounds__(256) k_bottom(double* out, int iters, const double* xin) {
  __shared__ double xs[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = xin[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, tg = lane & 3;
  double S3[8], bk[4], a1[2][8], a0[8], racc[2] = {0.0, 0.0};
#pragma unroll
  for (int e = 0; e < 8; ++e) { S3[e] = 1e-3 * e + lane; a1[0][e] = 0.5 + e; a1[1][e] = 0.25 - e; a0[e] = 0.125 * e; }
#pragma unroll
  for (int cf = 0; cf < 4; ++cf) bk[cf] = 0.1 * cf + tg;
  const int base = (lane & 31);
  for (int it = 0; it < iters; ++it) {
    const int o = ((it * 37) & 15) * 64 + base;
    double v[8];
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      double S2[8];
      const double x2 = xs[o + n * 32];
      if constexpr (V == 1) {
#pragma unroll
        for (int e = 0; e < 8; ++e) S2[e] = S3[e] + x2;
      } else {
#pragma unroll
        for (int cf = 0; cf < 4; ++cf) dmma_c(S2[2 * cf], S2[2 * cf + 1], x2, bk[cf], S3[2 * cf], S3[2 * cf + 1]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double S1[8];
        const double xa = xs[o + 1024 + n * 64 + h * 32], xb = xs[o + 1024 + n * 64 + h * 32 + 8];
        if constexpr (V == 3) {
          const double af = tg < 2 ? xa : 0.0;
#pragma unroll
          for (int cf = 0; cf < 4; ++cf) dmma_c(S1[2 * cf], S1[2 * cf + 1], af, bk[cf], S2[2 * cf], S2[2 * cf + 1]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) S1[e] = fma(xb, a1[1][e], fma(xa, a1[0][e], S2[e]));
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double x0 = xs[o + 2048 + n * 128 + h * 64 + q * 32];
          double Y[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) Y[e] = fma(x0, a0[e], S1[e]);
          if constexpr (V == 2) {
            v[4 * n + 2 * h + q] = Y[0] + Y[7];
          } else {
            v[4 * n + 2 * h + q] = ((Y[0] + Y[1]) + (Y[2] + Y[3])) + ((Y[4] + Y[5]) + (Y[6] + Y[7]));
          }
        }
      }
    }
    const bool hi1 = (tg & 2) != 0, hi0 = (tg & 1) != 0;
    double u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double keep = hi1 ? v[i + 4] : v[i];
      const double send = hi1 ? v[i] : v[i + 4];
      u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double keep = hi0 ? u[i + 2] : u[i];
      const double send = hi0 ? u[i] : u[i + 2];
      racc[i] += keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) S3[e] = S3[e] * 0.999 ;  // next parent tile (1 DMUL per element)
  }
  if (racc[0] + racc[1] == 12345.678) out[0] = racc[0];
}

template <int V>
float run(int ctas_per_sm, int iters, double* out, const double* x) {
  int sms = 148;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  k_bottom<V><<<sms * ctas_per_sm, 256>>>(out, iters, x);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  k_bottom<V><<<sms * ctas_per_sm, 256>>>(out, iters, x);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int main() {
  double *out, *x; CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&x, 4096 * 8));
  CK(cudaMemset(x, 0, 4096 * 8));
  const int iters = 4000;
  // pipe cycles per iteration per warp (fp64 datapath: DMMA 16, DFMA/DADD/DMUL 2 per warp instr)
  const double cyc[4] = {8 * 16 + (64 + 64 + 62 + 8) * 2.0, (8 + 64 + 64 + 62 + 8) * 2.0,
                         8 * 16 + (64 + 64 + 8 + 6 + 8) * 2.0, 24 * 16 + (64 + 62 + 8) * 2.0};
  for (int cps = 1; cps <= 2; ++cps) {
    float ms[4] = {run<0>(cps, iters, out, x), run<1>(cps, iters, out, x), run<2>(cps, iters, out, x),
                   run<3>(cps, iters, out, x)};
    for (int v = 0; v < 4; ++v) {
      // per SMSP: warps = 2 * cps, each iters iterations
      const double busy = cyc[v] * iters * 2 * cps / 1.965e6;  // ms if the pipe were 100 % busy at 1.965 GHz
      printf("{\"probe\":\"bottom\",\"variant\":%d,\"warps_per_sm\":%d,\"ms\":%.4f,\"pipe_frac\":%.3f}\n", v,
             8 * cps, ms[v], busy / ms[v]);
    }
  }
  return 0;
}
