// Dependent-chain latency of the fp64 instructions the fine kernel is built from (1 warp, 1 CTA):
// DMMA.8x8x4 (C == D chain), DFMA, DADD, SHFL.BFLY of a double, LDS.64.  Prints cycles/op.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, int iters) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = lane;
  __syncwarp();
  double a = 1.0000001 + lane * 1e-9, b = 0.9999999, d0 = 0.0, d1 = 0.0, x = lane * 1e-3;
  long long t0, t1;
  // DMMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  t1 = clock64();
  cyc[1] = t1 - t0;
  // DADD chain
  double y = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = y + b;
  t1 = clock64();
  cyc[2] = t1 - t0;
  // SHFL + DADD chain
  double z = y;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) z += __shfl_xor_sync(0xffffffffu, z, 1);
  t1 = clock64();
  cyc[3] = t1 - t0;
  // LDS chain (pointer chasing through smem index)
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = ((int)sm[idx] + 1) & 31;
  t1 = clock64();
  cyc[4] = t1 - t0;
  out[lane] = d0 + d1 + x + y + z + idx;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * 8); cudaMallocManaged(&cyc, 8 * 8);
  const int iters = 4096;
  k_lat<<<1, 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  k_lat<<<1, 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  const char* names[] = {"dmma_m8n8k4", "dfma", "dadd", "shfl_xor+dadd", "lds+cvt+add"};
  for (int i = 0; i < 5; ++i) printf("{\"probe\":\"latency\",\"op\":\"%s\",\"cycles_per_op\":%.2f}\n", names[i], (double)cyc[i] / iters);
  return 0;
}
