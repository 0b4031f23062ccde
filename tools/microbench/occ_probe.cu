// How many warps per SM x independent accumulator chains does it take to saturate the fp64 tensor
// pipe (DMMA.8x8x4) and the DFMA pipe on B200?  One CTA per SM (grid = 148), W warps per CTA.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_dmma(double* out, int iters) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = 0.0; acc[c][1] = 0.0; }
  double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.9999999;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1.2345) out[0] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = c * 1e-3;
  double a = 0.9999999 + threadIdx.x * 1e-9, b = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1.2345) out[0] = s;
}

template <int CH>
float run(bool mma, int warps, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto go = [&]() {
    if (mma) k_dmma<CH><<<148, warps * 32>>>(out, iters);
    else k_dfma<CH><<<148, warps * 32>>>(out, iters);
  };
  go(); cudaDeviceSynchronize();
  cudaEventRecord(e0); go(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = mma ? 148.0 * warps * iters * CH * 512.0 : 148.0 * warps * 32 * iters * CH * 2.0;
  return (float)(flops / ms / 1e9);
}

int main() {
  double* out; cudaMalloc(&out, 64);
  for (int w : {4, 8, 12, 16}) {
    printf("{\"probe\":\"occupancy\",\"op\":\"dmma\",\"warps_per_sm\":%d,\"tflops_by_chains\":{\"1\":%.2f,\"2\":%.2f,\"4\":%.2f,\"8\":%.2f}}\n", w,
           run<1>(true, w, 2048, out), run<2>(true, w, 2048, out), run<4>(true, w, 1024, out), run<8>(true, w, 512, out));
    printf("{\"probe\":\"occupancy\",\"op\":\"dfma\",\"warps_per_sm\":%d,\"tflops_by_chains\":{\"1\":%.2f,\"2\":%.2f,\"4\":%.2f,\"8\":%.2f}}\n", w,
           run<1>(false, w, 8192, out), run<2>(false, w, 8192, out), run<4>(false, w, 4096, out), run<8>(false, w, 2048, out));
  }
  return 0;
}
