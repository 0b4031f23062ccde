// fp64 pipe probes for B200 (sm_100a): fix the roofline denominators of
// SURVEY §8(d) "Microbenchmarks that fix the denominators" (probes 1-6).
//   1. DMMA.8x8x4 throughput (mma.sync m8n8k4 f64)
//   2. DFMA throughput (register-resident chains)
//   3. DMMA + DFMA interleaved (co-issue?)
//   4. HBM copy bandwidth, 5. store-only bandwidth, 6. L2-resident read of 64 MiB
// Prints one JSON line per probe. Standalone: nvcc -gencode arch=compute_100a,code=sm_100a.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a0, double b0) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = 0.0; acc[c][1] = 0.0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double a0, double b0) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = c * 1e-3;
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// interleave: per iteration CH DMMA + F DFMA (per thread)
template <int CH, int F>
__global__ void k_mix(double* out, int iters, double a0, double b0) {
  double acc[CH][2];
  double f[F];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = 0.0; acc[c][1] = 0.0; }
#pragma unroll
  for (int c = 0; c < F; ++c) f[c] = c * 1e-3;
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c], a, b);
#pragma unroll
    for (int c = 0; c < F; ++c) f[c] = fma(f[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
#pragma unroll
  for (int c = 0; c < F; ++c) s += f[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void k_store(double2* __restrict__ b, size_t n, double v) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = make_double2(v, v);
}
__global__ void k_read(const double2* __restrict__ a, size_t n, double* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  double s = 0;
  for (; i < n; i += st) { double2 v = __ldcg(a + i); s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

static float time_it(void (*launch)(void*), void* ctx, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch(ctx); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0)); launch(ctx); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

struct Ctx { double* out; int iters; int blocks; int threads; const double2* a; double2* b; size_t n; };

template <int CH> void L_dmma(void* p) { Ctx* c = (Ctx*)p; k_dmma<CH><<<c->blocks, c->threads>>>(c->out, c->iters, 1.0000001, 0.9999999); }
template <int CH> void L_dfma(void* p) { Ctx* c = (Ctx*)p; k_dfma<CH><<<c->blocks, c->threads>>>(c->out, c->iters, 0.9999999, 1e-7); }
template <int CH, int F> void L_mix(void* p) { Ctx* c = (Ctx*)p; k_mix<CH, F><<<c->blocks, c->threads>>>(c->out, c->iters, 0.9999999, 1e-7); }
void L_copy(void* p) { Ctx* c = (Ctx*)p; k_copy<<<c->blocks, c->threads>>>(c->a, c->b, c->n); }
void L_store(void* p) { Ctx* c = (Ctx*)p; k_store<<<c->blocks, c->threads>>>(c->b, c->n, 1.5); }
void L_read(void* p) { Ctx* c = (Ctx*)p; k_read<<<c->blocks, c->threads>>>(c->a, c->n, c->out); }

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"probe\":\"device\",\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_block_optin\":%zu,"
         "\"regs_per_sm\":%d,\"clock_khz\":%d}\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize,
         pr.sharedMemPerBlockOptin, pr.regsPerMultiprocessor, clk);
  double* out; CK(cudaMalloc(&out, 64));
  int sms = pr.multiProcessorCount;
  Ctx c{out, 4096, sms * 4, 256, nullptr, nullptr, 0};
  // DMMA: flops per thread-iter = CH * 512 / 32 = 16*CH
  for (int warps : {4, 8, 16}) {
    c.threads = warps * 32; c.blocks = sms * 2; c.iters = 4096;
    float ms = time_it(L_dmma<8>, &c, 5);
    double fl = (double)c.blocks * warps * c.iters * 8 * 512.0;
    printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"ctas\":%d,\"chains\":8,\"ms\":%.4f,\"tflops\":%.3f}\n",
           warps, c.blocks, ms, fl / ms / 1e9);
  }
  {
    c.threads = 256; c.blocks = sms * 2; c.iters = 4096;
    float ms = time_it(L_dmma<4>, &c, 5);
    double fl = (double)c.blocks * 8 * c.iters * 4 * 512.0;
    printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_cta\":8,\"ctas\":%d,\"chains\":4,\"ms\":%.4f,\"tflops\":%.3f}\n",
           c.blocks, ms, fl / ms / 1e9);
  }
  for (int warps : {8, 16, 32}) {
    c.threads = warps * 32; c.blocks = sms * 2; c.iters = 4096;
    float ms = time_it(L_dfma<8>, &c, 5);
    double fl = (double)c.blocks * c.threads * c.iters * 8 * 2.0;
    printf("{\"probe\":\"dfma\",\"warps_per_cta\":%d,\"ctas\":%d,\"chains\":8,\"ms\":%.4f,\"tflops\":%.3f}\n",
           warps, c.blocks, ms, fl / ms / 1e9);
  }
  {
    c.threads = 256; c.blocks = sms * 2; c.iters = 4096;
    float ms = time_it(L_mix<8, 8>, &c, 5);
    double fl = (double)c.blocks * 8 * c.iters * (8 * 512.0) + (double)c.blocks * 256 * c.iters * 8 * 2.0;
    printf("{\"probe\":\"dmma+dfma\",\"dmma_per_iter\":8,\"dfma_per_iter\":8,\"ms\":%.4f,\"tflops\":%.3f}\n", ms, fl / ms / 1e9);
    float ms2 = time_it(L_mix<8, 32>, &c, 5);
    double fl2 = (double)c.blocks * 8 * c.iters * (8 * 512.0) + (double)c.blocks * 256 * c.iters * 32 * 2.0;
    printf("{\"probe\":\"dmma+dfma\",\"dmma_per_iter\":8,\"dfma_per_iter\":32,\"ms\":%.4f,\"tflops\":%.3f}\n", ms2, fl2 / ms2 / 1e9);
  }
  // memory probes
  size_t bytes = (size_t)4 << 30;  // 4 GiB per buffer
  double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
  c.a = a; c.b = b; c.n = bytes / 16; c.threads = 256; c.blocks = sms * 8;
  {
    float ms = time_it(L_copy, &c, 5);
    printf("{\"probe\":\"hbm_copy\",\"bytes\":%zu,\"ms\":%.4f,\"gbs\":%.1f}\n", 2 * bytes, ms, 2.0 * bytes / ms / 1e6);
    ms = time_it(L_store, &c, 5);
    printf("{\"probe\":\"hbm_store\",\"bytes\":%zu,\"ms\":%.4f,\"gbs\":%.1f}\n", bytes, ms, 1.0 * bytes / ms / 1e6);
    ms = time_it(L_read, &c, 5);
    printf("{\"probe\":\"hbm_read\",\"bytes\":%zu,\"ms\":%.4f,\"gbs\":%.1f}\n", bytes, ms, 1.0 * bytes / ms / 1e6);
    c.n = ((size_t)64 << 20) / 16;
    ms = time_it(L_read, &c, 20);
    printf("{\"probe\":\"l2_read_64MiB\",\"bytes\":%zu,\"ms\":%.4f,\"gbs\":%.1f}\n", (size_t)64 << 20, ms, 64.0 * (1 << 20) / ms / 1e6);
  }
  return 0;
}
