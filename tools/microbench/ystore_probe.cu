// HBM write bandwidth of C4's Y store pattern (the fine kernel's only HBM-heavy stream).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ystore_probe ystore_probe.cu && ./ystore_probe
// C4: N = 3^12 rows x tau = 4096 fp64 (17.4 GB).  The fine kernel's CTA owns a bundle of BUN residues
// r of the checkpoint level (M = 3^9 rows) and writes rows k = r + t M (t < 27) column tile by column
// tile (W columns).  Patterns: "tree" (that order, W = 32 / 64 / 128 / 256), "rows" (each CTA writes
// whole contiguous rows, the streaming ideal).  Prints one JSON line per pattern.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tree_store(double* Y, long M, int tau, int bun, int leaves, int W) {
  const long r0 = (long)blockIdx.x * bun;
  const int nt = blockDim.x;
  const int per_row = W / 2;                              // 16-byte pieces per row segment
  for (int c0 = 0; c0 < tau; c0 += W)
    for (int e = threadIdx.x; e < bun * leaves * per_row; e += nt) {
      const int row = e / per_row, p = e % per_row;
      const long r = r0 + row % bun;
      const long k = r + (long)(row / bun) * M;
      if (r >= M) continue;
      double2 v = make_double2((double)k, (double)c0);
      *reinterpret_cast<double2*>(Y + k * tau + c0 + 2 * p) = v;
    }
}

// 32-byte stores (st.global.v4.f64, STG.256 on sm_100a): each lane writes 4 consecutive doubles
__global__ void tree_store4(double* Y, long M, int tau, int bun, int leaves, int W) {
  const long r0 = (long)blockIdx.x * bun;
  const int nt = blockDim.x;
  const int per_row = W / 4;
  for (int c0 = 0; c0 < tau; c0 += W)
    for (int e = threadIdx.x; e < bun * leaves * per_row; e += nt) {
      const int row = e / per_row, p = e % per_row;
      const long r = r0 + row % bun;
      const long k = r + (long)(row / bun) * M;
      if (r >= M) continue;
      double* q = Y + k * tau + c0 + 4 * p;
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(q), "d"((double)k), "d"((double)c0), "d"(1.0),
                   "d"(2.0) : "memory");
    }
}
__global__ void row_store4(double* Y, long N, int tau) {
  const long n4 = N * tau / 4;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(Y + 4 * i), "d"((double)i), "d"(0.0), "d"(1.0),
                 "d"(2.0) : "memory");
}

// streaming-hint stores (st.global.cs): v2 and v4
template <int V>
__global__ void tree_store_cs(double* Y, long M, int tau, int bun, int leaves, int W) {
  const long r0 = (long)blockIdx.x * bun;
  const int per_row = W / V;
  for (int c0 = 0; c0 < tau; c0 += W)
    for (int e = threadIdx.x; e < bun * leaves * per_row; e += blockDim.x) {
      const int row = e / per_row, p = e % per_row;
      const long r = r0 + row % bun;
      const long k = r + (long)(row / bun) * M;
      if (r >= M) continue;
      double* q = Y + k * tau + c0 + V * p;
      if (V == 2)
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(q), "d"((double)k), "d"((double)c0) : "memory");
      else
        asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(q), "d"((double)k), "d"((double)c0), "d"(1.0),
                     "d"(2.0) : "memory");
    }
}
// bulk copies: each CTA stages its 8-row x W tile of one leaf run in shared memory and writes every row
// segment (8 W bytes) with cp.async.bulk.global.shared::cta (one thread per row)
template <int NB>
__global__ void tree_store_bulk(double* Y, long M, int tau, int bun, int leaves, int W) {
  extern __shared__ __align__(128) double st[];   // NB buffers x bun x W (ring)
  const long r0 = (long)blockIdx.x * bun;
  int buf = 0;
  for (int c0 = 0; c0 < tau; c0 += W)
    for (int j = 0; j < leaves; ++j) {
      double* sb = st + buf * bun * W;
      // the buffer written NB rounds ago has been read by its bulk copies
      if (threadIdx.x < bun) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
      __syncthreads();
      for (int e = threadIdx.x; e < bun * W / 2; e += blockDim.x)
        reinterpret_cast<double2*>(sb)[e] = make_double2((double)j, (double)c0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < bun) {
        const long r = r0 + threadIdx.x;
        if (r < M) {
          const long k = r + (long)j * M;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(Y + k * tau + c0),
                       "r"((unsigned)__cvta_generic_to_shared(sb + threadIdx.x * W)), "r"(W * 8) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      buf = (buf + 1) % NB;
    }
  if (threadIdx.x < bun) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void row_store(double* Y, long N, int tau) {
  const long n2 = N * tau / 2;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x)
    reinterpret_cast<double2*>(Y)[i] = make_double2((double)i, 0.0);
}

int main() {
  const long M = 19683, N = 531441;
  const int tau = 4096, bun = 8, leaves = 27;
  double* Y;
  if (cudaMalloc(&Y, (size_t)N * tau * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = (double)N * tau * 8;
  for (int W : {32, 64, 128, 256}) {
    const int grid = (int)((M + bun - 1) / bun);
    tree_store<<<grid, 96>>>(Y, M, tau, bun, leaves, W);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) tree_store<<<grid, 96>>>(Y, M, tau, bun, leaves, W);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("{\"probe\":\"ystore\",\"pattern\":\"tree\",\"W\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", W, ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
  }
  row_store<<<148 * 8, 256>>>(Y, N, tau);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) row_store<<<148 * 8, 256>>>(Y, N, tau);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\":\"ystore\",\"pattern\":\"rows\",\"ms\":%.4f,\"gbs\":%.1f}\n", ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
  for (int W : {32, 64}) {
    const int grid = (int)((M + bun - 1) / bun);
    tree_store4<<<grid, 96>>>(Y, M, tau, bun, leaves, W);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) tree_store4<<<grid, 96>>>(Y, M, tau, bun, leaves, W);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"probe\":\"ystore\",\"pattern\":\"tree_v4\",\"W\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", W, ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
  }
  auto run = [&](const char* name, int W, auto launch) {
    launch();
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b);
    printf("{\"probe\":\"ystore\",\"pattern\":\"%s\",\"W\":%d,\"ms\":%.4f,\"gbs\":%.1f,\"err\":\"%s\"}\n", name, W,
           t / 5, bytes / (t / 5 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  const int grid = (int)((M + bun - 1) / bun);
  for (int W : {32, 64}) {
    run("tree_cs_v2", W, [&] { tree_store_cs<2><<<grid, 96>>>(Y, M, tau, bun, leaves, W); });
    run("tree_cs_v4", W, [&] { tree_store_cs<4><<<grid, 96>>>(Y, M, tau, bun, leaves, W); });
  }
  for (int W : {32, 64, 128, 256}) {
    const int sm2 = 2 * bun * W * 8, sm8 = 8 * bun * W * 8;
    cudaFuncSetAttribute(tree_store_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    cudaFuncSetAttribute(tree_store_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8);
    run("tree_bulk_ring2", W, [&] { tree_store_bulk<2><<<grid, 128, sm2>>>(Y, M, tau, bun, leaves, W); });
    run("tree_bulk_ring8", W, [&] { tree_store_bulk<8><<<grid, 128, sm8>>>(Y, M, tau, bun, leaves, W); });
  }
  row_store4<<<148 * 8, 256>>>(Y, N, tau);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) row_store4<<<148 * 8, 256>>>(Y, N, tau);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\":\"ystore\",\"pattern\":\"rows_v4\",\"ms\":%.4f,\"gbs\":%.1f}\n", ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) cudaMemsetAsync(Y, 0, (size_t)N * tau * 8);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\":\"ystore\",\"pattern\":\"memset\",\"ms\":%.4f,\"gbs\":%.1f}\n", ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
