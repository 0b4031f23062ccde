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
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
