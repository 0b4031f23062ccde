// Device helpers shared by the sm_100a kernel translation units (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>
#include <utility>
#include <vector>

#include "rqmc_internal.h"

#ifndef RQMC_PDL
#define RQMC_PDL 1
#endif

namespace rqmc {

// Programmatic dependent launch: every kernel of the path is launched with programmatic stream
// serialisation, so its launch processing and CTA rasterisation overlap the tail of the kernel before
// it.  Each kernel first waits for its predecessor grid to complete and flush (griddepcontrol.wait:
// nothing is read or written before), then allows its own successor to launch (its CTAs park at their
// own wait on slots this grid no longer needs -- all of this grid's CTAs have started by then).
__device__ __forceinline__ void pdl_enter() {
#if RQMC_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if RQMC_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// pdl = false: plain stream order (the fused fine-tree kernel: with programmatic launch its CTAs
// park on the SMs during the checkpoint GEMM's last wave, which measured 0.26 ms slower on C4 with
// 8-warp CTAs and neutral otherwise)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                            Args&&... args) {
#if RQMC_PDL
  if (!pdl) {
    k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
#else
  (void)pdl;
  k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
  return cudaGetLastError();
#endif
}

// cudaFuncSetAttribute(max dynamic smem) once per kernel, device and size (a driver call per launch
// costs microseconds: visible on the small configs C1/C2)
struct SmemAttr { const void* fn; int dev; int bytes; };
inline cudaError_t set_smem_once_raw(const void* fn, int bytes) {
  static std::mutex mu;
  static std::vector<SmemAttr> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (const SmemAttr& d : done)
    if (d.fn == fn && d.dev == dev && d.bytes >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back({fn, dev, bytes});
  return e;
}
template <class F>
inline cudaError_t set_smem_once(F* kern, int bytes) {
  return set_smem_once_raw(reinterpret_cast<const void*>(kern), bytes);
}

// ------------------------------------------------------------------------------------------
// Debug build (-DRQMC_DEBUG=1, `_build.py --variant debug`): every cp.async source and every global
// store of the path is checked against the buffers of the current run (workspace, A, Y, f-sums, plan
// tables), set per launch sequence by debug_set_ranges(); a violation prints the site and traps.
// (A bounds-checked stand-in for compute-sanitizer, which is closed on this pool.)
// ------------------------------------------------------------------------------------------
#ifndef RQMC_DEBUG
#define RQMC_DEBUG 0
#endif
#if RQMC_DEBUG
static __constant__ DbgRanges c_dbg;     // one copy per translation unit
__device__ __forceinline__ bool dbg_ok(const void* p, size_t n) {
  const char* q = static_cast<const char*>(p);
#pragma unroll
  for (int i = 0; i < 6; ++i)
    if (q >= c_dbg.lo[i] && q + n <= c_dbg.hi[i]) return true;
  return false;
}
#define RQMC_DCHECK(p, n)                                                                        \
  do {                                                                                           \
    if (!dbg_ok((p), (n))) {                                                                     \
      printf("RQMC_DEBUG out-of-bounds %s:%d block (%d,%d,%d) thread %d addr %p\n", __FILE__,      \
             __LINE__, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, (const void*)(p));          \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
static inline cudaError_t dbg_set_tu(const DbgRanges& r, cudaStream_t st) {
  return cudaMemcpyToSymbolAsync(c_dbg, &r, sizeof(r), 0, cudaMemcpyHostToDevice, st);
}
#else
#define RQMC_DCHECK(p, n) do { } while (0)
#endif

// ------------------------------------------------------------------------------------------
// async copy helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  if (valid) RQMC_DCHECK(src, 16);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  if (valid) RQMC_DCHECK(src, 8);
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
  int64_t ybase, ystride;  // Y row of this lane's residue (leaf run 0) and the step per leaf run
  const double* as;      // A slab of the current column tile
};

// D = A B + C with C and D in distinct registers (DMMA.8x8x4)
__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

extern __shared__ __align__(16) double fsm[];  // dynamic smem of the fine kernels

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

// F(mean) of f(y) = F(tau^-1 sum_c g(y_c)) (reading C-17): fk 0 exp, 1 max(. - p1, 0), else identity
__device__ __forceinline__ double f_of_mean(const FineArgs& a, double mean) {
  switch (a.fk) {
    case 0: return exp(mean);
    case 1: { const double v = mean - a.fp1; return v > 0.0 ? v : 0.0; }
    default: return mean;
  }
}

// The tent transformation phi(u) = 1 - |1 - 2u|, evaluated as written with
// round-to-nearest adds (2u exact): the oracle's orc_tent bit for bit.
__device__ __forceinline__ double tent_map(double u) {
  return __dadd_rn(1.0, -fabs(__dadd_rn(1.0, __dmul_rn(-2.0, u))));
}

// a5: fixed-order final reduction fused into the fine kernels (FineArgs::fsum).  Called by every
// thread of a CTA that has just written its partial (thread 0 wrote it); the last CTA of the replica to
// arrive sums the replica's nparts partials -- thread t adds partials t, t + NT, ... in order, warps
// reduce by xor shuffles, thread 0 adds the warp sums in warp order -- so the result does not depend on
// which CTA arrives last.  Replaces the k_reduce launch (one launch latency on the small configs).
template <int NT>
__device__ __forceinline__ void finish_fsum(const FineArgs& a, int64_t rep, int64_t nparts) {
  if (a.fsum == nullptr) return;
  __shared__ int s_last;
  __shared__ double s_red[NT / 32];
  unsigned int* cnt = a.rcnt + kSplitSlots + rep * 2 * a.partrep;
  __threadfence();   // the partial is visible device-wide before its arrival is counted
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1u) == (unsigned int)(nparts - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double* p = a.partial + rep * a.partrep;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < nparts; i += NT) s += __ldcg(p + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += s_red[w];
    RQMC_DCHECK(a.fsum + rep, 8);
    a.fsum[rep] = t;
    *cnt = 0u;   // ready for the next call (k_gen zeroes it as well)
  }
}

// Y row of local row l (identity, or the residue chunk's row map, FineArgs::ym_nc) and the Y row step
// per leaf run (see FineArgs::ym_nc): evaluated once per thread
__device__ __forceinline__ int64_t y_row(const FineArgs& a, int64_t l) {
  if (a.ym_nc == 0) return l;
  const int64_t q = l / a.ym_nc;
  return a.ym_c0 + (l - q * a.ym_nc) + a.ym_ncls * q;
}
__device__ __forceinline__ int64_t y_stride(const FineArgs& a) {
  return a.ym_nc == 0 ? a.Mroot : a.ym_ncls * (a.Mroot / a.ym_nc);
}

template <bool STY>
__device__ __forceinline__ void store_leaf(const FineArgs& a, const double (&S)[8], int j, const FineCtx& c) {
  if constexpr (STY) {
    if (c.t < c.beff) {
      double* yr = a.Y + (c.ybase + (int64_t)j * c.ystride) * a.ldy;
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) {
        const int col = c.c0 + cf * 8 + 2 * c.tg;
        if (col < a.tau) RQMC_DCHECK(yr + col, col + 1 < a.tau ? 16 : 8);
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


}  // namespace rqmc
