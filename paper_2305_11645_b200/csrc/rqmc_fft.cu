// NEXT-4: the per-level [DKLS15] FFT product for UNSHIFTED base-2 lattice levels
// ("reordering ... into a circulant structure" + FFT; used inside each level of
// Alg. 2 by the cost proof P:522-526; valid only when every coordinate of the level has the same map,
// i.e. no per-coordinate shift).
//
// Level w has M = 2^k distinct rows; its points are x_{r,j} = phi((r z'_j mod M) / M) with
// one map phi (identity or Phi^-1 with the zero rule, reading C-5) for all coordinates j of the level.
// Split the rows by 2-adic valuation: r = 2^v u, u odd, K = k - v.  For K >= 3 the odd residues mod 2^K
// form {+-1} x <5> (5 has order L = 2^(K-2)), so u = sigma 5^e and z'_j = sigma_j 5^(e_j) (mod 2^K):
//   P[2^v sigma 5^e, c] = sum_{sigma'} sum_{e'} H_v(sigma sigma', e + e') a_v(sigma', e', c),
//   H_v(tau, e) = phi(2^v (tau 5^e mod 2^K) / M),   a_v(sigma', e', c) = sum_{j: sigma_j = sigma',
//   e_j = e' (mod L)} A[j, c]
// -- a cyclic cross-correlation over Z_L per column c, computed with FFTs of length L:
//   P^+ = H^+ conj(a^+) + H^- conj(a^-),  P^- = H^- conj(a^+) + H^+ conj(a^-)  (per frequency),
// the two real sequences of each pair packed into one complex FFT.  The valuations K <= 2 (rows 0,
// 2^(k-1), 2^(k-2), 3 2^(k-2)) are computed directly by the definition (k_fft_rows).  The level's R
// (R_w[r] = P_w[r] + R_w'[r mod M_w']) is written exactly as the GEMM path writes it.
//
// An FFT of length L = L1 L2 (L1 <= 256) is the four-step decomposition over HBM: pass A = FFTs of
// length L1 across e1 (e = e1 L2 + e2) + twiddles w_L^(e2 f1); pass B = FFTs of length L2 across e2 for
// each f1 (spectrum f = f1 + L1 f2 stored at f1 L2 + f2).  Three kernels per level:
//   k_fft_pass1  gather a_v from A's rows (coordinates sorted by (sigma, bit-reversed e_j)) + pass A;
//                (mode 1: generate H_v instead, one column)
//   k_fft_pass2  pass B on the rows f1 and -f1 together, unpack, multiply by H's spectrum, repack,
//                inverse pass B (mode 1: forward pass B only -> H's spectrum)
//   k_fft_pass3  inverse pass A, 1/L, unpack P^+, P^-, scatter rows r = 2^v (+-5^e mod 2^K) + parent
// Each CTA transforms kFftCT = 16 columns (256-byte row segments in HBM) in shared memory, radix 2.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rqmc_device.cuh"

namespace rqmc {

constexpr int kFftCT = 16;
constexpr int kFftThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // a conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cexpi(int64_t num, int64_t den) {   // exp(-2 pi i num / den)
  double s, c;
  sincospi(-2.0 * (double)num / (double)den, &s, &c);
  return make_double2(c, s);
}
__device__ __forceinline__ int brev(int x, int lg) { return lg == 0 ? 0 : (int)(__brev((unsigned)x) >> (32 - lg)); }
__device__ __forceinline__ uint32_t pow5(int e, int K) {            // 5^e mod 2^K (K <= 32)
  uint64_t r = 1, b = 5;
  for (uint32_t x = (uint32_t)e; x; x >>= 1) {
    if (x & 1u) r = (r * b) & 0xffffffffull;
    b = (b * b) & 0xffffffffull;
  }
  return (uint32_t)(K >= 32 ? r : (r & ((1ull << K) - 1)));
}

// phi(t / 2^k): identity or Phi^-1 with the zero rule (unshifted lattice levels only)
__device__ __forceinline__ double fft_phi(const FftArgs& a, uint64_t t) {
  double u = (double)(uint32_t)t * a.inv_M;
  if (a.map == 1) {
    if (u == 0.0) u = a.zero_u;
    u = normcdfinv(u);
  }
  return u;
}

// twiddles tw[j] = exp(-2 pi i j / n), j < n / 2
__device__ __forceinline__ void fft_twiddles(double2* tw, int n) {
  for (int j = threadIdx.x; j < n / 2; j += blockDim.x) tw[j] = cexpi(j, n);
}

// radix-2 DIT over the rows of buf[row * kFftCT + col], n = 2^lg rows stored in bit-reversed order;
// natural order on return.  inv: conjugate twiddles (unscaled inverse).
__device__ void fft_rows(double2* buf, int lg, bool inv, const double2* tw) {
  const int n = 1 << lg;
  for (int s = 0; s < lg; ++s) {
    const int h = 1 << s, tsh = lg - 1 - s;   // twiddle index i * n / (2h)
    for (int idx = threadIdx.x; idx < (n / 2) * kFftCT; idx += blockDim.x) {
      const int col = idx & (kFftCT - 1), b = idx / kFftCT;
      const int i = b & (h - 1), r0 = ((b >> s) << (s + 1)) + i, r1 = r0 + h;
      double2 w = tw[i << tsh];
      if (inv) w.y = -w.y;
      const double2 x0 = buf[r0 * kFftCT + col];
      const double2 t = cmul(w, buf[r1 * kFftCT + col]);
      buf[r0 * kFftCT + col] = cadd(x0, t);
      buf[r1 * kFftCT + col] = csub(x0, t);
    }
    __syncthreads();
  }
}

// blockIdx.y -> (v, idx) where valuation v owns cnt(v) consecutive indices
template <class F>
__device__ __forceinline__ bool fft_task(const FftArgs& a, int y, F cnt, int* v, int* idx) {
  for (int vv = 0; vv < a.nv; ++vv) {
    const int c = cnt(a.v[vv]);
    if (y < c) { *v = vv; *idx = y; return true; }
    y -= c;
  }
  return false;
}

// lower bound of key >= x in keys[lo, hi)
__device__ __forceinline__ int lbound(const uint32_t* keys, int lo, int hi, uint32_t x) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (keys[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// pass 1: (mode 0) a_v(+-, e) for e = e1 L2 + e2, e1 < L1, packed a^+ + i a^-; (mode 1) H_v(+-, e);
// FFT over e1; times w_L^(e2 f1); stored at row f1 L2 + e2
__global__ void __launch_bounds__(kFftThreads) k_fft_pass1(const FftArgs a, int mode) {
  pdl_enter();
  int vi, e2;
  if (!fft_task(a, blockIdx.y, [](const FftV& V) { return V.L2; }, &vi, &e2)) return;
  const FftV V = a.v[vi];
  const int c0 = blockIdx.x * kFftCT;
  extern __shared__ __align__(16) double2 fbuf[];
  double2* buf = fbuf;                       // L1 x kFftCT
  double2* tw = buf + V.L1 * kFftCT;         // L1 / 2
  int* rng = reinterpret_cast<int*>(tw + V.L1 / 2 + 1);   // 4 L1 bucket bounds
  fft_twiddles(tw, V.L1);
  const int K = a.k - vi;
  if (mode == 0) {
    // bucket of (sigma, e mod L): keys are e_j bit-reversed over k-2 bits, so e_j = e (mod 2^p)
    // <-> key in [rev_p(e) << vi, (rev_p(e) + 1) << vi)
    for (int e1 = threadIdx.x; e1 < V.L1; e1 += blockDim.x) {
      const int e = e1 * V.L2 + e2;
      const uint32_t lo = (uint32_t)brev(e, V.p) << vi, hi = lo + (1u << vi);
      rng[4 * e1 + 0] = lbound(a.key, 0, a.nplus, lo);
      rng[4 * e1 + 1] = lbound(a.key, 0, a.nplus, hi);
      rng[4 * e1 + 2] = lbound(a.key, a.nplus, a.s_w, lo);
      rng[4 * e1 + 3] = lbound(a.key, a.nplus, a.s_w, hi);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < V.L1 * kFftCT; t += blockDim.x) {
      const int e1 = t / kFftCT, col = t & (kFftCT - 1), c = c0 + col;
      double sp = 0.0, sm = 0.0;
      if (c < a.ncol) {
        for (int q = rng[4 * e1]; q < rng[4 * e1 + 1]; ++q) sp += a.A[(int64_t)a.jsort[q] * a.lda + c];
        for (int q = rng[4 * e1 + 2]; q < rng[4 * e1 + 3]; ++q) sm += a.A[(int64_t)a.jsort[q] * a.lda + c];
      }
      buf[brev(e1, V.lgL1) * kFftCT + col] = make_double2(sp, sm);
    }
  } else {
    const uint32_t mK = (K >= 32) ? 0xffffffffu : ((1u << K) - 1);
    for (int t = threadIdx.x; t < V.L1 * kFftCT; t += blockDim.x) {
      const int e1 = t / kFftCT, col = t & (kFftCT - 1);
      double2 h = make_double2(0.0, 0.0);
      if (c0 + col < a.ncol) {
        const uint32_t u = pow5(e1 * V.L2 + e2, K);
        h.x = fft_phi(a, (uint64_t)u << vi);
        h.y = fft_phi(a, (uint64_t)((0u - u) & mK) << vi);
      }
      buf[brev(e1, V.lgL1) * kFftCT + col] = h;
    }
  }
  __syncthreads();
  fft_rows(buf, V.lgL1, false, tw);
  for (int t = threadIdx.x; t < V.L1 * kFftCT; t += blockDim.x) {
    const int f1 = t / kFftCT, col = t & (kFftCT - 1), c = c0 + col;
    if (c < a.ncol) {
      const double2 w = cexpi(((int64_t)e2 * f1) & (V.L - 1), V.L);
      a.Z[V.zoff + (int64_t)(f1 * V.L2 + e2) * a.ldz + c] = cmul(buf[f1 * kFftCT + col], w);
    }
  }
}

// pass 2 on the rows f1 and f1b = -f1 (mod L1): forward FFT over e2 -> f2; (mode 0) unpack a^+-,
// multiply with H's spectrum, repack P^+ + i P^-, inverse FFT over f2, times conj(w_L^(e2 f1));
// (mode 1) store the forward spectrum (H)
__global__ void __launch_bounds__(kFftThreads) k_fft_pass2(const FftArgs a, int mode) {
  pdl_enter();
  int vi, f1;
  if (!fft_task(a, blockIdx.y, [](const FftV& V) { return V.L1 / 2 + 1; }, &vi, &f1)) return;
  const FftV V = a.v[vi];
  const int c0 = blockIdx.x * kFftCT;
  const int f1b = (V.L1 - f1) & (V.L1 - 1);
  const bool two = f1b != f1;
  extern __shared__ __align__(16) double2 fbuf[];
  double2* b0 = fbuf;
  double2* b1 = b0 + V.L2 * kFftCT;
  double2* tw = b1 + V.L2 * kFftCT;
  fft_twiddles(tw, V.L2);
  const double2* z0 = a.Z + V.zoff + (int64_t)f1 * V.L2 * a.ldz;
  const double2* z1 = a.Z + V.zoff + (int64_t)f1b * V.L2 * a.ldz;
  for (int t = threadIdx.x; t < V.L2 * kFftCT; t += blockDim.x) {
    const int e2 = t / kFftCT, col = t & (kFftCT - 1), c = c0 + col;
    const int d = brev(e2, V.lgL2) * kFftCT + col;
    b0[d] = c < a.ncol ? z0[(int64_t)e2 * a.ldz + c] : make_double2(0.0, 0.0);
    if (two) b1[d] = c < a.ncol ? z1[(int64_t)e2 * a.ldz + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_rows(b0, V.lgL2, false, tw);
  if (two) fft_rows(b1, V.lgL2, false, tw);
  if (mode == 1) {
    for (int t = threadIdx.x; t < V.L2 * kFftCT; t += blockDim.x) {
      const int f2 = t / kFftCT, col = t & (kFftCT - 1), c = c0 + col;
      if (c < a.ncol) {
        a.Z[V.zoff + (int64_t)(f1 * V.L2 + f2) * a.ldz + c] = b0[t];
        if (two) a.Z[V.zoff + (int64_t)(f1b * V.L2 + f2) * a.ldz + c] = b1[t];
      }
    }
    return;
  }
  // pairs {f, -f}: f = f1 + L1 f2 in b0[f2]; -f in (two ? b1 : b0)[f2'], f2' = L2-1-f2 (f1 != 0) or
  // (L2 - f2) mod L2 (f1 = 0).  One thread per unordered pair, results written in place.
  const double2* H = a.H + V.hoff;
  for (int t = threadIdx.x; t < V.L2 * kFftCT; t += blockDim.x) {
    const int f2 = t / kFftCT, col = t & (kFftCT - 1);
    const int f2p = f1 != 0 ? V.L2 - 1 - f2 : ((V.L2 - f2) & (V.L2 - 1));
    if (!two && f2p < f2) continue;          // the partner's thread handles this pair
    double2* pa = b0 + f2 * kFftCT + col;
    double2* pb = (two ? b1 : b0) + f2p * kFftCT + col;
    const double2 za = *pa, zb = *pb;         // Z(f), Z(-f)
    const double2 ha = H[f1 * V.L2 + f2], hb = H[f1b * V.L2 + f2p];   // Hc(f), Hc(-f)
    // a^+(f) = (Z(f) + conj Z(-f)) / 2, a^-(f) = (Z(f) - conj Z(-f)) / 2i; likewise H^+-(f) from Hc
    const double2 ap = make_double2(0.5 * (za.x + zb.x), 0.5 * (za.y - zb.y));
    const double2 am = make_double2(0.5 * (za.y + zb.y), -0.5 * (za.x - zb.x));
    const double2 hp = make_double2(0.5 * (ha.x + hb.x), 0.5 * (ha.y - hb.y));
    const double2 hm = make_double2(0.5 * (ha.y + hb.y), -0.5 * (ha.x - hb.x));
    // spectra at -f are the conjugates (real sequences)
    const double2 apb = make_double2(ap.x, -ap.y), amb = make_double2(am.x, -am.y);
    const double2 hpb = make_double2(hp.x, -hp.y), hmb = make_double2(hm.x, -hm.y);
    const double2 Pp = cadd(cmulc(hp, ap), cmulc(hm, am)), Pm = cadd(cmulc(hm, ap), cmulc(hp, am));
    const double2 Ppb = cadd(cmulc(hpb, apb), cmulc(hmb, amb)), Pmb = cadd(cmulc(hmb, apb), cmulc(hpb, amb));
    *pa = make_double2(Pp.x - Pm.y, Pp.y + Pm.x);          // P^+ + i P^- at f
    if (pb != pa) *pb = make_double2(Ppb.x - Pmb.y, Ppb.y + Pmb.x);
  }
  __syncthreads();
  // bit-reverse the rows in place, then the inverse FFT over f2
  for (int t = threadIdx.x; t < V.L2 * kFftCT; t += blockDim.x) {
    const int i = t / kFftCT, col = t & (kFftCT - 1), j = brev(i, V.lgL2);
    if (i < j) {
      double2 x = b0[i * kFftCT + col]; b0[i * kFftCT + col] = b0[j * kFftCT + col]; b0[j * kFftCT + col] = x;
      if (two) { x = b1[i * kFftCT + col]; b1[i * kFftCT + col] = b1[j * kFftCT + col]; b1[j * kFftCT + col] = x; }
    }
  }
  __syncthreads();
  fft_rows(b0, V.lgL2, true, tw);
  if (two) fft_rows(b1, V.lgL2, true, tw);
  for (int t = threadIdx.x; t < V.L2 * kFftCT; t += blockDim.x) {
    const int e2 = t / kFftCT, col = t & (kFftCT - 1), c = c0 + col;
    if (c < a.ncol) {
      double2 w = cexpi(((int64_t)e2 * f1) & (V.L - 1), V.L);
      w.y = -w.y;
      a.Z[V.zoff + (int64_t)(f1 * V.L2 + e2) * a.ldz + c] = cmul(b0[t], w);
      if (two) {
        double2 wb = cexpi(((int64_t)e2 * f1b) & (V.L - 1), V.L);
        wb.y = -wb.y;
        a.Z[V.zoff + (int64_t)(f1b * V.L2 + e2) * a.ldz + c] = cmul(b1[t], wb);
      }
    }
  }
}

// pass 3: inverse FFT over f1 -> e1, 1/L, P^+ = Re, P^- = Im at e = e1 L2 + e2, rows
// r = 2^v (+-5^e mod 2^K): R[r, c] = P + R_parent[r mod M_parent, c]
__global__ void __launch_bounds__(kFftThreads) k_fft_pass3(const FftArgs a) {
  pdl_enter();
  int vi, e2;
  if (!fft_task(a, blockIdx.y, [](const FftV& V) { return V.L2; }, &vi, &e2)) return;
  const FftV V = a.v[vi];
  const int c0 = blockIdx.x * kFftCT;
  extern __shared__ __align__(16) double2 fbuf[];
  double2* buf = fbuf;
  double2* tw = buf + V.L1 * kFftCT;
  int64_t* rows = reinterpret_cast<int64_t*>(tw + V.L1 / 2 + 1);   // 2 L1
  fft_twiddles(tw, V.L1);
  const int K = a.k - vi;
  const uint32_t mK = (K >= 32) ? 0xffffffffu : ((1u << K) - 1);
  for (int e1 = threadIdx.x; e1 < V.L1; e1 += blockDim.x) {
    const uint32_t u = pow5(e1 * V.L2 + e2, K);
    rows[2 * e1] = (int64_t)u << vi;
    rows[2 * e1 + 1] = (int64_t)((0u - u) & mK) << vi;
  }
  for (int t = threadIdx.x; t < V.L1 * kFftCT; t += blockDim.x) {
    const int f1 = t / kFftCT, col = t & (kFftCT - 1), c = c0 + col;
    buf[brev(f1, V.lgL1) * kFftCT + col] =
        c < a.ncol ? a.Z[V.zoff + (int64_t)(f1 * V.L2 + e2) * a.ldz + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_rows(buf, V.lgL1, true, tw);
  const double sc = 1.0 / (double)V.L;
  for (int t = threadIdx.x; t < 2 * V.L1 * kFftCT; t += blockDim.x) {
    const int col = t & (kFftCT - 1), q = t / kFftCT, e1 = q >> 1, sg = q & 1, c = c0 + col;
    if (c >= a.ncol) continue;
    const double2 x = buf[e1 * kFftCT + col];
    const int64_t r = rows[2 * e1 + sg];
    double v = (sg ? x.y : x.x) * sc;
    if (a.Rp) v += a.Rp[(r % a.Mp) * a.ldp + c];
    a.R[r * a.ldr + c] = v;
  }
}

// rows with valuation >= k-2 (0, 2^(k-1), 2^(k-2), 3 2^(k-2)) by the definition: P[r, c] =
// sum_j phi((r z'_j mod M) / M) A[j, c] in increasing j, plus the parent row
__global__ void __launch_bounds__(256) k_fft_rows(const FftArgs a) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ double xs[4][256];
  const uint64_t M = 1ull << a.k;
  const uint64_t rr[4] = {0, M >> 1, M >> 2, 3 * (M >> 2)};
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j0 = 0; j0 < a.s_w; j0 += 256) {
    __syncthreads();
    for (int t = threadIdx.x; t < 4 * 256; t += blockDim.x) {
      const int q = t >> 8, j = j0 + (t & 255);
      if (j < a.s_w) xs[q][t & 255] = fft_phi(a, (rr[q] * a.z[j]) & (M - 1));
    }
    __syncthreads();
    if (c < a.ncol) {
      const int n = min(256, a.s_w - j0);
      for (int jj = 0; jj < n; ++jj) {
        const double av = a.A[(int64_t)(j0 + jj) * a.lda + c];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(xs[q][jj], av, acc[q]);
      }
    }
  }
  if (c < a.ncol) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double v = acc[q];
      if (a.Rp) v += a.Rp[(int64_t)(rr[q] % (uint64_t)a.Mp) * a.ldp + c];
      a.R[(int64_t)rr[q] * a.ldr + c] = v;
    }
  }
}

static int fft_smem_bytes(const FftArgs& a, int pass) {
  int L1 = 1, L2 = 1;
  for (int i = 0; i < a.nv; ++i) { L1 = max(L1, a.v[i].L1); L2 = max(L2, a.v[i].L2); }
  if (pass == 2) return (int)sizeof(double2) * (2 * L2 * kFftCT + L2 / 2 + 1);
  return (int)sizeof(double2) * (L1 * kFftCT + L1 / 2 + 1) + 4 * L1 * (int)sizeof(int64_t);
}

cudaError_t launch_fft_level(const FftArgs& a0, cudaStream_t st) {
  int n1 = 0, n2 = 0;
  for (int i = 0; i < a0.nv; ++i) {
    n1 += a0.v[i].L2;
    n2 += a0.v[i].L1 / 2 + 1;
  }
  const int s1 = fft_smem_bytes(a0, 1), s2 = fft_smem_bytes(a0, 2);
  cudaError_t e;
  if ((e = set_smem_once(k_fft_pass1, s1)) != cudaSuccess) return e;
  if ((e = set_smem_once(k_fft_pass2, s2)) != cudaSuccess) return e;
  if ((e = set_smem_once(k_fft_pass3, s1)) != cudaSuccess) return e;
  // H_v and its spectrum (one column), then the data
  FftArgs h = a0;
  h.Z = a0.H; h.ldz = 1; h.ncol = 1;
  for (int i = 0; i < h.nv; ++i) h.v[i].zoff = h.v[i].hoff;
  if ((e = launch_k(k_fft_pass1, dim3(1, n1), dim3(kFftThreads), s1, st, true, h, 1)) != cudaSuccess) return e;
  if ((e = launch_k(k_fft_pass2, dim3(1, n2), dim3(kFftThreads), s2, st, true, h, 1)) != cudaSuccess) return e;
  const unsigned gx = (unsigned)((a0.ncol + kFftCT - 1) / kFftCT);
  if ((e = launch_k(k_fft_pass1, dim3(gx, n1), dim3(kFftThreads), s1, st, true, a0, 0)) != cudaSuccess) return e;
  if ((e = launch_k(k_fft_pass2, dim3(gx, n2), dim3(kFftThreads), s2, st, true, a0, 0)) != cudaSuccess) return e;
  if ((e = launch_k(k_fft_pass3, dim3(gx, n1), dim3(kFftThreads), s1, st, true, a0)) != cudaSuccess) return e;
  return launch_k(k_fft_rows, dim3((unsigned)((a0.ncol + 255) / 256)), dim3(256), 0, st, true, a0);
}

}  // namespace rqmc
