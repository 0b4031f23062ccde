// NEXT-4: the per-level [DKLS15] FFT product for UNSHIFTED base-2 lattice levels
// ("reordering ... into a circulant structure" + FFT; used inside each level of
// Alg. 2 by the cost proof P:522-526; valid only when every coordinate of the level has the same map,
// i.e. no per-coordinate shift).
//
// Level w has M = 2^k distinct rows; its points are x_{r,j} = phi((r z'_j mod M) / M) with
// one map phi (identity, Phi^-1 with the zero rule, reading C-5, or the tent map) for all
// coordinates j of the level.
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
// Valuations with L <= 256 run whole in one CTA per column tile (k_fft_small: gather a_v, FFT, multiply
// by H's spectrum, inverse FFT, scatter).  Longer ones (L = L1 L2, L1, L2 <= 256) use the four-step
// decomposition over HBM: pass A = FFTs of length L1 across e1 (e = e1 L2 + e2) + twiddles
// w_L^(e2 f1); pass B = FFTs of length L2 across e2 for each f1 (spectrum f = f1 + L1 f2 stored at
// f1 L2 + f2):
//   k_fft_pass1  gather a_v from A's rows (coordinates sorted by (sigma, bit-reversed e_j)) + pass A;
//                (mode 1: generate H_v instead, one column -- for every valuation)
//   k_fft_pass2  pass B on the rows f1 and -f1 together, unpack, multiply by H's spectrum, repack,
//                inverse pass B (mode 1: forward pass B only -> H's spectrum)
//   k_fft_pass3  inverse pass A, 1/L, unpack P^+, P^-, scatter rows r = 2^v (+-5^e mod 2^K) + parent
// In shared memory an FFT of length n <= 256 is itself split n = n1 n2 (n1, n2 <= 16): each thread
// does a length-n1 then a length-n2 DFT in registers (radix 2, unrolled), one exchange in between.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rqmc_device.cuh"

namespace rqmc {

#ifndef RQMC_FFT_CT          // columns per CTA of the pass-1/3 and short-valuation kernels (pass 2: half,
#define RQMC_FFT_CT 16       // two sequences); 16 workers per column and sequence (8 measured 2 % slower)
#endif
constexpr int kFftCT = RQMC_FFT_CT;
constexpr int kFftThreads = 16 * kFftCT;
constexpr int kFftSmallLg = 8;     // valuations with L <= 2^8 run in k_fft_small

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // a conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
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

// phi(t / 2^k): identity, Phi^-1 with the zero rule, or the tent map (unshifted lattice levels only;
// one map for every coordinate of the level)
__device__ __forceinline__ double fft_phi(const FftArgs& a, uint64_t t) {
  double u = (double)(uint32_t)t * a.inv_M;
  if (a.map == 1) {
    if (u == 0.0) u = a.zero_u;
    u = normcdfinv(u);
  } else if (a.map == 2) {
    u = tent_map(u);
  }
  return u;
}

// tw[j] = exp(-2 pi i j / n), j < n
__device__ __forceinline__ void fft_twiddles(double2* tw, int n) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) tw[j] = cexpi(j, n);
}

// in-register DFT of length N (radix-2 DIT, compile-time indices); twiddle w_N^j = tw[j * ts]
template <int N, bool INV>
__device__ __forceinline__ void dft_reg(double2 (&r)[16], const double2* tw, int ts) {
  constexpr int LG = N <= 1 ? 0 : (N == 2 ? 1 : (N == 4 ? 2 : (N == 8 ? 3 : 4)));
#pragma unroll
  for (int i = 0; i < N; ++i) {
    int j = 0;
#pragma unroll
    for (int b = 0; b < LG; ++b) j |= ((i >> b) & 1) << (LG - 1 - b);
    if (i < j) { const double2 t = r[i]; r[i] = r[j]; r[j] = t; }
  }
#pragma unroll
  for (int h = 1; h < N; h <<= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i & h) continue;
      const int jj = i & (h - 1);
      double2 w = tw[jj * (N / (2 * h)) * ts];
      if (INV) w.y = -w.y;
      const double2 t = cmul(w, r[i + h]);
      r[i + h] = csub(r[i], t);
      r[i] = cadd(r[i], t);
    }
  }
}

template <int CT, int S, bool INV, int LG>
__device__ __forceinline__ void fft_smem_t(double2* buf, const double2* tw) {
  constexpr int QW = kFftThreads / (S * CT);
  constexpr int n = 1 << LG, L1 = (LG + 1) >> 1, L2 = LG >> 1, n1 = 1 << L1, n2 = 1 << L2;
  static_assert(n1 <= QW && n2 <= QW, "one sequence position per worker");
  const int col = threadIdx.x % CT, s = (threadIdx.x / CT) % S, q = threadIdx.x / (CT * S);
  double2* b = buf + (size_t)s * n * CT + col;
  if (q < n2) {
    double2 r[16];
#pragma unroll
    for (int i = 0; i < n1; ++i) r[i] = b[(i * n2 + q) * CT];
    dft_reg<n1, INV>(r, tw, n / n1);
#pragma unroll
    for (int i = 0; i < n1; ++i) {
      double2 w = tw[(q * i) & (n - 1)];
      if (INV) w.y = -w.y;
      b[(i * n2 + q) * CT] = cmul(r[i], w);
    }
  }
  __syncthreads();
  if constexpr (L2 > 0) {
    double2 r2[16];
    if (q < n1) {
#pragma unroll
      for (int i = 0; i < n2; ++i) r2[i] = b[(q * n2 + i) * CT];
      dft_reg<n2, INV>(r2, tw, n / n2);
    }
    __syncthreads();
    if (q < n1) {
#pragma unroll
      for (int i = 0; i < n2; ++i) b[(q + n1 * i) * CT] = r2[i];
    }
    __syncthreads();
  }
}

// FFT of length n = 2^lg (lg <= 8) along the rows of S sequences x CT columns in shared memory,
// buf[(s n + row) CT + col], natural order in and out; kFftThreads = S x CT x 16 workers.
// n = n1 n2 (n1 = 2^ceil(lg/2), n2 = 2^floor(lg/2)): worker q < n2 transforms x[i1 n2 + q] over i1 and
// applies w_n^(q k1); worker q < n1 then transforms over the n2 rows q n2 + i2 into X[q + n1 k2].
// tw: w_n^j, j < n.  INV: conjugate twiddles (unscaled).  Compile-time sizes per lg.  Ends with a barrier.
template <int CT, int S, bool INV>
__device__ __forceinline__ void fft_smem(double2* buf, int lg, const double2* tw) {
  switch (lg) {
    case 1: fft_smem_t<CT, S, INV, 1>(buf, tw); break;
    case 2: fft_smem_t<CT, S, INV, 2>(buf, tw); break;
    case 3: fft_smem_t<CT, S, INV, 3>(buf, tw); break;
    case 4: fft_smem_t<CT, S, INV, 4>(buf, tw); break;
    case 5: fft_smem_t<CT, S, INV, 5>(buf, tw); break;
    case 6: fft_smem_t<CT, S, INV, 6>(buf, tw); break;
    case 7: fft_smem_t<CT, S, INV, 7>(buf, tw); break;
    default: fft_smem_t<CT, S, INV, 8>(buf, tw); break;
  }
}

// blockIdx.y -> (v, idx) for v in [vlo, vhi) where valuation v owns cnt(v) consecutive indices
template <class F>
__device__ __forceinline__ bool fft_task(const FftArgs& a, int vlo, int vhi, int y, F cnt, int* v, int* idx) {
  for (int vv = vlo; vv < vhi; ++vv) {
    const int c = cnt(a.v[vv]);
    if (y < c) { *v = vv; *idx = y; return true; }
    y -= c;
  }
  return false;
}

// a_v(+, e) + i a_v(-, e) for column c (bucket bounds rg[0..3] of (sigma, e mod L), see k_fft_pass1)
__device__ __forceinline__ double2 fft_gather(const FftArgs& a, const int* rg, int c) {
  double sp = 0.0, sm = 0.0;
  for (int q = rg[0]; q < rg[1]; ++q) sp += a.A[(int64_t)a.jsort[q] * a.lda + c];
  for (int q = rg[2]; q < rg[3]; ++q) sm += a.A[(int64_t)a.jsort[q] * a.lda + c];
  return make_double2(sp, sm);
}
// bucket bounds of e at valuation v: the coordinates are sorted by (sigma, bitrev_{k-2}(e_j)), so the
// bucket e_j = e (mod 2^p) is the contiguous range of key rev_p(e) (host table FftV::boff: for
// sigma = +, -, L + 1 range starts in key order)
__device__ __forceinline__ void fft_bounds(const FftArgs& a, const FftV& V, int e, int* rg) {
  const int* b = a.boff + V.boff;
  const int r = brev(e, V.p);
  rg[0] = b[r]; rg[1] = b[r + 1];
  rg[2] = b[V.L + 1 + r]; rg[3] = b[V.L + 2 + r];
}
// H_v(+, e) + i H_v(-, e)
__device__ __forceinline__ double2 fft_hval(const FftArgs& a, int vi, int e) {
  const int K = a.k - vi;
  const uint32_t mK = (K >= 32) ? 0xffffffffu : ((1u << K) - 1);
  const uint32_t u = pow5(e, K);
  return make_double2(fft_phi(a, (uint64_t)u << vi), fft_phi(a, (uint64_t)((0u - u) & mK) << vi));
}
// P^+ + i P^- at f and at -f from the packed spectra Z(f), Z(-f) of a^+- and Hc(f), Hc(-f) of H^+-:
// a^+(f) = (Z(f) + conj Z(-f)) / 2, a^-(f) = (Z(f) - conj Z(-f)) / 2i (likewise H), spectra at -f
// are the conjugates (real sequences); P^+ = H^+ conj(a^+) + H^- conj(a^-), P^- = H^- conj(a^+) +
// H^+ conj(a^-)
__device__ __forceinline__ void fft_mult(double2 za, double2 zb, double2 ha, double2 hb, double2* wa, double2* wb) {
  const double2 ap = make_double2(0.5 * (za.x + zb.x), 0.5 * (za.y - zb.y));
  const double2 am = make_double2(0.5 * (za.y + zb.y), -0.5 * (za.x - zb.x));
  const double2 hp = make_double2(0.5 * (ha.x + hb.x), 0.5 * (ha.y - hb.y));
  const double2 hm = make_double2(0.5 * (ha.y + hb.y), -0.5 * (ha.x - hb.x));
  const double2 Pp = cadd(cmulc(hp, ap), cmulc(hm, am)), Pm = cadd(cmulc(hm, ap), cmulc(hp, am));
  *wa = make_double2(Pp.x - Pm.y, Pp.y + Pm.x);   // P^+(f) + i P^-(f)
  *wb = make_double2(Pp.x + Pm.y, Pm.x - Pp.y);   // conj(P^+(f)) + i conj(P^-(f)) = value at -f
}
// rows[2 i], rows[2 i + 1] = 2^v (5^e mod 2^K), 2^v (-5^e mod 2^K) for e = i es + e0, i < nr (once per
// CTA and row: the CT columns of a row share them)
__device__ __forceinline__ void fft_rows_of(const FftArgs& a, int vi, int e0, int es, int nr, int64_t* rows) {
  const int K = a.k - vi;
  const uint32_t mK = (K >= 32) ? 0xffffffffu : ((1u << K) - 1);
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    const uint32_t w5 = pow5(i * es + e0, K);
    rows[2 * i] = (int64_t)w5 << vi;
    rows[2 * i + 1] = (int64_t)((0u - w5) & mK) << vi;
  }
}

// R[r, c] = P / L + R_parent[r mod M_parent, c] for the rows r = rows[2 (t / CT)] (P^+) and
// rows[2 (t / CT) + 1] (P^-) of the n entries buf[t] (column c0 + t % CT); 4 entries per thread in
// flight (parent loads)
template <int CT>
__device__ __forceinline__ void fft_scatter(const FftArgs& a, const FftV& V, const double2* buf, const int64_t* rows,
                                            int n, int c0) {
  const double sc = 1.0 / (double)V.L;
  for (int t0 = threadIdx.x; t0 < n; t0 += 4 * blockDim.x) {
    int64_t rp[4], rm[4];
    double pp[4], pm[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * blockDim.x, c = c0 + (t % CT);
      rp[u] = -1;
      if (t < n && c < a.ncol) {
        rp[u] = rows[2 * (t / CT)];
        rm[u] = rows[2 * (t / CT) + 1];
        pp[u] = a.Rp ? a.Rp[(rp[u] % a.Mp) * a.ldp + c] : 0.0;
        pm[u] = a.Rp ? a.Rp[(rm[u] % a.Mp) * a.ldp + c] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * blockDim.x, c = c0 + (t % CT);
      if (rp[u] >= 0) {
        const double2 x = buf[t];
        RQMC_DCHECK(a.R + rp[u] * a.ldr + c, 8);
        RQMC_DCHECK(a.R + rm[u] * a.ldr + c, 8);
        a.R[rp[u] * a.ldr + c] = x.x * sc + pp[u];
        a.R[rm[u] * a.ldr + c] = x.y * sc + pm[u];
      }
    }
  }
}

// pass 1 (valuations [vlo, vhi)): (mode 0) a_v for e = e1 L2 + e2, e1 < L1; (mode 1) H_v; FFT over e1;
// times w_L^(e2 f1); stored at row f1 L2 + e2
__global__ void __launch_bounds__(kFftThreads, 512 / kFftThreads) k_fft_pass1(const FftArgs a, int mode, int vlo, int vhi) {
  pdl_enter();
  constexpr int CT = kFftCT;
  int vi, e2;
  if (!fft_task(a, vlo, vhi, blockIdx.y, [](const FftV& V) { return V.L2; }, &vi, &e2)) return;
  const FftV V = a.v[vi];
  const int c0 = blockIdx.x * CT;
  extern __shared__ __align__(16) double2 fbuf[];
  double2* buf = fbuf;                       // L1 x CT
  double2* tw = buf + V.L1 * CT;             // L1
  double2* tr = tw + V.L1;                   // row twiddles w_L^(e2 f1), L1
  int* rng = reinterpret_cast<int*>(tr + V.L1);   // 4 L1 bucket bounds
  fft_twiddles(tw, V.L1);
  for (int f1 = threadIdx.x; f1 < V.L1; f1 += blockDim.x) tr[f1] = cexpi(((int64_t)e2 * f1) & (V.L - 1), V.L);
  if (mode == 0) {
    for (int e1 = threadIdx.x; e1 < V.L1; e1 += blockDim.x) fft_bounds(a, V, e1 * V.L2 + e2, rng + 4 * e1);
    __syncthreads();
#pragma unroll 4
    for (int t = threadIdx.x; t < V.L1 * CT; t += blockDim.x) {
      const int e1 = t / CT, c = c0 + (t % CT);
      buf[t] = c < a.ncol ? fft_gather(a, rng + 4 * e1, c) : make_double2(0.0, 0.0);
    }
  } else {
    for (int t = threadIdx.x; t < V.L1 * CT; t += blockDim.x) {
      const int e1 = t / CT;
      buf[t] = c0 + (t % CT) < a.ncol ? fft_hval(a, vi, e1 * V.L2 + e2) : make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
  fft_smem<CT, 1, false>(buf, V.lgL1, tw);
  for (int t = threadIdx.x; t < V.L1 * CT; t += blockDim.x) {
    const int f1 = t / CT, c = c0 + (t % CT);
    if (c < a.ncol) a.Z[V.zoff + (int64_t)(f1 * V.L2 + e2) * a.ldz + c] = cmul(buf[t], tr[f1]);
  }
}

// pass 2 (valuations [vlo, vhi), L2 >= 2) on the rows f1 and f1b = -f1 (mod L1): forward FFT over e2;
// (mode 0) unpack, multiply with H's spectrum, repack, inverse FFT, times conj(w_L^(e2 f1));
// (mode 1) store the forward spectrum (H)
__global__ void __launch_bounds__(kFftThreads, 512 / kFftThreads) k_fft_pass2(const FftArgs a, int mode, int vlo, int vhi) {
  pdl_enter();
  constexpr int CT = kFftCT / 2;
  int vi, f1;
  if (!fft_task(a, vlo, vhi, blockIdx.y, [](const FftV& V) { return V.L1 / 2 + 1; }, &vi, &f1)) return;
  const FftV V = a.v[vi];
  const int c0 = blockIdx.x * CT;
  const int f1b = (V.L1 - f1) & (V.L1 - 1);
  const bool two = f1b != f1;
  extern __shared__ __align__(16) double2 fbuf[];
  double2* b0 = fbuf;                        // sequence 0 (row f1), then sequence 1 (row f1b)
  double2* b1 = b0 + V.L2 * CT;
  double2* tw = b1 + V.L2 * CT;              // L2
  double2* tr = tw + V.L2;                   // 2 L2 row twiddles
  double2* hs = tr + 2 * V.L2;               // H's spectrum on the rows f1, f1b (2 L2; mode 0)
  fft_twiddles(tw, V.L2);
  for (int e2 = threadIdx.x; e2 < V.L2; e2 += blockDim.x) {
    tr[e2] = cexpi(((int64_t)e2 * f1) & (V.L - 1), V.L);
    tr[V.L2 + e2] = cexpi(((int64_t)e2 * f1b) & (V.L - 1), V.L);
  }
  const double2* z0 = a.Z + V.zoff + (int64_t)f1 * V.L2 * a.ldz;
  const double2* z1 = a.Z + V.zoff + (int64_t)f1b * V.L2 * a.ldz;
  for (int t = threadIdx.x; t < 2 * V.L2 * CT; t += blockDim.x) {   // all loads in flight (cp.async)
    const int sq = t / (V.L2 * CT), tt = t - sq * V.L2 * CT, e2 = tt / CT, c = c0 + (tt % CT);
    const bool ok = c < a.ncol && (sq == 0 || two);
    cp_async16(b0 + t, ok ? (sq ? z1 : z0) + (int64_t)e2 * a.ldz + c : a.Z, ok);
  }
  if (mode == 0)   // H's rows f1 and f1b (contiguous in its block) come in with the data
    for (int t = threadIdx.x; t < 2 * V.L2; t += blockDim.x)
      cp_async16(hs + t, a.H + V.hoff + (int64_t)((t < V.L2 ? f1 : f1b) * V.L2 + (t % V.L2)), true);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  fft_smem<CT, 2, false>(b0, V.lgL2, tw);
  if (mode == 1) {
    for (int t = threadIdx.x; t < 2 * V.L2 * CT; t += blockDim.x) {
      const int sq = t / (V.L2 * CT), tt = t - sq * V.L2 * CT, f2 = tt / CT, c = c0 + (tt % CT);
      if (c < a.ncol && (sq == 0 || two)) a.Z[V.zoff + (int64_t)((sq ? f1b : f1) * V.L2 + f2) * a.ldz + c] = b0[t];
    }
    return;
  }
  // pairs {f, -f}: f = f1 + L1 f2 in b0[f2]; -f in (two ? b1 : b0)[f2'], f2' = L2-1-f2 (f1 != 0) or
  // (L2 - f2) mod L2 (f1 = 0).  One thread per unordered pair, results written in place.
  for (int t = threadIdx.x; t < V.L2 * CT; t += blockDim.x) {
    const int f2 = t / CT, col = t % CT;
    const int f2p = f1 != 0 ? V.L2 - 1 - f2 : ((V.L2 - f2) & (V.L2 - 1));
    if (!two && f2p < f2) continue;
    double2* pa = b0 + f2 * CT + col;
    double2* pb = (two ? b1 : b0) + f2p * CT + col;
    double2 wa, wb;
    fft_mult(*pa, *pb, hs[f2], hs[V.L2 + f2p], &wa, &wb);
    *pa = wa;
    if (pb != pa) *pb = wb;
  }
  __syncthreads();
  fft_smem<CT, 2, true>(b0, V.lgL2, tw);
  for (int t = threadIdx.x; t < 2 * V.L2 * CT; t += blockDim.x) {
    const int sq = t / (V.L2 * CT), tt = t - sq * V.L2 * CT, e2 = tt / CT, c = c0 + (tt % CT);
    if (c < a.ncol && (sq == 0 || two))
      a.Z[V.zoff + (int64_t)((sq ? f1b : f1) * V.L2 + e2) * a.ldz + c] = cmul(b0[t], cconj(tr[sq * V.L2 + e2]));
  }
}

// pass 3 (valuations [vlo, vhi)): inverse FFT over f1 -> e1, 1/L, scatter of P^+ (Re) and P^- (Im)
// at e = e1 L2 + e2
__global__ void __launch_bounds__(kFftThreads, 512 / kFftThreads) k_fft_pass3(const FftArgs a, int vlo, int vhi) {
  pdl_enter();
  constexpr int CT = kFftCT;
  int vi, e2;
  if (!fft_task(a, vlo, vhi, blockIdx.y, [](const FftV& V) { return V.L2; }, &vi, &e2)) return;
  const FftV V = a.v[vi];
  const int c0 = blockIdx.x * CT;
  extern __shared__ __align__(16) double2 fbuf[];
  double2* buf = fbuf;
  double2* tw = buf + V.L1 * CT;
  int64_t* rows = reinterpret_cast<int64_t*>(tw + V.L1);   // 2 L1 (the pass-1 layout's tr / rng space)
  fft_twiddles(tw, V.L1);
  fft_rows_of(a, vi, e2, V.L2, V.L1, rows);
  for (int t = threadIdx.x; t < V.L1 * CT; t += blockDim.x) {
    const int f1 = t / CT, c = c0 + (t % CT);
    cp_async16(buf + t, c < a.ncol ? a.Z + V.zoff + (int64_t)(f1 * V.L2 + e2) * a.ldz + c : a.Z, c < a.ncol);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  fft_smem<CT, 1, true>(buf, V.lgL1, tw);
  fft_scatter<CT>(a, V, buf, rows, V.L1 * CT, c0);
}

// valuations [vlo, nv) with L <= 256 (L2 = 1), all in one CTA per column tile: gather a_vlo, then per
// valuation FFT, multiply by H's spectrum (natural order: from k_fft_pass1 mode 1), inverse FFT,
// scatter, and fold a_(v+1)(e) = a_v(e) + a_v(e + L/2) for the next (coarser) valuation
__global__ void __launch_bounds__(kFftThreads, 1) k_fft_small(const FftArgs a, int vlo) {
  pdl_enter();
  constexpr int CT = kFftCT;
  const FftV V0 = a.v[vlo];
  const int Ls = V0.L, c0 = blockIdx.x * CT;
  extern __shared__ __align__(16) double2 fbuf[];
  double2* acc = fbuf;                       // a_v, Ls x CT
  double2* buf = acc + Ls * CT;              // work, Ls x CT
  double2* twL = buf + Ls * CT;              // w_Ls^j, j < Ls
  double2* tw = twL + Ls;                    // w_L^j of the current valuation (unit stride: constant
                                             // twiddle offsets in the unrolled sub-DFTs)
  int* rng = reinterpret_cast<int*>(tw + Ls);
  fft_twiddles(twL, Ls);
  for (int e = threadIdx.x; e < Ls; e += blockDim.x) fft_bounds(a, V0, e, rng + 4 * e);
  __syncthreads();
#pragma unroll 4
  for (int t = threadIdx.x; t < Ls * CT; t += blockDim.x) {
    const int c = c0 + (t % CT);
    acc[t] = c < a.ncol ? fft_gather(a, rng + 4 * (t / CT), c) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int vi = vlo; vi < a.nv; ++vi) {
    const FftV V = a.v[vi];
    const int n = V.L * CT, tws = Ls / V.L;
    for (int t = threadIdx.x; t < n; t += blockDim.x) buf[t] = acc[t];
    for (int j = threadIdx.x; j < V.L; j += blockDim.x) tw[j] = twL[j * tws];
    __syncthreads();
    fft_smem<CT, 1, false>(buf, V.p, tw);
    int64_t* rows = reinterpret_cast<int64_t*>(rng);            // the gather bounds are dead by now
    fft_rows_of(a, vi, 0, 1, V.L, rows);
    const double2* H = a.H + V.hoff;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int f = t / CT, col = t % CT, fb = (V.L - f) & (V.L - 1);
      if (fb < f) continue;
      double2 wa, wb;
      fft_mult(buf[f * CT + col], buf[fb * CT + col], H[f], H[fb], &wa, &wb);
      buf[f * CT + col] = wa;
      if (fb != f) buf[fb * CT + col] = wb;
    }
    __syncthreads();
    fft_smem<CT, 1, true>(buf, V.p, tw);
    fft_scatter<CT>(a, V, buf, rows, n, c0);
    for (int t = threadIdx.x; t < n / 2; t += blockDim.x) acc[t] = cadd(acc[t], acc[t + n / 2]);
    __syncthreads();
  }
}

// rows with valuation >= k-2 (0, 2^(k-1), 2^(k-2), 3 2^(k-2)) by the definition: P[r, c] =
// sum_j phi((r z'_j mod M) / M) A[j, c], plus the parent row.  CTA = 32 columns x 8 warps; warp w sums
// j = w (mod 8), the 8 partial sums are added in fixed order.
__global__ void __launch_bounds__(256) k_fft_rows(const FftArgs a) {
  pdl_enter();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  __shared__ double xs[4][256];
  __shared__ double red[8][4][32];
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
      for (int jj = warp; jj < n; jj += 8) {
        const double av = a.A[(int64_t)(j0 + jj) * a.lda + c];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(xs[q][jj], av, acc[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) red[warp][q][lane] = acc[q];
  __syncthreads();
  if (warp < 4 && c < a.ncol) {
    const int q = warp;
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][q][lane];
    if (a.Rp) v += a.Rp[(int64_t)(rr[q] % (uint64_t)a.Mp) * a.ldp + c];
    RQMC_DCHECK(a.R + (int64_t)rr[q] * a.ldr + c, 8);
    a.R[(int64_t)rr[q] * a.ldr + c] = v;
  }
}

cudaError_t launch_fft_level(const FftArgs& a0, cudaStream_t st) {
  // valuations [0, vs) have L > 256 (four-step over HBM), [vs, nv) run in k_fft_small
  int vs = 0;
  while (vs < a0.nv && a0.v[vs].p > kFftSmallLg) ++vs;
  int n1 = 0, n1h = 0, n2 = 0, L1 = 1, L2 = 1, Ls = 1;
  for (int i = 0; i < a0.nv; ++i) {
    n1h += a0.v[i].L2;
    if (i < vs) { n1 += a0.v[i].L2; n2 += a0.v[i].L1 / 2 + 1; L1 = max(L1, a0.v[i].L1); L2 = max(L2, a0.v[i].L2); }
    else Ls = max(Ls, a0.v[i].L);
  }
  for (int i = vs; i < a0.nv; ++i) L1 = max(L1, a0.v[i].L1);   // pass 1 (mode 1) covers every valuation
  const int s1 = (int)sizeof(double2) * (L1 * kFftCT + 2 * L1) + 4 * L1 * (int)sizeof(int);
  const int s2 = (int)sizeof(double2) * (2 * L2 * (kFftCT / 2) + 5 * L2);
  const int ss = (int)sizeof(double2) * (2 * Ls * kFftCT + 2 * Ls) + 4 * Ls * (int)sizeof(int);
  cudaError_t e;
  if ((e = set_smem_once(k_fft_pass1, s1)) != cudaSuccess) return e;
  if ((e = set_smem_once(k_fft_pass2, s2)) != cudaSuccess) return e;
  if ((e = set_smem_once(k_fft_pass3, s1)) != cudaSuccess) return e;
  if ((e = set_smem_once(k_fft_small, ss)) != cudaSuccess) return e;
  // H_v and its spectrum (one column): pass 1 for every valuation, pass 2 for the long ones
  FftArgs h = a0;
  h.Z = a0.H; h.ldz = 1; h.ncol = 1;
  for (int i = 0; i < h.nv; ++i) h.v[i].zoff = h.v[i].hoff;
  if ((e = launch_k(k_fft_pass1, dim3(1, n1h), dim3(kFftThreads), s1, st, true, h, 1, 0, h.nv)) != cudaSuccess) return e;
  if (vs > 0 && (e = launch_k(k_fft_pass2, dim3(1, n2), dim3(kFftThreads), s2, st, true, h, 1, 0, vs)) != cudaSuccess)
    return e;
  const unsigned g16 = (unsigned)((a0.ncol + kFftCT - 1) / kFftCT);
  const unsigned g8 = (unsigned)((a0.ncol + kFftCT / 2 - 1) / (kFftCT / 2));
  if (vs > 0) {
    if ((e = launch_k(k_fft_pass1, dim3(g16, n1), dim3(kFftThreads), s1, st, true, a0, 0, 0, vs)) != cudaSuccess) return e;
    if ((e = launch_k(k_fft_pass2, dim3(g8, n2), dim3(kFftThreads), s2, st, true, a0, 0, 0, vs)) != cudaSuccess) return e;
    if ((e = launch_k(k_fft_pass3, dim3(g16, n1), dim3(kFftThreads), s1, st, true, a0, 0, vs)) != cudaSuccess) return e;
  }
  if (vs < a0.nv && (e = launch_k(k_fft_small, dim3(g16), dim3(kFftThreads), ss, st, true, a0, vs)) != cudaSuccess)
    return e;
  return launch_k(k_fft_rows, dim3((unsigned)((a0.ncol + 31) / 32)), dim3(256), 0, st, true, a0);
}

#if RQMC_DEBUG
cudaError_t dbg_set_fft(const DbgRanges& r, cudaStream_t st) { return dbg_set_tu(r, st); }
#else
cudaError_t dbg_set_fft(const DbgRanges&, cudaStream_t) { return cudaSuccess; }
#endif

}  // namespace rqmc
