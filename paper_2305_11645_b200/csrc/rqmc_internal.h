// Internal interface between the host planner (rqmc_plan.cpp) and the sm_100a kernels
// (rqmc_kernels.cu).  Not part of the public C ABI (include/rqmc.h).
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace rqmc {

constexpr int kMaxLevels = 64;
constexpr int kMaxFine = 7;       // fused fine levels (compile-time DFS depth; 8 never fits the smem bound)
constexpr int kFineSlots = 8;     // FineArgs::lv entries (kept at 8: the kernels' parameter layout with 8
                                  // slots lets ptxas allocate the C5 tree without spills)
constexpr int kBundle = 32;       // residues of the checkpoint level per fine CTA
constexpr int kSplitSlots = 512;  // max tail bundles split over two CTAs (FineArgs::rscr)
constexpr int kFineBN = 32;       // column tile of the fine kernel
constexpr int kFinePad = 36;      // padded t / c stride (doubles) of the fine kernel's smem tiles
constexpr int kFineThreads = 256;
constexpr int kMaxSeg = 8;        // merged coarse levels per gathered GEMM (GemmArgs::nseg)

// Point-generation view of one level (local rows r'' of this rank).
struct GenLevel {
  int64_t M;      // global distinct rows b^{m-w}
  int64_t Ml;     // local rows
  int64_t xoff;   // offset (doubles) of X^red in the workspace
  int j_lo, s_w, ldx, tc_log;   // tc_log: log2 of the generator's column-tile width min(32, pow2 >= ldx)
  double inv_M;   // 2^-(m-w) for b = 2 (exact scaling of t / M)
  int mixed;      // merged coarse levels (Layout::absorb): coordinate j has its own M_j = b^(m - w_j)
};

struct GenArgs {
  int kind, map, b, m, shifted, nlev;
  // residue-class partition: this rank owns classes c0 .. c0+nc-1 of k mod ncls (ncls = b^gamma);
  // local row l of a level with M >= ncls is global residue c0 + (l mod nc) + ncls (l div nc), of a
  // level with M < ncls residue (c0 + l) mod M (nc replicated rows)
  int64_t ncls, c0; int nc;
  double zero_u;                 // u substituted for 0 under Phi^-1 (reading C-5)
  const uint64_t* z;             // lattice z'_j
  const double* shift;           // lattice Delta_j
  const uint64_t* C;             // net column words (row-zeroed)
  const uint64_t* dshift;        // net sigma_j
  uint64_t seed;                 // reduced MC generator seed
  const int* wcl;                // min(w_j, m) per coordinate (merged levels, GenLevel::mixed)
  // replicas (batched randomisation, NEXT-2): replica r = blockIdx.z uses shift[r*srep + j] /
  // dshift[r*srep + j] / seeds[r] (seeds NULL: seed) and writes X + r*xrep
  int srep;
  int64_t xrep;
  const uint64_t* seeds;
  double* X;                     // workspace base
  unsigned int* zcnt; int nzcnt; // fine-kernel split counters to zero (replica stride 2 xrep)
  GenLevel lv[kMaxLevels];
};

struct GemmArgs {                // one coarse level: R = tile(Rp) + X A_w
  const double* X; int64_t ldx;
  int64_t M;                     // local rows of this level
  int K;                         // s_w
  const double* A; int64_t lda;  // A + j_lo * lda
  int tau;
  const double* Rp; int64_t ldp; int64_t Mp;   // parent R (nullptr: zero)
  double* R; int64_t ldr;
  int64_t xrep, rrep;            // replica strides (doubles) of X and of the R buffers (grid.z = replica)
  // pair mode (Xc != nullptr): this level's R stays on chip and seeds the next finer level c, whose
  // local rows u M + r (u < ncu) have parent row r; R (this level) is not written, Rc (ldr) is
  const double* Xc; int64_t ldxc; int Kc; const double* Ac; double* Rc; int ncu;
  // merged coarse levels by gather (Layout::gather): column q of this GEMM's X operand lies in segment
  // i (segq[i] <= q < segq[i+1]), i.e. at row r mod segM[i], column q - segq[i] of the X^red segX[i]
  // (leading dimension segld[i]) of one merged level -- the same points (x_{r,j} depends on r mod M_j,
  // P:307-309) without generating them again at the absorbing level's rows.  nseg = 0: X is one
  // level's X^red.
  int nseg; int segq[kMaxSeg + 1]; const double* segX[kMaxSeg]; int64_t segld[kMaxSeg], segM[kMaxSeg];
};

struct FineLevel {
  const double* X; int ldx; int K; int j_lo; int fan; int runs; int xs_off; int as_off;
};

struct FineArgs {
  const double* root; int64_t ldroot; int64_t Mroot;
  int NF;
  FineLevel lv[kFineSlots];
  const double* A; int64_t lda; int tau; int a_vec;  // a_vec: 16B cp.async allowed
  double* Y; int64_t ldy; int y_vec;  // y_vec: 16B stores allowed
  int fk; double fp0, fp1;
  double* partial;
  int leafruns;
  int as_stride;      // doubles per A buffer
  int root_off;       // root tile buffers offset (doubles), 2 x kBundle x kFinePad
  int acc_off;        // rowacc offset (doubles)
  int smem_bytes;
  int64_t xrep, rootrep, partrep;  // replica strides (doubles): X^red, root R, partials (grid.y = replica)
  // tail split (b = 3 tree kernel): the last bundles of a grid whose final wave would be at most half
  // full run as two CTAs over half the column tiles each; their per-row g sums meet in rscr and the
  // second CTA to finish (counter rcnt[slot], zeroed by k_gen) applies F in fixed order (half 0 + 1)
  double* rscr; int64_t rscr_cap;  // scratch (doubles per replica slice)
  unsigned int* rcnt; int ncnt;    // counters per replica slice (stride 2 partrep)
  int64_t nfull; int nsplit;       // set by the launcher
  // Y row map of a residue chunk (rqmc_plan.cpp, chunked xa): local row l is stored at global row
  // ym_c0 + (l mod ym_nc) + ym_ncls (l div ym_nc); ym_nc = 0: row l.  Leaf rows of one residue are
  // l = r + j Mroot (Mroot a multiple of ym_nc), i.e. global rows y_row(r) + j ystride with
  // ystride = Mroot (ym_nc = 0) or ym_ncls Mroot / ym_nc: the kernels map once per thread.
  int64_t ym_c0, ym_ncls; int ym_nc;
  // a5 final reduction fused into the fine kernel (finish_fsum): the last CTA of replica r to write its
  // partial (arrival counter rcnt[kSplitSlots + r * 2 partrep], zeroed by k_gen every call) adds the
  // replica's partials in fixed order into fsum[r].  fsum = nullptr: the partials are left for k_reduce.
  // (One pointer only: ptxas's allocation of the C5 tree is sensitive to this struct's layout.)
  double* fsum;
};

// NEXT-4: one FFT-product level (rqmc_fft.cu).  Per valuation v (K = k - v >= 3): L = 2^(K-2) = L1 L2,
// lgL1/lgL2 = log2, p = k - 2 - v bits of e, boff = offset of its bucket table (2 (L + 1) starts into
// jsort: sigma = + then -, in bit-reversed e order), zoff / hoff = offsets (complex elements) of its
// block in the data buffer Z (L rows x ldz) and in the H buffer (L entries).
struct FftV { int L, L1, L2, lgL1, lgL2, p, boff; int64_t zoff, hoff; };
struct FftArgs {
  int k, nv, s_w, ncol, ldz, map;
  double zero_u, inv_M;                         // unshifted zero rule, 2^-k
  const double* A; int64_t lda;                 // the level's rows of A (A + j_lo lda)
  const int* jsort; const int* boff;            // coordinates sorted by (sigma, bitrev(e_j)); bucket starts
  const uint64_t* z;                            // the level's z'_j
  double2* Z; double2* H;                       // scratch
  const double* Rp; int64_t ldp, Mp;            // parent R (nullptr: top level)
  double* R; int64_t ldr;
  FftV v[32];
};
cudaError_t launch_fft_level(const FftArgs& a, cudaStream_t st);

// debug build (RQMC_DEBUG): device address ranges a run may touch; each translation unit keeps its
// own __constant__ copy, set by its dbg_set_* before the run's launches (rqmc_device.cuh)
struct DbgRanges { const char* lo[6]; const char* hi[6]; };
cudaError_t dbg_set_gen(const DbgRanges& r, cudaStream_t st);
cudaError_t dbg_set_gemm(const DbgRanges& r, cudaStream_t st);
cudaError_t dbg_set_fine(const DbgRanges& r, cudaStream_t st);
cudaError_t dbg_set_tree(const DbgRanges& r, cudaStream_t st);
cudaError_t dbg_set_fft(const DbgRanges& r, cudaStream_t st);

cudaError_t launch_gen(const GenArgs& a, int64_t max_entries, int nrep, cudaStream_t st);
cudaError_t launch_points(const GenArgs& a, int lev, int64_t r0, int64_t count, uint64_t* words,
                          double* vals, cudaStream_t st);
cudaError_t launch_gemm(const GemmArgs& a, int nrep, cudaStream_t st);
// nparts: partial sums left for k_reduce per replica, 0 when the kernel added them itself (finish_fsum)
// (the tree kernel's bundles may be smaller than kBundle;
// the workspace holds 4 nbundles partials per replica)
cudaError_t launch_fine(const FineArgs& a, int64_t nbundles, int nrep, cudaStream_t st, int64_t* nparts);
// host only: the fine-kernel template launch_fine would pick (for tests / rqmc_plan_dispatch)
int describe_fine(const FineArgs& a, char* buf, size_t n);
cudaError_t launch_reduce(const double* partial, int64_t n, int64_t stride, int nrep, double* out, cudaStream_t st);

}  // namespace rqmc
