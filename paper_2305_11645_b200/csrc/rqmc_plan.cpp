// Host side of the C ABI (include/rqmc.h): validation, the level planner,
// workspace layout and the launch sequence of one run.  No arithmetic of the product lives here.
//
// Level planner: levels w = min(w_j, m) are contiguous j-ranges because w is
// nondecreasing; s* = max{j : w_j < m} drops the zero columns j > s*
// unless a shift or the Phi^-1 map makes them a constant row (reading C-4, kept as a 1-row level m).
// Each non-empty level's parent is the next coarser non-empty level w' (tile factor b^{w'-w},
// reading C-3).  A checkpoint level splits the table into coarse levels (one DMMA GEMM launch each,
// R materialised in the workspace) and <= 8 fine levels fused into k_fine.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: phase ranges for nsys / ncu --nvtx

#include "../../include/rqmc.h"
#include "rqmc_internal.h"

#ifndef RQMC_DEBUG
#define RQMC_DEBUG 0
#endif

using namespace rqmc;

namespace {

struct Level {
  int w, j_lo, s_w, parent, coarse;
  int fft_tab;    // index into rqmc_plan_s::fft (FFT-eligible level, NEXT-4), -1 otherwise
  int fft;        // layout: this coarse level runs as the FFT product (rqmc_fft.cu) instead of the GEMM
  int absorbed;   // layout: merged into the absorbing level below it (Layout::absorb)
  int s_gemm;     // layout: coordinates of this level's GEMM (s_w, or all merged levels' for the absorbing one)
  int fused;      // coarse pair parent: R stays on chip, computed with its child (next level) in one launch
  int64_t M, Ml;
  int ldx;
  int64_t xoff;   // doubles
  int rbuf;       // coarse: which R buffer
};

// Everything that depends on the checkpoint level: which levels are coarse, X^red strides and
// offsets, R buffers, fine-kernel shared-memory layout, workspace offsets.
struct Layout {
  int ckpt = -1, nfine = 0;
  int absorb = 0;            // levels 0 .. absorb-1 merged into level `absorb` (one GEMM, latency regime)
  int gather = 0;            // merged levels keep their own X^red; the GEMM gathers (GemmArgs::nseg)
  int64_t nbundles = 0;
  std::vector<Level> lv;     // copy of the plan's levels with coarse / ldx / xoff / rbuf filled
  int ldr = 0;               // row stride of R buffers
  size_t off_x = 0, off_r[2] = {0, 0}, off_part = 0, off_a = 0, off_fsum = 0, total = 0;
  size_t off_split = 0, off_cnt = 0; int64_t split_cap = 0;   // fine-kernel tail split (FineArgs::rscr)
  size_t off_fz = 0, off_fh = 0;   // FFT levels: complex scratch (data, H) shared by the FFT levels
  int64_t max_gen_entries = 0;
  int fine_smem = 0, fine_as_stride = 0, fine_acc_off = 0, leafruns = 1;
  std::vector<int> fine_xs_off, fine_as_off;
};

int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
bool is_prime(int b) {
  if (b < 2) return false;
  for (int d = 2; (int64_t)d * d <= b; ++d)
    if (b % d == 0) return false;
  return true;
}
int64_t gcd64(int64_t a, int64_t b) {
  while (b) { int64_t t = a % b; a = b; b = t; }
  return a;
}
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// NVTX range per phase of a run (host-side markers; free when no tool is attached).  During CUDA-graph
// capture they mark the captured sequence once.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
struct NvtxPhase {            // consecutive phases: next() closes the previous range
  bool open = false;
  void next(const char* name) { if (open) nvtxRangePop(); nvtxRangePushA(name); open = true; }
  ~NvtxPhase() { if (open) nvtxRangePop(); }
};

// NEXT-4 FFT level tables: coordinates of the level sorted by (sigma_j, bitrev_{k-2}(e_j)) where
// z'_j = sigma_j 5^(e_j) (mod 2^k), k = m - w (rqmc_fft.cu)
struct FftTab {
  int k = 0, nplus = 0;
  std::vector<int> jsort;        // level-relative coordinate indices
  std::vector<uint32_t> key;
  std::vector<int> boff;         // per valuation v: 2 (L_v + 1) bucket starts (sigma = +, -)
  std::vector<int> boff_v;       // offset of valuation v's table in boff
  size_t dev_j = 0, dev_k = 0;   // element offsets into the plan's device table
};

// discrete log base 5 in U_{2^k} (k >= 3): the e in [0, 2^(k-2)) with 5^e = z (mod 2^k), z = 1 (mod 4).
// Bit i of e is fixed modulo 2^(i+3), since 5^(2^i) = 1 + 2^(i+2) (mod 2^(i+3)).
uint32_t dlog5(uint64_t z, int k) {
  const uint64_t mask = (1ull << k) - 1;
  uint64_t p = 1, g = 5;
  uint32_t e = 0;
  for (int i = 0; i < k - 2; ++i) {
    const uint64_t mi = (1ull << (i + 3)) - 1;
    if ((p & mi) != (z & mi)) { e |= 1u << i; p = (p * g) & mask; }
    g = (g * g) & mask;
  }
  return e;
}

// FFT-eligible levels (NEXT-4): unshifted base-2 lattice, one process (the FFT computes every row of a
// level), 3 <= k = m - w <= 18 (FFT lengths L = 2^(k-2-v) <= 2^16 = 256 x 256, two passes)
constexpr int kFftMinK = 3, kFftMaxK = 18;
// default rule: the FFT replaces s_w M tau MACs by ~5 M log2 M tau flops plus three passes over its
// scratch (HBM-bound, 1.2-2.2 TB/s measured) while the DMMA GEMM costs ~60 fs per coordinate and
// element; measured crossover at s_w = 512 (C5U: w = 11 / 10 / 9 FFT 0.87 / 1.23 / 1.91 ms vs GEMM
// 2.01-2.03 ms; w = 8 3.18 vs 2.02 ms; profiles/r02_fft_levels_C5U_v2.txt).  RQMC_FFT=1 forces every
// eligible coarse level, RQMC_FFT=0 disables.
constexpr int kFftMinS = 512;

}  // namespace

struct rqmc_plan_s {
  int b = 0, m = 0, s = 0, tau = 0, kind = 0, map = 0, rank = 0, world = 1;
  int64_t ncls = 1, c0 = 0; int nc = 1;   // residue classes k mod ncls; this rank owns [c0, c0 + nc)
  bool shifted = false;
  uint64_t seed = 0;         // reduced MC
  int64_t N = 0, Nl = 0;
  int s_star = 0;
  std::vector<int32_t> w;
  std::vector<int> wlev;     // level w of each coordinate (device: merged levels' per-coordinate period)
  int* d_wl = nullptr;
  std::vector<uint64_t> z, C, dshift;
  std::vector<double> shift;
  std::vector<Level> lv;     // coarse -> fine (checkpoint-independent fields)
  std::vector<FftTab> fft;   // FFT-eligible levels' tables
  int* d_fft = nullptr;      // device copy: all jsort then all keys
  Layout L1;                 // layout of single runs (and the default workspace)
  std::mutex lay_mu;         // batch layouts (deeper checkpoints when replicas add parallelism)
  std::vector<std::unique_ptr<Layout>> lay_cache;
  // device tables (uploaded once, lazily)
  std::once_flag up_once;
  // CUDA graphs of single runs (launch overhead dominates the small configs): key -> executable graph
  struct GraphEntry {
    const void *dA, *dY, *d_fsum, *dwork;
    int64_t lda, ldy;
    int f;
    double fp0, fp1;
    cudaGraphExec_t exec;
    uint64_t last_use;
  };
  std::mutex graph_mu;
  std::vector<GraphEntry> graphs;
  uint64_t graph_clock = 0;
  cudaStream_t cap_stream = nullptr;
  // rqmc_qn_host: copy stream + events so that the H2D of A overlaps the point generation
  std::mutex h2d_mu;
  cudaStream_t h2d_stream = nullptr;
  cudaEvent_t h2d_ev[2] = {nullptr, nullptr};
  // A arrives in the order the run reads it: one copy (and event) per coarse level, then the fine rows
  std::vector<cudaEvent_t> h2d_lv_ev;   // per level index; the last entry: the fine levels' rows
  double* h_fsum_pin = nullptr;         // pinned landing slot of the f-sum (graph-captured host runs)
  struct HostGraph { const void *hA, *dwork; const void* dY; int64_t lda, ldy; int f; double fp0, fp1; cudaGraphExec_t exec; };
  std::vector<HostGraph> host_graphs;
  cudaError_t up_err = cudaSuccess;
  uint64_t* d_z = nullptr;
  double* d_shift = nullptr;
  uint64_t* d_C = nullptr;
  uint64_t* d_ds = nullptr;
  std::vector<int> fft_host; // staging of d_fft
  // residue-chunk pipeline of rqmc_xa (Y stored, one process): sub-plans over contiguous groups of
  // the residue classes k mod chunk_ncls, whose coarse GEMMs (main stream) overlap the previous
  // chunk's HBM-bound fine kernel (side stream)
  std::vector<std::unique_ptr<rqmc_plan_s>> chunks;
  std::vector<size_t> chunk_off;       // workspace offset of each chunk's slice
  size_t chunk_sums = 0, chunk_total = 0;
  int64_t chunk_ncls = 0;
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  // phase profiling: 5 events per recorded run
  std::vector<cudaEvent_t> prof_ev;
  int prof_max = 0, prof_runs = 0;
  std::string err;
};

namespace {

rqmc_status fail(rqmc_plan_s* p, rqmc_status st, const std::string& msg) {
  if (p) p->err = msg;
  return st;
}

thread_local std::string g_create_err;

// Shared-memory bytes of the fine kernel when the checkpoint is level index c.
int fine_smem_bytes(const rqmc_plan_s& p, int c, std::vector<int>* xs_off, std::vector<int>* as_off,
                    int* as_stride, int* acc_off, int* leafruns) {
  const int nl = (int)p.lv.size();
  size_t xs = 0, as = 0;
  if (xs_off) xs_off->clear();
  if (as_off) as_off->clear();
  const int64_t Mroot = p.lv[c].Ml;
  int lr = 1;
  for (int i = c + 1; i < nl; ++i) {
    const int64_t runs = p.lv[i].Ml / Mroot;
    if (xs_off) xs_off->push_back((int)xs);
    if (as_off) as_off->push_back((int)as);
    xs += (size_t)runs * p.lv[i].s_w * kFinePad;
    as += (size_t)p.lv[i].s_w * kFinePad;
    lr = (int)runs;
  }
  xs = align_up(xs, 2);
  as = align_up(as, 2);
  const size_t acc = (size_t)lr * kBundle;  // one row-sum slot per leaf row (groups are disjoint)
  // layout: [A buf 0][A buf 1][root buf 0][root buf 1][X subtree][rowacc]
  const size_t roots = 2 * (size_t)kBundle * kFinePad;
  if (as_stride) *as_stride = (int)as;
  if (xs_off)
    for (auto& o : *xs_off) o += (int)(2 * as + roots);
  if (acc_off) *acc_off = (int)(2 * as + roots + xs);
  if (leafruns) *leafruns = lr;
  return (int)((2 * as + roots + xs + acc) * sizeof(double));
}

#ifndef RQMC_FINE_SMEM_LIMIT_KB   // A/B builds: admit deeper fused subtrees (the kernel's own SMEM still bounds them)
#define RQMC_FINE_SMEM_LIMIT_KB 200
#endif
constexpr int kFineSmemLimit = RQMC_FINE_SMEM_LIMIT_KB * 1024;

// Checkpoint choice: the most fused fine levels subject to depth <= kMaxFine, shared memory, and at
// least 2 waves of fine CTAs (bundles x replicas >= 2 x 148 SMs) -- replicas of a batched run add
// parallelism, so a batch may fuse more levels than a single run of the same plan.  With few column
// tiles (tau < 1024) a deep subtree's X^red load is amortised over too little work: depth <= 4
// (C2 x 64 replicas: 2.83 ms fused 4 deep, 4.19 ms 6 deep, 3.61 ms 2 deep).
int choose_ckpt(const rqmc_plan_s& p, int64_t reps) {
  const int nl = (int)p.lv.size();
  const int max_nf = p.tau < 1024 ? 4 : kMaxFine;
  int best = -1;
  for (int c = 0; c < nl; ++c) {
    const int nf = nl - 1 - c;
    if (nf > max_nf && c + 1 < nl) continue;
    if (fine_smem_bytes(p, c, nullptr, nullptr, nullptr, nullptr, nullptr) > kFineSmemLimit) continue;
    const int64_t nb = (p.lv[c].Ml + kBundle - 1) / kBundle;
    if (best < 0) best = c;
    // enough bundles (kBundle = 32 residues) for >= 148 16-residue tree CTAs: a finer checkpoint
    // costs one more GEMM launch, which measured worse than a partial wave (C2: 85.7 vs 90.2 us)
    if (nb * reps >= 74) { best = c; break; }
    best = c;  // keep moving finer while parallelism is insufficient
  }
  const char* env = std::getenv("RQMC_CKPT_W");        // tuning override: checkpoint at level w
  if (env && *env) {
    const int wv = std::atoi(env);
    for (int c = 0; c < nl; ++c)
      if (p.lv[c].w == wv && nl - 1 - c <= kMaxFine &&
          fine_smem_bytes(p, c, nullptr, nullptr, nullptr, nullptr, nullptr) <= kFineSmemLimit)
        best = c;
  }
  return best;
}

// Workspace layout for checkpoint c: [X^red of every level][R buf 0][R buf 1][partials] (one
// replica's slice, off_fsum bytes) then [f-sum][A staging] for the host entry point.
// Latency regime of small problems: the top coarse levels 0 .. a-1 are merged into level a (one GEMM
// over all their coordinates at level a's M_a rows: x_{r,j} depends on r mod M_j, so the
// merged rows are the same points): one launch instead of a + 1 dependent ones, for more MACs
// (Σ_{i<a} s_i (M_a - M_i) τ) and as many more generated entries (each a Φ^-1 when mapped).  Taken
// while the merged GEMM stays under kAbsorbMacs multiply-adds (replicas together) and the extra
// entries under a x 2^20 (unit map; a x 2^17 for reduced-MC draws).  C1: 6 coarse GEMMs -> 1
// (43.9 -> 18.9 us).  RQMC_ABSORB=0 disables.
constexpr double kAbsorbMacs = 268435456.0;   // 2^28 (~7 us at the fp64 peak)
constexpr double kGatherMacs = 67108864.0;    // 2^26: the gathered GEMM stays in k_level_gemm_lat's regime
// Φ^-1-mapped points merge by gather (Layout::gather): generating the merged columns at level a's rows
// would evaluate Σ_{i<a} s_i (M_a - M_i) extra Φ^-1 (C2: all coarse levels merged that way 93 -> 112 us,
// three of five 91 -> 100 us), so the merged levels keep their own X^red and the latency-regime GEMM
// reads column q of level i at row r mod M_i.  Every merged level but the coarsest must start a 16-byte
// chunk (even cumulative s_w), and level a's rows fit one grid (< 2^21: 32-row tiles, grid.y <= 65535).
int choose_absorb_gather(const rqmc_plan_s& p, const Layout& L, int c, int64_t reps) {
  int a = 0;
  for (int i = 1; i <= c && i < kMaxSeg; ++i) {
    if (L.lv[0].fft || L.lv[i].fft) break;
    double K = 0.0;
    bool even = true;
    for (int q = i; q >= 0; --q) {
      if (q < i && ((int64_t)K % 2) != 0) even = false;   // segment q starts at column K
      K += L.lv[q].s_w;
    }
    if (!even || L.lv[i].Ml >= (int64_t(1) << 21) || (double)L.lv[i].Ml * p.tau * K * reps > kGatherMacs) break;
    a = i;
  }
  return a;
}
int choose_absorb(const rqmc_plan_s& p, const Layout& L, int c, int64_t reps) {
  const char* e = std::getenv("RQMC_ABSORB");
  if (e && *e && *e == '0') return 0;
  if (p.map != RQMC_MAP_UNIT) return choose_absorb_gather(p, L, c, reps);
  const double per = p.kind == RQMC_REDUCED_MC ? 131072.0 : 1048576.0;
  int a = 0;
  for (int i = 1; i <= c; ++i) {
    if (L.lv[0].fft || L.lv[i].fft) break;
    double s_acc = 0.0, extra = 0.0;
    for (int q = 0; q <= i; ++q) {
      s_acc += L.lv[q].s_w;
      extra += (double)L.lv[q].s_w * (double)(L.lv[i].Ml - L.lv[q].Ml);
    }
    if ((double)L.lv[i].Ml * p.tau * s_acc * reps > kAbsorbMacs || extra * reps > per * i) break;
    a = i;
  }
  return a;
}

void make_layout(const rqmc_plan_s& p, int c, Layout& L, int64_t reps = 1) {
  const int nl = (int)p.lv.size();
  L.ckpt = c;
  L.nfine = nl - 1 - c;
  L.lv = p.lv;
  for (int i = 0; i < nl; ++i) L.lv[i].coarse = i <= c;
  const char* fe = std::getenv("RQMC_FFT");   // read per plan (tests switch it)
  const int fft_mode = fe && *fe ? std::atoi(fe) : -1;
  for (int i = 0; i < nl; ++i) {
    Level& V = L.lv[i];
    V.fft = V.coarse && V.fft_tab >= 0 && fft_mode != 0 && (fft_mode == 1 || V.s_w >= kFftMinS);
    V.absorbed = 0;
    V.s_gemm = V.s_w;
  }
  L.absorb = choose_absorb(p, L, c, reps);
  L.gather = L.absorb > 0 && p.map != RQMC_MAP_UNIT;
  for (int i = 0; i < L.absorb; ++i) {
    L.lv[i].absorbed = 1;
    L.lv[L.absorb].s_gemm += L.lv[i].s_w;   // coarser coordinates follow level a's contiguously in j
  }
  if (L.absorb > 0) L.lv[L.absorb].parent = -1;
  L.nbundles = (L.lv[c].Ml + kBundle - 1) / kBundle;
  L.fine_smem = fine_smem_bytes(p, c, &L.fine_xs_off, &L.fine_as_off, &L.fine_as_stride, &L.fine_acc_off,
                                &L.leafruns);
  size_t off = 0;
  L.off_x = 0;
  L.max_gen_entries = 0;
  for (auto& V : L.lv) {
    V.ldx = V.coarse ? ((L.gather ? V.s_w : V.s_gemm) + 1) / 2 * 2 : V.s_w;
    V.xoff = (int64_t)(off / sizeof(double));
    if (V.fft || (V.absorbed && !L.gather)) continue;   // FFT levels need no X^red (H tables in rqmc_fft.cu);
                                         // merged ones are generated as the absorbing level's columns
                                         // (unit map) or keep their own X^red (gather)
    off = align_up(off + (size_t)V.Ml * V.ldx * sizeof(double), 256);
    L.max_gen_entries = std::max<int64_t>(L.max_gen_entries, V.Ml * V.ldx);
  }
  L.ldr = (p.tau + 1) / 2 * 2;
  // coarse pairs (c-1, c), (c-3, c-2), ...: the parent's R stays on chip when each of its rows has
  // <= 4 child rows.  Opt-in (RQMC_GEMM_PAIR=1): bit-identical, but the pair kernel holds two
  // accumulator tiles (167 registers, 3 CTAs per SM) and measured slower on C5 (coarse 15.06 vs
  // 13.54 ms) although it saves R_7's 4.3 GB round trip.  Stored levels alternate R buffers.
  static const bool no_pair = [] { const char* e = std::getenv("RQMC_GEMM_PAIR"); return !(e && *e && *e != '0'); }();
  for (int i = 0; i <= c; ++i) L.lv[i].fused = 0;
  for (int i = c - 1; i >= L.absorb + L.gather && !no_pair; i -= 2) {   // (a gathered GEMM is never a pair)
    const Level &P = L.lv[i], &C = L.lv[i + 1];
    const int64_t ncu = C.Ml / P.Ml;
    if (C.parent == i && ncu * P.Ml == C.Ml && ncu >= 1 && ncu <= 4 && !P.fft && !C.fft) L.lv[i].fused = 1;
  }
  size_t rsz[2] = {0, 0};
  int nstored = 0;
  for (int i = 0; i <= c; ++i) {
    if (L.lv[i].fused || L.lv[i].absorbed) { L.lv[i].rbuf = -1; continue; }
    const int b = nstored++ & 1;
    L.lv[i].rbuf = b;
    rsz[b] = std::max(rsz[b], (size_t)L.lv[i].Ml * L.ldr * sizeof(double));
  }
  L.off_r[0] = off; off = align_up(off + rsz[0], 256);
  L.off_r[1] = off; off = align_up(off + rsz[1], 256);
  L.off_part = off; off = align_up(off + (size_t)4 * L.nbundles * sizeof(double), 256);  // see launch_fine
  {  // tail-split scratch (b = 3 trees): up to kSplitSlots bundles x 2 halves x kBundle b^nfine rows
    int64_t rows = kBundle;
    for (int i = 0; i < L.nfine && rows <= (int64_t(1) << 30); ++i) rows *= p.b;
    const int64_t cap = (int64_t)kSplitSlots * 2 * rows;
    L.split_cap = (p.b == 3 && L.nfine > 0 && cap * 8 <= (int64_t(64) << 20)) ? cap : 0;
    L.off_split = off; off = align_up(off + (size_t)L.split_cap * sizeof(double), 256);
    // counters: kSplitSlots split counters, then the fine kernel's arrival counter (finish_fsum)
    L.off_cnt = off; off = align_up(off + (size_t)(kSplitSlots + 1) * sizeof(unsigned int), 256);
  }
  {  // FFT scratch: sum_v L_v complex per column (ldz = ldr) and per H, for the largest FFT level
    size_t zc = 0, hc = 0;
    for (const Level& V : L.lv)
      if (V.fft) {
        const int k = p.m - V.w;
        size_t sl = 0;
        for (int v = 0; v <= k - 3; ++v) sl += (size_t)1 << (k - 2 - v);
        zc = std::max(zc, sl * (size_t)L.ldr);
        hc = std::max(hc, sl);
      }
    L.off_fz = off; off = align_up(off + zc * 2 * sizeof(double), 256);
    L.off_fh = off; off = align_up(off + hc * 2 * sizeof(double), 256);
  }
  L.off_fsum = off; off = align_up(off + sizeof(double), 256);
  L.off_a = off; off = align_up(off + (size_t)p.s * L.ldr * sizeof(double), 256);
  L.total = off;
}

// Layout for a batch of `reps` concurrent replicas (cached; the single-run layout when equal).
// (f is kept for the ABI: the choice no longer depends on it.)
const Layout& layout_for(rqmc_plan_s* p, int64_t reps, int f) {
  (void)f;
  const int c = choose_ckpt(*p, reps);
  if (c < 0) return p->L1;
  Layout probe;
  make_layout(*p, c, probe, reps);
  if (c == p->L1.ckpt && probe.absorb == p->L1.absorb) return p->L1;
  std::lock_guard<std::mutex> lk(p->lay_mu);
  for (auto& L : p->lay_cache)
    if (L->ckpt == c && L->absorb == probe.absorb) return *L;
  p->lay_cache.emplace_back(new Layout(std::move(probe)));
  return *p->lay_cache.back();
}

// Residue-chunk pipeline for rqmc_xa (Y stored): the N x tau Y stream makes the fine kernel HBM-bound
// while the coarse GEMMs are fp64-bound, so splitting the problem into nchunk groups of the residue
// classes k mod ncls (ncls = the smallest coarse level M >= 8 nchunk; every subtree under one residue
// is independent) lets chunk i+1's coarse GEMMs overlap chunk i's fine kernel.  Each
// chunk is a sub-plan with the same levels and checkpoint and local rows c0 + (l mod nc) + ncls (l div
// nc); its fine kernel stores those rows of the caller's Y directly.  Y is bit-identical to the
// unchunked run (the same per-row arithmetic); the f-sum is the fixed-order sum of the chunk sums.
// Only for one process (world = 1), Y >= 2 GB (N tau >= 2^28), no FFT levels.  OPT-IN (RQMC_CHUNKS=n,
// n >= 2): measured slower on C4 (4.52 ms unchunked; 2 / 4 / 8 chunks 5.49 / 5.96 / 7.08 ms): a chunk's
// fine grid is 1.4 waves (638 CTAs on 444 slots, 1.16 ms vs 3.29 / 4 = 0.82), and the fine kernel
// holds every SM, so the next chunk's GEMMs barely overlap it (serialised kernel sum 6.39 ms vs 5.96 ms
// wall; profiles/r02_c4_chunks.txt).
void make_chunks(rqmc_plan_s* p) {
  const char* e = std::getenv("RQMC_CHUNKS");
  const int nch = e && *e ? std::atoi(e) : 0;
#if RQMC_DEBUG
  (void)nch;
  return;   // debug builds set their bounds per launch sequence on one stream
#else
  if (nch < 2 || p->world != 1 || p->ncls != 1 || (double)p->N * p->tau < (double)(1ull << 28)) return;
  const Layout& L = p->L1;
  for (int i = 0; i <= L.ckpt; ++i)
    if (L.lv[i].fft) return;
  int64_t ncls = 0;
  for (int i = 0; i <= L.ckpt; ++i)
    if (L.lv[i].M >= 8 * nch && (ncls == 0 || L.lv[i].M < ncls)) ncls = L.lv[i].M;
  if (ncls == 0) return;
  size_t off = 0;
  for (int c = 0; c < nch; ++c) {
    std::unique_ptr<rqmc_plan_s> q(new rqmc_plan_s());
    q->b = p->b; q->m = p->m; q->s = p->s; q->tau = p->tau; q->kind = p->kind; q->map = p->map;
    q->shifted = p->shifted; q->seed = p->seed; q->N = p->N; q->s_star = p->s_star;
    q->w = p->w; q->z = p->z; q->C = p->C; q->dshift = p->dshift; q->shift = p->shift; q->wlev = p->wlev;
    q->ncls = ncls;
    q->c0 = ncls * c / nch;
    q->nc = (int)(ncls * (c + 1) / nch - q->c0);
    q->Nl = q->nc * (p->N / ncls);
    q->lv = p->lv;
    for (Level& V : q->lv) {
      V.Ml = V.M >= ncls ? q->nc * (V.M / ncls) : q->nc;
      V.fft_tab = -1;
    }
    make_layout(*q, L.ckpt, q->L1);
    p->chunk_off.push_back(off);
    off = align_up(off + q->L1.total, 256);
    p->chunks.push_back(std::move(q));
  }
  p->chunk_sums = off;
  p->chunk_total = align_up(off + nch * sizeof(double), 256);
  p->chunk_ncls = ncls;
#endif
}

}  // namespace

extern "C" {

const char* rqmc_strerror(rqmc_status s) {
  switch (s) {
    case RQMC_OK: return "ok";
    case RQMC_EINVAL: return "invalid argument";
    case RQMC_ENOTPRIME: return "base b is not prime";
    case RQMC_EWORDER: return "reduction indices must be nondecreasing with w_1 = 0";
    case RQMC_EZUNIT: return "generating vector component is not a unit mod b^(m-w_j)";
    case RQMC_ESHIFT: return "shift outside [0,1) (or digital shift >= 2^53)";
    case RQMC_ENETMAT: return "invalid or non-periodic digital net generating matrices";
    case RQMC_EDIM: return "dimension mismatch";
    case RQMC_EDOMAIN: return "inverse normal domain error";
    case RQMC_ECUDA: return "CUDA error";
    case RQMC_ENOMEM: return "out of memory";
    case RQMC_EUNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

const char* rqmc_plan_last_error(rqmc_plan_t p) { return p ? p->err.c_str() : g_create_err.c_str(); }

rqmc_status rqmc_plan_create(const rqmc_plan_desc* d, rqmc_plan_t* out) {
  g_create_err.clear();
  if (!d || !out) return RQMC_EINVAL;
  *out = nullptr;
  auto bad = [&](rqmc_status st, const std::string& m) { g_create_err = m; return st; };
  if (d->m < 1 || d->s < 1 || d->tau < 1) return bad(RQMC_EDIM, "m, s, tau must be >= 1");
  if (!is_prime(d->b)) return bad(RQMC_ENOTPRIME, "b = " + std::to_string(d->b) + " is not prime");
  if (!d->w) return bad(RQMC_EINVAL, "w is NULL");
  if (d->kind != RQMC_LATTICE && d->kind != RQMC_DIGITAL_NET && d->kind != RQMC_REDUCED_MC &&
      d->kind != RQMC_DIGITAL_NET_ROWS)
    return bad(RQMC_EINVAL, "bad kind");
  // row-zeroed net (Alg. 3/4): the same generator as a net; only the level table differs
  const bool rowzero = d->kind == RQMC_DIGITAL_NET_ROWS;
  if (d->map != RQMC_MAP_UNIT && d->map != RQMC_MAP_INVNORM && d->map != RQMC_MAP_TENT) return bad(RQMC_EINVAL, "bad map");
  if (d->m * std::log2((double)d->b) > 32.0 + 1e-9) return bad(RQMC_EUNSUPPORTED, "N = b^m > 2^32");
  if ((d->kind == RQMC_DIGITAL_NET || rowzero) && (d->b != 2 || d->m > 32))
    return bad(RQMC_EUNSUPPORTED, "digital nets need b = 2, m <= 32");
  if (d->w[0] != 0) return bad(RQMC_EWORDER, "w_1 != 0 (P:284)");
  for (int j = 1; j < d->s; ++j)
    if (d->w[j] < d->w[j - 1])
      return bad(RQMC_EWORDER, "w decreases at j = " + std::to_string(j + 1));

  auto* p = new rqmc_plan_s();
  p->b = d->b; p->m = d->m; p->s = d->s; p->tau = d->tau; p->map = d->map;
  p->kind = rowzero ? RQMC_DIGITAL_NET : d->kind;
  p->N = ipow(d->b, d->m);
  p->world = d->world <= 0 ? 1 : d->world;
  p->rank = d->rank;
  {  // residue-class partition: world a power of b dividing N -> one class per rank;
     // else ncls = b^gamma (gamma <= m, the smallest with b^gamma >= 32 world) classes in contiguous
     // groups of floor / ceil(ncls / world) per rank (imbalance <= 1 + world / ncls <= 1.03)
    if (p->rank < 0 || p->rank >= p->world) {
      delete p;
      return bad(RQMC_EINVAL, "need 0 <= rank < world");
    }
    int64_t g = p->world;
    while (g > 1 && g % p->b == 0) g /= p->b;
    if (g == 1 && p->N % p->world == 0) {
      p->ncls = p->world; p->c0 = p->rank; p->nc = 1;
    } else {
      int64_t cl = 1;
      int gam = 0;
      while (gam < d->m && cl < 32 * (int64_t)p->world) { cl *= p->b; ++gam; }
      if (cl < p->world) {
        delete p;
        return bad(RQMC_EUNSUPPORTED, "world > N: fewer points than ranks");
      }
      p->ncls = cl;
      p->c0 = cl * p->rank / p->world;
      p->nc = (int)(cl * (p->rank + 1) / p->world - p->c0);
    }
  }
  p->Nl = p->nc * (p->N / p->ncls);
  p->w.assign(d->w, d->w + d->s);
  p->s_star = 0;
  for (int j = 0; j < d->s; ++j)
    if (d->w[j] < d->m) p->s_star = j + 1;

  if (d->kind == RQMC_REDUCED_MC) {
    // i.i.d. draws per coordinate: no generating vector, matrices or shifts
    if (d->shift || d->dshift) { delete p; return bad(RQMC_ESHIFT, "reduced MC takes no shift (its draws are random)"); }
    p->seed = d->seed;
  } else if (d->kind == RQMC_LATTICE) {
    if (!d->z) { delete p; return bad(RQMC_EINVAL, "z is NULL"); }
    p->z.assign(d->z, d->z + d->s);
    for (int j = 0; j < d->s; ++j) {
      const int wj = std::min<int>(d->w[j], d->m);
      const int64_t Mj = ipow(d->b, d->m - wj);
      const uint64_t zj = d->z[j];
      const bool ok = (Mj == 1) ? (zj == 1) : (zj >= 1 && zj < (uint64_t)Mj && gcd64((int64_t)zj, d->b) == 1);
      if (!ok) {
        delete p;
        return bad(RQMC_EZUNIT, "z'_" + std::to_string(j + 1) + " = " + std::to_string(zj) +
                                    " not in U_{b^{m-w_j}} (P:287-292)");
      }
    }
    if (d->shift) {
      p->shifted = true;
      p->shift.assign(d->shift, d->shift + d->s);
      for (int j = 0; j < d->s; ++j)
        if (!(d->shift[j] >= 0.0 && d->shift[j] < 1.0)) {
          delete p;
          return bad(RQMC_ESHIFT, "shift_" + std::to_string(j + 1) + " outside [0,1)");
        }
    }
  } else {
    if (!d->C) { delete p; return bad(RQMC_EINVAL, "C is NULL"); }
    p->C.assign(d->C, d->C + (size_t)d->s * d->m);
    for (int j = 0; j < d->s; ++j) {
      const int wj = std::min<int>(d->w[j], d->m);
      const uint64_t low = wj >= 64 ? ~0ull : ((1ull << wj) - 1);  // rows p > m - w_j <-> bits < w_j
      for (int q = 0; q < d->m; ++q) {
        uint64_t& col = p->C[(size_t)j * d->m + q];
        if (col >> d->m) {
          delete p;
          return bad(RQMC_ENETMAT, "column word j=" + std::to_string(j + 1) + " q=" + std::to_string(q) + " >= 2^m");
        }
        col &= ~low;  // Eq. reduced_genmat_net2: zero the last min(w_j,m) rows
        if (!rowzero && q >= d->m - wj && col != 0) {
          delete p;
          return bad(RQMC_ENETMAT, "reduced net coordinate j=" + std::to_string(j + 1) +
                                       " depends on digit " + std::to_string(q) +
                                       " >= m - w_j: not periodic; Alg. 2 needs column deletion (P:671)");
        }
      }
    }
    if (d->dshift) {
      p->shifted = true;
      p->dshift.assign(d->dshift, d->dshift + d->s);
      for (int j = 0; j < d->s; ++j)
        if (d->dshift[j] >> 53) {
          delete p;
          return bad(RQMC_ESHIFT, "digital shift_" + std::to_string(j + 1) + " >= 2^53");
        }
    }
  }

  // ---- level table (coarse -> fine) ----
  {
    std::vector<Level> fine_to_coarse;
    int j = 0;
    // row-zeroed nets: coordinate j takes 2^{m-w_j} values but with no common period in k
    // (P:667-669), so every j <= s* sits in one dense level of N rows (w = 0)
    auto level_of = [&](int jj) {
      const int wl = std::min<int>(d->w[jj], d->m);
      return rowzero ? (wl < d->m ? 0 : d->m) : wl;
    };
    while (j < d->s) {
      const int wl = level_of(j);
      int j2 = j;
      while (j2 < d->s && level_of(j2) == wl) ++j2;
      // columns j > s* are x = 0: dropped, unless a shift or the map makes them the
      // constant phi_j(Delta_j) / Phi^-1(zero rule) -- then a 1-row level m (reading C-4); the tent
      // map keeps 0 at 0 (phi(0) = 0), so unshifted tent columns are dropped like unit-map ones
      // (reduced MC: N_j = 1 for w_j >= m -- one i.i.d. draw per coordinate, P:981 N_{s+1} = 1)
      if (wl < d->m || p->shifted || d->map == RQMC_MAP_INVNORM || d->kind == RQMC_REDUCED_MC) {
        Level L{};
        L.w = wl; L.j_lo = j; L.s_w = j2 - j; L.fft_tab = -1;
        L.M = ipow(d->b, d->m - wl);
        L.Ml = L.M >= p->ncls ? p->nc * (L.M / p->ncls) : p->nc;
        fine_to_coarse.push_back(L);
      }
      j = j2;
    }
    p->lv.assign(fine_to_coarse.rbegin(), fine_to_coarse.rend());
    for (size_t i = 0; i < p->lv.size(); ++i) p->lv[i].parent = (int)i - 1;
    p->wlev.assign(d->s, d->m);
    for (const Level& L : p->lv)
      for (int q = 0; q < L.s_w; ++q) p->wlev[L.j_lo + q] = L.w;
  }
  const int nl = (int)p->lv.size();

  // ---- FFT-eligible levels (NEXT-4, valid without per-coordinate shifts)
  if (p->kind == RQMC_LATTICE && p->b == 2 && !p->shifted && p->ncls == 1) {
    for (int i = 0; i < nl; ++i) {
      Level& V = p->lv[i];
      const int k = p->m - V.w;
      if (k < kFftMinK || k > kFftMaxK) continue;
      FftTab t;
      t.k = k;
      std::vector<std::pair<uint64_t, int>> order;   // (sigma- flag << 32 | key, j)
      for (int q = 0; q < V.s_w; ++q) {
        const uint64_t zj = p->z[V.j_lo + q] & ((1ull << k) - 1);
        const bool minus = (zj & 3u) == 3u;
        const uint64_t z1 = minus ? (((1ull << k) - zj) & ((1ull << k) - 1)) : zj;   // = 1 (mod 4)
        const uint32_t e = dlog5(z1, k);
        uint32_t key = 0;
        for (int b = 0; b < k - 2; ++b) key |= ((e >> b) & 1u) << (k - 3 - b);
        order.push_back({((uint64_t)minus << 32) | key, q});
        if (!minus) ++t.nplus;
      }
      std::stable_sort(order.begin(), order.end(),
                       [](const auto& x, const auto& y) { return x.first < y.first; });
      for (auto& o : order) { t.jsort.push_back(o.second); t.key.push_back((uint32_t)o.first); }
      // bucket e (mod 2^p) of valuation v = keys [rho << v, (rho + 1) << v), rho = bitrev_p(e)
      for (int v = 0; v <= k - 3; ++v) {
        const int L = 1 << (k - 2 - v);
        t.boff_v.push_back((int)t.boff.size());
        for (int sg = 0; sg < 2; ++sg) {
          const auto b = t.key.begin() + (sg ? t.nplus : 0), e = t.key.begin() + (sg ? V.s_w : t.nplus);
          for (int rho = 0; rho <= L; ++rho)
            t.boff.push_back((int)(std::lower_bound(b, e, (uint32_t)rho << v) - t.key.begin()));
        }
      }
      V.fft_tab = (int)p->fft.size();
      p->fft.push_back(std::move(t));
    }
    for (auto& t : p->fft) {
      t.dev_j = p->fft_host.size();
      p->fft_host.insert(p->fft_host.end(), t.jsort.begin(), t.jsort.end());
      t.dev_k = p->fft_host.size();
      p->fft_host.insert(p->fft_host.end(), t.boff.begin(), t.boff.end());
    }
  }

  // ---- checkpoint and workspace layout of single runs ----
  {
    const int c = choose_ckpt(*p, 1);
    if (c < 0) { delete p; return bad(RQMC_EUNSUPPORTED, "no feasible checkpoint level"); }
    make_layout(*p, c, p->L1);
  }
  make_chunks(p);
  *out = p;
  return RQMC_OK;
}

void rqmc_plan_destroy(rqmc_plan_t p) {
  if (!p) return;
  for (auto e : p->prof_ev) cudaEventDestroy(e);
  for (auto e : p->h2d_ev)
    if (e) cudaEventDestroy(e);
  if (p->h2d_stream) cudaStreamDestroy(p->h2d_stream);
  for (auto e : p->h2d_lv_ev)
    if (e) cudaEventDestroy(e);
  for (auto& hg : p->host_graphs) cudaGraphExecDestroy(hg.exec);
  if (p->h_fsum_pin) cudaFreeHost(p->h_fsum_pin);
  for (auto& ge : p->graphs) cudaGraphExecDestroy(ge.exec);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->d_z) cudaFree(p->d_z);
  if (p->d_shift) cudaFree(p->d_shift);
  if (p->d_C) cudaFree(p->d_C);
  if (p->d_ds) cudaFree(p->d_ds);
  if (p->d_fft) cudaFree(p->d_fft);
  if (p->d_wl) cudaFree(p->d_wl);
  for (auto e : p->chunk_ev) cudaEventDestroy(e);
  if (p->side) cudaStreamDestroy(p->side);
  delete p;
}

rqmc_status rqmc_plan_summary_get(rqmc_plan_t p, rqmc_plan_summary* o) {
  if (!p || !o) return RQMC_EINVAL;
  o->n_levels = (int)p->lv.size();
  o->checkpoint = p->L1.ckpt;
  o->n_fine = p->L1.nfine;
  o->n_bundles = p->L1.nbundles;
  o->N_local = p->Nl;
  o->s_star = p->s_star;
  return RQMC_OK;
}

rqmc_status rqmc_plan_summary_batch(rqmc_plan_t p, int R, int f, rqmc_plan_summary* o) {
  if (!p || !o || R < 1) return RQMC_EINVAL;
  if (rqmc_status s = rqmc_plan_summary_get(p, o)) return s;
  const Layout& L = layout_for(p, R, f);
  o->checkpoint = L.ckpt;
  o->n_fine = L.nfine;
  o->n_bundles = L.nbundles;
  return RQMC_OK;
}

rqmc_status rqmc_plan_level(rqmc_plan_t p, int idx, rqmc_level_info* o) {
  if (!p || !o || idx < 0 || idx >= (int)p->lv.size()) return RQMC_EINVAL;
  const Level& L = p->lv[idx];
  o->w = L.w; o->j_lo = L.j_lo; o->s_w = L.s_w; o->M = L.M; o->M_local = L.Ml;
  o->parent = L.parent; o->coarse = p->L1.lv[idx].coarse; o->fft = p->L1.lv[idx].fft;
  o->absorbed = p->L1.lv[idx].absorbed;
  return RQMC_OK;
}

int64_t rqmc_plan_global_row(rqmc_plan_t p, int64_t i) {
  if (!p || i < 0 || i >= p->Nl) return -1;
  return p->c0 + i % p->nc + p->ncls * (i / p->nc);
}

rqmc_status rqmc_plan_partition(rqmc_plan_t p, int64_t* classes, int64_t* first, int64_t* count) {
  if (!p) return RQMC_EINVAL;
  if (classes) *classes = p->ncls;
  if (first) *first = p->c0;
  if (count) *count = p->nc;
  return RQMC_OK;
}

rqmc_status rqmc_plan_stats(rqmc_plan_t p, int want_y, int64_t* rows, double* macs, double* bytes) {
  if (!p) return RQMC_EINVAL;
  double mac = 0.0;
  for (auto& L : p->lv) mac += (double)L.Ml * L.s_w * p->tau;  // tau sum_w M_w s_w
  if (rows) *rows = p->Nl;
  if (macs) *macs = mac;
  if (bytes) *bytes = 8.0 * p->s * p->tau + (want_y ? 8.0 * p->Nl * p->tau : 0.0);
  return RQMC_OK;
}

rqmc_status rqmc_workspace_size(rqmc_plan_t p, size_t* bytes) {
  if (!p || !bytes) return RQMC_EINVAL;
  *bytes = std::max(p->L1.total, p->chunk_total);
  return RQMC_OK;
}

}  // extern "C"

namespace {

rqmc_status upload(rqmc_plan_s* p) {
  std::call_once(p->up_once, [p]() {
    auto cp = [&](auto& dst, const auto& src) {
      if (src.empty() || p->up_err != cudaSuccess) return;
      const size_t n = src.size() * sizeof(src[0]);
      p->up_err = cudaMalloc((void**)&dst, n);
      if (p->up_err == cudaSuccess) p->up_err = cudaMemcpy(dst, src.data(), n, cudaMemcpyHostToDevice);
    };
#if RQMC_DEBUG
    // the bounds checks spill the largest trees to a ~1.3 KB stack frame (above the 1 KB default)
    if (p->up_err == cudaSuccess) p->up_err = cudaDeviceSetLimit(cudaLimitStackSize, 4096);
#endif
    cp(p->d_z, p->z);
    cp(p->d_shift, p->shift);
    cp(p->d_C, p->C);
    cp(p->d_ds, p->dshift);
    cp(p->d_fft, p->fft_host);
    cp(p->d_wl, p->wlev);
  });
  if (p->up_err != cudaSuccess)
    return fail(p, RQMC_ECUDA, std::string("device table upload: ") + cudaGetErrorString(p->up_err));
  for (auto& q : p->chunks)
    if (rqmc_status s = upload(q.get())) return fail(p, s, q->err);
  return RQMC_OK;
}

GenArgs gen_args(const rqmc_plan_s* p, const Layout& lay, void* work) {
  GenArgs g{};
  g.kind = p->kind; g.map = p->map; g.b = p->b; g.m = p->m; g.shifted = p->shifted;
  g.ncls = p->ncls; g.c0 = p->c0; g.nc = p->nc; g.nlev = (int)p->lv.size();
  g.zero_u = p->shifted ? std::ldexp(1.0, -53) : 0.5 / (double)p->N;
  g.seed = p->seed;
  g.z = p->d_z; g.shift = p->d_shift; g.C = p->d_C; g.dshift = p->d_ds; g.wcl = p->d_wl;
  g.X = reinterpret_cast<double*>(static_cast<char*>(work) + lay.off_x);
  for (size_t i = 0; i < lay.lv.size(); ++i) {
    const Level& L = lay.lv[i];
    int tcl = 0;
    while (tcl < 5 && (1 << tcl) < L.ldx) ++tcl;
    const bool own = lay.gather || !L.absorbed;   // gather: every merged level generates its own X^red
    g.lv[i] = GenLevel{L.M, (L.fft || !own) ? 0 : L.Ml, L.xoff, L.j_lo, lay.gather ? L.s_w : L.s_gemm, L.ldx, tcl,
                       std::ldexp(1.0, -(p->m - L.w)),
                       (!lay.gather && L.coarse && i == (size_t)lay.absorb && lay.absorb > 0) ? 1 : 0};
  }
  return g;
}

rqmc_status check_cuda(rqmc_plan_s* p, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RQMC_OK;
  return fail(p, RQMC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Arguments of one FFT level (NEXT-4) on workspace w.
FftArgs fft_args(const rqmc_plan_s* p, const Layout& lay, const Level& L, char* w, const double* dA, int64_t lda,
                 const double* Rp, int64_t ldp, int64_t Mp, double* R) {
  const FftTab& t = p->fft[L.fft_tab];
  FftArgs a{};
  a.k = t.k; a.nv = t.k - 2; a.s_w = L.s_w; a.ncol = p->tau; a.ldz = lay.ldr; a.map = p->map;
  a.zero_u = 0.5 / (double)p->N; a.inv_M = std::ldexp(1.0, -t.k);
  a.A = dA + (int64_t)L.j_lo * lda; a.lda = lda;
  a.jsort = p->d_fft + t.dev_j; a.boff = p->d_fft + t.dev_k;
  a.z = p->d_z + L.j_lo;
  a.Z = reinterpret_cast<double2*>(w + lay.off_fz); a.H = reinterpret_cast<double2*>(w + lay.off_fh);
  a.Rp = Rp; a.ldp = ldp; a.Mp = Mp;
  a.R = R; a.ldr = lay.ldr;
  int64_t zo = 0;
  for (int v = 0; v < a.nv; ++v) {
    FftV& V = a.v[v];
    V.p = t.k - 2 - v;
    V.L = 1 << V.p;
    V.lgL1 = V.p <= 8 ? V.p : (V.p + 1) / 2;   // L <= 256: one CTA (L2 = 1); else balanced L1 L2
    V.lgL2 = V.p - V.lgL1;
    V.L1 = 1 << V.lgL1; V.L2 = 1 << V.lgL2;
    V.boff = t.boff_v[v];
    V.hoff = zo;
    V.zoff = zo * lay.ldr;
    zo += V.L;
  }
  return a;
}

// Arguments of the fused fine kernel for layout `lay` on workspace w (X: X^red base of the slice).
FineArgs fine_args(const rqmc_plan_s* p, const Layout& lay, char* w, double* X, const double* dA, int64_t lda,
                   double* dY, int64_t ldy, int fk, const double* fparam, int64_t rep_d) {
  FineArgs fa{};
  const Level& R = lay.lv[lay.ckpt];
  fa.root = reinterpret_cast<const double*>(w + lay.off_r[R.rbuf]); fa.ldroot = lay.ldr; fa.Mroot = R.Ml;
  fa.NF = lay.nfine;
  for (int i = 0; i < lay.nfine; ++i) {
    const Level& L = lay.lv[lay.ckpt + 1 + i];
    FineLevel& F = fa.lv[i];
    F.X = X + L.xoff; F.ldx = L.ldx; F.K = L.s_w; F.j_lo = L.j_lo;
    F.runs = (int)(L.Ml / R.Ml);
    F.fan = i == 0 ? F.runs : F.runs / fa.lv[i - 1].runs;
    F.xs_off = lay.fine_xs_off[i]; F.as_off = lay.fine_as_off[i];
  }
  fa.A = dA; fa.lda = lda; fa.tau = p->tau;
  fa.a_vec = ((uintptr_t)dA % 16 == 0) && (lda % 2 == 0) && (p->tau % 2 == 0);
  fa.Y = dY; fa.ldy = ldy;
  fa.y_vec = ((uintptr_t)dY % 16 == 0) && (ldy % 2 == 0);
  fa.fk = fk;
  fa.fp0 = fparam ? fparam[0] : 0.0;
  fa.fp1 = fparam ? fparam[1] : 0.0;
  fa.partial = reinterpret_cast<double*>(w + lay.off_part);
  fa.leafruns = lay.leafruns;
  fa.as_stride = lay.fine_as_stride;
  fa.root_off = 2 * lay.fine_as_stride;
  fa.acc_off = lay.fine_acc_off;
  fa.smem_bytes = lay.fine_smem;
  fa.xrep = rep_d; fa.rootrep = rep_d; fa.partrep = rep_d;
  if (lay.split_cap) {
    fa.rscr = reinterpret_cast<double*>(w + lay.off_split); fa.rscr_cap = lay.split_cap;
    fa.rcnt = reinterpret_cast<unsigned int*>(w + lay.off_cnt); fa.ncnt = kSplitSlots;
  }
  return fa;
}

// One pass of the hot path for nrep replicas (batched randomisation) whose workspace slices of
// rep_bytes each start at `base`: replica r uses shift[r*srep + j] / dshift[...] / seeds[r].
// nrep = 1 with the plan's own tables is the plain run.
struct RunRand {
  const double* shift;
  const uint64_t* dshift;
  const uint64_t* seeds;
  int srep;
};

// A residue chunk of a chunked rqmc_xa: the fine kernel and its reduction run on fine_st after the
// chunk's coarse levels (event ev), storing the chunk's rows of the caller's Y (row map).
struct ChunkCtx {
  cudaStream_t fine_st;
  cudaEvent_t ev;
  int64_t ym_c0, ym_ncls;
  int ym_nc;
};

rqmc_status run_core(rqmc_plan_s* p, const Layout& lay, int nrep, char* w, size_t rep_bytes, const RunRand& rr,
                     const cudaEvent_t* a_ready /* nullable: A arrives on another stream; [i] before coarse
                                                   level i reads its rows, [nl] before the fine levels */,
                     const double* dA,
                     int64_t lda, double* dY, int64_t ldy, rqmc_f f, const double* fparam, double* d_fsum,
                     cudaStream_t st, const ChunkCtx* cx = nullptr) {
  const bool want_f = f != RQMC_F_NONE && d_fsum;
#if RQMC_DEBUG
  if (!cx) {  // debug build: the buffers this run may touch (workspace slices, A, Y, f-sums, plan tables)
    DbgRanges dr{};
    auto set = [&](int i, const void* p, size_t n) {
      dr.lo[i] = static_cast<const char*>(p); dr.hi[i] = p ? static_cast<const char*>(p) + n : nullptr;
    };
    set(0, w, (size_t)nrep * rep_bytes + lay.total);   // slices + shift table (superset)
    set(1, dA, (size_t)p->s * lda * sizeof(double));
    set(2, dY, dY ? (size_t)p->Nl * ldy * sizeof(double) : 0);
    set(3, d_fsum, d_fsum ? (size_t)nrep * sizeof(double) : 0);
    set(4, p->d_fft, p->fft_host.size() * sizeof(int));
    set(5, p->d_z, p->z.size() * sizeof(uint64_t));
    for (auto fn : {dbg_set_gen, dbg_set_gemm, dbg_set_fine, dbg_set_tree, dbg_set_fft})
      if (rqmc_status s = check_cuda(p, fn(dr, st), "debug ranges")) return s;
  }
#endif
  cudaEvent_t* ev = nullptr;
  if (p->prof_runs < p->prof_max) ev = &p->prof_ev[5 * p->prof_runs++];
  auto mark = [&](int i) { if (ev) cudaEventRecord(ev[i], st); };
  const int64_t rep_d = (int64_t)(rep_bytes / sizeof(double));
  mark(0);
  NvtxRange r_run("rqmc:run");
  NvtxPhase phase;
  phase.next("rqmc:a2 points (k_gen)");

  // a2: reduced points of every level (all replicas: grid.z)
  GenArgs g = gen_args(p, lay, w);
  // k_gen zeroes the fine kernel's split and arrival counters (stream order, every call)
  g.zcnt = reinterpret_cast<unsigned int*>(w + lay.off_cnt); g.nzcnt = kSplitSlots + 1;
  g.shift = rr.shift; g.dshift = rr.dshift; g.seeds = rr.seeds; g.srep = rr.srep; g.xrep = rep_d;
  if (rqmc_status s = check_cuda(p, launch_gen(g, lay.max_gen_entries, nrep, st), "k_gen")) return s;
  mark(1);
  phase.next("rqmc:a3+a4 coarse levels (k_level_gemm / k_fft)");

  // a3+a4 coarse levels: R_w = tile(R_w') + X_w A_w, coarse -> fine.  A fused pair (Layout) runs as
  // one launch whose parent R never leaves the chip (bit-identical to two launches).
  for (int i = 0; i <= lay.ckpt; ++i) {
    const Level& L = lay.lv[i];
    if (L.absorbed) continue;    // merged into level lay.absorb's GEMM
    if (a_ready && a_ready[i])   // this level's rows of A have landed
      if (rqmc_status s = check_cuda(p, cudaStreamWaitEvent(st, a_ready[i], 0), "wait for A")) return s;
    GemmArgs a{};
    a.X = g.X + L.xoff; a.ldx = L.ldx; a.M = L.Ml; a.K = L.s_gemm;
    a.A = dA + (int64_t)L.j_lo * lda; a.lda = lda; a.tau = p->tau;
    if (L.parent >= 0) {
      const Level& P = lay.lv[L.parent];
      a.Rp = reinterpret_cast<const double*>(w + lay.off_r[P.rbuf]); a.ldp = lay.ldr; a.Mp = P.Ml;
    }
    a.ldr = lay.ldr;
    a.xrep = rep_d; a.rrep = rep_d;
    if (lay.gather && i == lay.absorb) {   // merged levels absorb, absorb-1, ..., 0 in increasing j
      int q = 0;
      for (int t = i; t >= 0; --t) {
        const Level& S = lay.lv[t];
        a.segq[a.nseg] = q; a.segX[a.nseg] = g.X + S.xoff; a.segld[a.nseg] = S.ldx; a.segM[a.nseg] = S.Ml;
        ++a.nseg;
        q += S.s_w;
      }
      a.segq[a.nseg] = q;
    }
    if (L.fft) {   // NEXT-4: the level's product by FFTs over the unit group (rqmc_fft.cu); nrep == 1
      const FftArgs fa = fft_args(p, lay, L, w, dA, lda, a.Rp, a.ldp, a.Mp,
                                  reinterpret_cast<double*>(w + lay.off_r[L.rbuf]));
      if (rqmc_status s = check_cuda(p, launch_fft_level(fa, st), "k_fft")) return s;
      continue;
    }
    if (L.fused) {
      const Level& Cl = lay.lv[i + 1];
      a.Xc = g.X + Cl.xoff; a.ldxc = Cl.ldx; a.Kc = Cl.s_w; a.Ac = dA + (int64_t)Cl.j_lo * lda;
      a.Rc = reinterpret_cast<double*>(w + lay.off_r[Cl.rbuf]); a.ncu = (int)(Cl.Ml / L.Ml);
      if (rqmc_status s = check_cuda(p, launch_gemm(a, nrep, st), "k_level_gemm (pair)")) return s;
      ++i;   // level i + 1 done in the same launch
      continue;
    }
    a.R = reinterpret_cast<double*>(w + lay.off_r[L.rbuf]);
    if (rqmc_status s = check_cuda(p, launch_gemm(a, nrep, st), "k_level_gemm")) return s;
  }

  mark(2);
  phase.next("rqmc:a3-a5 fused fine levels + f (k_fine, k_reduce)");

  // a3+a4+a5 fine levels fused with f / Y store
  if (a_ready && a_ready[lay.lv.size()])
    if (rqmc_status s = check_cuda(p, cudaStreamWaitEvent(st, a_ready[lay.lv.size()], 0), "wait for A")) return s;
  FineArgs fa = fine_args(p, lay, w, g.X, dA, lda, dY, ldy, want_f ? (int)f : -1, fparam, rep_d);
  if (cx) {   // chunk: continue on the fine stream once the coarse levels are done
    fa.ym_c0 = cx->ym_c0; fa.ym_ncls = cx->ym_ncls; fa.ym_nc = cx->ym_nc;
    cudaError_t e = cudaEventRecord(cx->ev, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cx->fine_st, cx->ev, 0);
    if (rqmc_status s = check_cuda(p, e, "chunk fork")) return s;
    st = cx->fine_st;
  }
  // a5's final fixed-order reduction runs in the fine kernel's last CTA (finish_fsum; k_fine and the
  // trees with <= 4 fused levels) -- one launch fewer
  if (want_f) {
    fa.fsum = d_fsum;
    fa.rcnt = reinterpret_cast<unsigned int*>(w + lay.off_cnt);   // [kSplitSlots] = the arrival counter
  }
  int64_t nparts = 0;
  if (rqmc_status s = check_cuda(p, launch_fine(fa, lay.nbundles, nrep, st, &nparts), "k_fine")) return s;
  mark(3);
  if (want_f && nparts > 0)   // the large trees leave the fixed-order sum of their partials to k_reduce
    if (rqmc_status s = check_cuda(p, launch_reduce(fa.partial, nparts, rep_d, nrep, d_fsum, st), "k_reduce"))
      return s;
  mark(4);
  return RQMC_OK;
}

// Chunked rqmc_xa (make_chunks): chunk i's points and coarse levels on st, its fine kernel (and f
// partial reduction into the chunk sums) on the plan's side stream after them; the side stream joins
// st at the end, and one fixed-order reduction adds the chunk sums.
rqmc_status run_chunked(rqmc_plan_s* p, const double* dA, int64_t lda, double* dY, int64_t ldy, rqmc_f f,
                        const double* fparam, double* d_fsum, char* w, cudaStream_t st) {
  const int n = (int)p->chunks.size();
  cudaError_t e = cudaSuccess;
  if (!p->side) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, lo);   // lowest: coarse GEMMs first
    p->chunk_ev.resize(n + 1);
    for (int i = 0; i <= n && e == cudaSuccess; ++i)
      e = cudaEventCreateWithFlags(&p->chunk_ev[i], cudaEventDisableTiming);
    if (rqmc_status s = check_cuda(p, e, "chunk streams")) return s;
  }
  const bool want_f = f != RQMC_F_NONE && d_fsum;
  double* sums = reinterpret_cast<double*>(w + p->chunk_sums);
  for (int i = 0; i < n; ++i) {
    rqmc_plan_s* q = p->chunks[i].get();
    const ChunkCtx cx{p->side, p->chunk_ev[i], q->c0, q->ncls, q->nc};
    const RunRand rr{q->d_shift, q->d_ds, nullptr, 0};
    if (rqmc_status s = run_core(q, q->L1, 1, w + p->chunk_off[i], q->L1.off_fsum, rr, nullptr, dA, lda, dY, ldy, f,
                                 fparam, want_f ? sums + i : nullptr, st, &cx))
      return fail(p, s, q->err);
  }
  e = cudaEventRecord(p->chunk_ev[n], p->side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, p->chunk_ev[n], 0);
  if (rqmc_status s = check_cuda(p, e, "chunk join")) return s;
  if (want_f)
    if (rqmc_status s = check_cuda(p, launch_reduce(sums, n, 0, 1, d_fsum, st), "k_reduce (chunks)")) return s;
  return RQMC_OK;
}

rqmc_status check_f(rqmc_plan_s* p, rqmc_f f, const double* fparam) {
  if (f < RQMC_F_NONE || f > RQMC_F_MEAN) return fail(p, RQMC_EINVAL, "bad f");
  if (f == RQMC_F_CALL_MEAN_EXP && !fparam) return fail(p, RQMC_EINVAL, "f needs fparam");
  return RQMC_OK;
}

rqmc_status run(rqmc_plan_s* p, const double* dA, int64_t lda, double* dY, int64_t ldy, rqmc_f f,
                const double* fparam, double* d_fsum, void* dwork, size_t wbytes, cudaStream_t st) {
  if (!p || !dA || !dwork) return fail(p, RQMC_EINVAL, "null pointer");
  if (wbytes < p->L1.total) return fail(p, RQMC_EINVAL, "workspace too small: need " + std::to_string(p->L1.total));
  if (lda < p->tau || (dY && ldy < p->tau)) return fail(p, RQMC_EDIM, "lda/ldy < tau");
  if (rqmc_status s = check_f(p, f, fparam)) return s;
  const bool want_f = f != RQMC_F_NONE && d_fsum;
  if (!want_f && !dY) return RQMC_OK;
  if (rqmc_status s = upload(p)) return s;
  const RunRand rr{p->d_shift, p->d_ds, nullptr, 0};
  const bool chunked = dY != nullptr && !p->chunks.empty() && p->prof_max == 0;
  if (chunked && wbytes < p->chunk_total)
    return fail(p, RQMC_EINVAL, "workspace too small: need " + std::to_string(p->chunk_total));
  auto direct = [&] {
    if (chunked) return run_chunked(p, dA, lda, dY, ldy, f, fparam, d_fsum, static_cast<char*>(dwork), st);
    return run_core(p, p->L1, 1, static_cast<char*>(dwork), p->L1.off_fsum, rr, nullptr, dA, lda, dY, ldy, f, fparam,
                    d_fsum, st);
  };
  // The launch sequence of a run depends only on these arguments: capture it once as a CUDA graph and
  // replay it (one launch instead of ~9; ~60 us -> ~15 us on C1).  Not while phase profiling records
  // per-run events, nor with RQMC_NO_GRAPH=1.
  // (debug builds launch directly: their per-run range uploads are host copies)
  static const bool no_graph = RQMC_DEBUG || [] { const char* e = std::getenv("RQMC_NO_GRAPH"); return e && *e && *e != '0'; }();
  if (no_graph || p->prof_max > 0) return direct();
  const double fp0 = fparam ? fparam[0] : 0.0, fp1 = fparam ? fparam[1] : 0.0;
  const int fk = want_f ? (int)f : -1;
  std::lock_guard<std::mutex> lk(p->graph_mu);
  for (auto& ge : p->graphs)
    if (ge.dA == dA && ge.dY == dY && ge.d_fsum == (want_f ? d_fsum : nullptr) && ge.dwork == dwork && ge.lda == lda &&
        ge.ldy == ldy && ge.f == fk && ge.fp0 == fp0 && ge.fp1 == fp1) {
      ge.last_use = ++p->graph_clock;
      return check_cuda(p, cudaGraphLaunch(ge.exec, st), "cudaGraphLaunch");
    }
  cudaError_t e = cudaSuccess;
  if (!p->cap_stream) e = cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return direct();
  // the capture stream starts after earlier work on st (the graph itself is launched on st)
  e = cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return direct();
  const rqmc_status s =
      chunked ? run_chunked(p, dA, lda, dY, ldy, f, fparam, d_fsum, static_cast<char*>(dwork), p->cap_stream)
              : run_core(p, p->L1, 1, static_cast<char*>(dwork), p->L1.off_fsum, rr, nullptr, dA, lda, dY, ldy, f,
                         fparam, d_fsum, p->cap_stream);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(p->cap_stream, &graph);
  cudaGraphExec_t exec = nullptr;
  if (s == RQMC_OK && e == cudaSuccess && graph) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (s != RQMC_OK || e != cudaSuccess || !exec) {
    cudaGetLastError();  // clear a capture error; run directly
    return direct();
  }
  if (p->graphs.size() >= 8) {  // evict the least recently used
    auto it = std::min_element(p->graphs.begin(), p->graphs.end(),
                               [](const auto& x, const auto& y) { return x.last_use < y.last_use; });
    cudaGraphExecDestroy(it->exec);
    p->graphs.erase(it);
  }
  p->graphs.push_back({dA, dY, want_f ? d_fsum : nullptr, dwork, lda, ldy, fk, fp0, fp1, exec, ++p->graph_clock});
  return check_cuda(p, cudaGraphLaunch(exec, st), "cudaGraphLaunch");
}

// bytes of one replica's workspace slice [X^red][R0][R1][partials] and of a chunk of n replicas
size_t rep_slice_bytes(const Layout& lay) { return lay.off_fsum; }
size_t batch_bytes(const rqmc_plan_s* p, const Layout& lay, int64_t n) {
  const size_t tab = (p->kind == RQMC_REDUCED_MC ? 1 : (size_t)p->s) * sizeof(double);
  return (size_t)n * rep_slice_bytes(lay) + align_up((size_t)n * tab, 256);
}

}  // namespace

extern "C" {

rqmc_status rqmc_xa(rqmc_plan_t p, const double* dA, int64_t lda, double* dY, int64_t ldy, rqmc_f f,
                    const double* fparam, double* d_fsum, void* dwork, size_t wbytes, void* stream) {
  return run(p, dA, lda, dY, ldy, f, fparam, d_fsum, dwork, wbytes, static_cast<cudaStream_t>(stream));
}

rqmc_status rqmc_qn(rqmc_plan_t p, const double* dA, int64_t lda, rqmc_f f, const double* fparam,
                    double* d_fsum, void* dwork, size_t wbytes, void* stream) {
  if (!d_fsum || f == RQMC_F_NONE) return fail(p, RQMC_EINVAL, "rqmc_qn needs f and d_fsum");
  return run(p, dA, lda, nullptr, 0, f, fparam, d_fsum, dwork, wbytes, static_cast<cudaStream_t>(stream));
}

// H2D of A in the order the run reads it -- each coarse level's rows (coarse -> fine), then the fine
// levels' rows -- on the copy stream, one event per piece: the first GEMM waits for its own rows only,
// the later copies overlap the GEMMs before them (C3: the 8 MB of A took 0.26 ms before the first GEMM).
static cudaError_t issue_h2d(rqmc_plan_s* p, const double* hA, int64_t lda, double* dA, cudaStream_t st) {
  const Layout& L = p->L1;
  const size_t nl = L.lv.size();
  cudaError_t e = cudaEventRecord(p->h2d_ev[0], st);   // after earlier work on st: A's buffer is free
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->h2d_stream, p->h2d_ev[0], 0);
  int jmin = p->s;
  // Small A (C1 8 KB, C2 512 KB) goes in one copy: each piece costs a copy's fixed latency, more than
  // the overlap gains (e2e C1 86 -> 59 us, C2 139 -> 132 us; C3 / C4 keep the pieces: 1.09 -> 1.01 ms,
  // 5.72 -> 5.30 ms; profiles/r02f_h2d_pieces_ab.txt).  RQMC_H2D_ONE=0/1 forces either form.
  static const int one_env = [] { const char* v = std::getenv("RQMC_H2D_ONE"); return v && *v ? (*v != '0') : -1; }();
  const bool one_piece = one_env >= 0 ? one_env == 1 : (double)p->s * p->tau * sizeof(double) < 2.0 * (1 << 20);
  if (one_piece) {   // all of A in one copy, every level waits for it
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(dA, (size_t)L.ldr * sizeof(double), hA, (size_t)lda * sizeof(double),
                            (size_t)p->tau * sizeof(double), (size_t)p->s, cudaMemcpyHostToDevice, p->h2d_stream);
    for (size_t i = 0; i <= nl && e == cudaSuccess; ++i) e = cudaEventRecord(p->h2d_lv_ev[i], p->h2d_stream);
    return e;
  }
  auto copy = [&](int j0, int nj, cudaEvent_t ev) {
    if (e != cudaSuccess) return;
    if (nj > 0 && lda == L.ldr)   // equal pitches: one linear copy
      e = cudaMemcpyAsync(dA + (int64_t)j0 * L.ldr, hA + (int64_t)j0 * lda, (size_t)nj * lda * sizeof(double),
                          cudaMemcpyHostToDevice, p->h2d_stream);
    else if (nj > 0)
      e = cudaMemcpy2DAsync(dA + (int64_t)j0 * L.ldr, (size_t)L.ldr * sizeof(double), hA + (int64_t)j0 * lda,
                            (size_t)lda * sizeof(double), (size_t)p->tau * sizeof(double), (size_t)nj,
                            cudaMemcpyHostToDevice, p->h2d_stream);
    if (e == cudaSuccess) e = cudaEventRecord(ev, p->h2d_stream);
  };
  for (size_t i = 0; i <= (size_t)L.ckpt && i < nl; ++i) {
    const Level& V = L.lv[i];
    if (V.absorbed) continue;
    const int nj = std::min(V.fft ? V.s_w : V.s_gemm, p->s - V.j_lo);
    copy(V.j_lo, nj, p->h2d_lv_ev[i]);
    jmin = std::min(jmin, V.j_lo);
  }
  copy(0, jmin, p->h2d_lv_ev[nl]);   // the fine levels' rows (j < the finest coarse level's first row)
  return e;
}

// Host-buffer runs (rqmc_qn_host, rqmc_xa_host): A from host memory (piecewise H2D on the copy stream,
// overlapped with the run), Y (xa only) into the caller's device buffer, the local f-sum back to host.
static rqmc_status run_host(rqmc_plan_s* p, const double* hA, int64_t lda, double* dY, int64_t ldy, rqmc_f f,
                            const double* fparam, double* h_fsum, void* dwork, size_t wbytes, void* stream) {
  if (wbytes < p->L1.total) return fail(p, RQMC_EINVAL, "workspace too small");
  if (lda < p->tau || (dY && ldy < p->tau)) return fail(p, RQMC_EDIM, "lda/ldy < tau");
  if (rqmc_status s = check_f(p, f, fparam)) return s;
  const bool want_f = f != RQMC_F_NONE;
  if (want_f && !h_fsum) return fail(p, RQMC_EINVAL, "f needs h_fsum");
  if (rqmc_status s = upload(p)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(dwork);
  double* dA = reinterpret_cast<double*>(w + p->L1.off_a);
  double* dsum = reinterpret_cast<double*>(w + p->L1.off_fsum);
  std::lock_guard<std::mutex> lk(p->h2d_mu);
  cudaError_t e = cudaSuccess;
  const size_t nl = p->L1.lv.size();
  if (!p->h2d_stream) {
    e = cudaStreamCreateWithFlags(&p->h2d_stream, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&p->h2d_ev[i], cudaEventDisableTiming);
    p->h2d_lv_ev.assign(nl + 1, nullptr);
    for (size_t i = 0; i <= nl && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&p->h2d_lv_ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocHost(&p->h_fsum_pin, sizeof(double));
    if (rqmc_status s = check_cuda(p, e, "copy stream")) return s;
  }
  const RunRand rr{p->d_shift, p->d_ds, nullptr, 0};
  auto sequence = [&](double* out_host) -> rqmc_status {
    if (rqmc_status s = check_cuda(p, issue_h2d(p, hA, lda, dA, st), "H2D A")) return s;
    if (rqmc_status s = run_core(p, p->L1, 1, w, p->L1.off_fsum, rr, p->h2d_lv_ev.data(), dA, p->L1.ldr, dY,
                                 ldy, f, fparam, want_f ? dsum : nullptr, st))
      return s;
    if (!want_f) {   // A's staging buffer is read until the run ends: join the copy stream into st
      cudaError_t ej = cudaEventRecord(p->h2d_ev[1], p->h2d_stream);
      if (ej == cudaSuccess) ej = cudaStreamWaitEvent(st, p->h2d_ev[1], 0);
      return check_cuda(p, ej, "copy stream join");
    }
    return check_cuda(p, cudaMemcpyAsync(out_host, dsum, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H fsum");
  };
  // Page-locked A (the bench's pinned buffer): the whole sequence -- the copy-stream fork, the piecewise
  // H2D, the kernels, the D2H into a pinned slot -- is captured once as a CUDA graph and replayed (the
  // small configs are dominated by ~10 launches from the host otherwise).  Pageable A runs directly.
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, hA) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  static const bool no_graph = RQMC_DEBUG || [] { const char* v = std::getenv("RQMC_NO_GRAPH"); return v && *v && *v != '0'; }();
  if (!pinned || no_graph || p->prof_max > 0) {
    if (rqmc_status s = sequence(h_fsum)) return s;
    return check_cuda(p, cudaStreamSynchronize(st), "host run");
  }
  const double fp0 = fparam ? fparam[0] : 0.0, fp1 = fparam ? fparam[1] : 0.0;
  cudaGraphExec_t exec = nullptr;
  for (auto& hg : p->host_graphs)
    if (hg.hA == hA && hg.dwork == dwork && hg.dY == dY && hg.lda == lda && hg.ldy == ldy && hg.f == (int)f &&
        hg.fp0 == fp0 && hg.fp1 == fp1)
      exec = hg.exec;
  if (!exec) {
    if (!p->cap_stream) e = cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (rqmc_status s = check_cuda(p, e, "capture")) return s;
    cudaStream_t keep = st;
    st = p->cap_stream;
    const rqmc_status s = sequence(p->h_fsum_pin);
    st = keep;
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(p->cap_stream, &graph);
    if (s == RQMC_OK && e == cudaSuccess && graph) e = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (s != RQMC_OK || e != cudaSuccess || !exec) {   // run directly
      cudaGetLastError();
      if (rqmc_status s2 = sequence(h_fsum)) return s2;
      return check_cuda(p, cudaStreamSynchronize(st), "host run");
    }
    if (p->host_graphs.size() >= 8) {
      cudaGraphExecDestroy(p->host_graphs.front().exec);
      p->host_graphs.erase(p->host_graphs.begin());
    }
    p->host_graphs.push_back({hA, dwork, dY, lda, ldy, (int)f, fp0, fp1, exec});
  }
  e = cudaGraphLaunch(exec, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (rqmc_status s = check_cuda(p, e, "host graph")) return s;
  if (want_f) *h_fsum = *p->h_fsum_pin;
  return RQMC_OK;
}

rqmc_status rqmc_qn_host(rqmc_plan_t p, const double* hA, int64_t lda, rqmc_f f, const double* fparam,
                         double* h_fsum, void* dwork, size_t wbytes, void* stream) {
  if (!p || !hA || !h_fsum || !dwork) return fail(p, RQMC_EINVAL, "null pointer");
  if (f == RQMC_F_NONE) return fail(p, RQMC_EINVAL, "rqmc_qn_host needs f");
  return run_host(p, hA, lda, nullptr, 0, f, fparam, h_fsum, dwork, wbytes, stream);
}

rqmc_status rqmc_xa_host(rqmc_plan_t p, const double* hA, int64_t lda, double* dY, int64_t ldy, rqmc_f f,
                         const double* fparam, double* h_fsum, void* dwork, size_t wbytes, void* stream) {
  if (!p || !hA || !dY || !dwork) return fail(p, RQMC_EINVAL, "null pointer");
  return run_host(p, hA, lda, dY, ldy, f, fparam, h_fsum, dwork, wbytes, stream);
}

rqmc_status rqmc_workspace_size_batch(rqmc_plan_t p, int R, size_t* bytes) {
  if (!p || !bytes || R < 1) return RQMC_EINVAL;
  // enough for either layout a batch of R may use (the choice depends on f)
  *bytes = std::max(batch_bytes(p, layout_for(p, R, RQMC_F_MEAN), R), batch_bytes(p, p->L1, R));
  return RQMC_OK;
}

rqmc_status rqmc_qn_batch(rqmc_plan_t p, int R, const double* hshifts, const uint64_t* hdshifts,
                          const uint64_t* hseeds, const double* dA, int64_t lda, rqmc_f f, const double* fparam,
                          double* d_fsum, void* dwork, size_t wbytes, void* stream) {
  if (!p || !dA || !dwork || !d_fsum || R < 1) return fail(p, RQMC_EINVAL, "null pointer or R < 1");
  if (f == RQMC_F_NONE) return fail(p, RQMC_EINVAL, "rqmc_qn_batch needs f");
  if (lda < p->tau) return fail(p, RQMC_EDIM, "lda < tau");
  if (rqmc_status s = check_f(p, f, fparam)) return s;
  const void* tab = nullptr;
  size_t per = (size_t)p->s * sizeof(double);
  if (p->kind == RQMC_LATTICE) {
    if (!hshifts || !p->shifted) return fail(p, RQMC_EINVAL, "lattice batch needs hshifts and a shifted plan");
    for (int64_t i = 0; i < (int64_t)R * p->s; ++i)
      if (!(hshifts[i] >= 0.0 && hshifts[i] < 1.0))
        return fail(p, RQMC_ESHIFT, "batch shift " + std::to_string(i / p->s) + "," + std::to_string(i % p->s) +
                                        " outside [0,1)");
    tab = hshifts;
  } else if (p->kind == RQMC_DIGITAL_NET) {
    if (!hdshifts || !p->shifted) return fail(p, RQMC_EINVAL, "net batch needs hdshifts and a shifted plan");
    for (int64_t i = 0; i < (int64_t)R * p->s; ++i)
      if (hdshifts[i] >> 53) return fail(p, RQMC_ESHIFT, "batch digital shift >= 2^53");
    tab = hdshifts;
  } else {
    if (!hseeds) return fail(p, RQMC_EINVAL, "reduced-MC batch needs hseeds");
    tab = hseeds;
    per = sizeof(uint64_t);
  }
  // layout for the replicas that run together; a smaller workspace means smaller chunks, which
  // may in turn want a finer checkpoint (re-evaluated until stable)
  // (chunks <= 65535 replicas: the replica count is a grid dimension of every kernel)
  const int64_t cmax = std::min<int64_t>(R, 65535);
  auto fit = [&](const Layout& L) {
    int64_t n = cmax;
    while (n > 0 && batch_bytes(p, L, n) > wbytes) --n;
    return n;
  };
  const Layout* lay = &layout_for(p, cmax, f);
  int64_t chunk = fit(*lay);
  for (int it = 0; it < 8 && chunk > 0; ++it) {
    const Layout* l2 = &layout_for(p, chunk, f);
    if (l2 == lay) break;
    lay = l2;
    chunk = fit(*lay);   // the chunk is always sized for the layout it runs with
  }
  if (chunk == 0) {
    lay = &p->L1;
    chunk = fit(*lay) > 0 ? 1 : 0;
  }
  if (chunk == 0) return fail(p, RQMC_EINVAL, "workspace too small for one replica: need " +
                                                  std::to_string(batch_bytes(p, p->L1, 1)));
  if (batch_bytes(p, *lay, chunk) > wbytes)
    return fail(p, RQMC_EINVAL, "internal: batch chunk exceeds the workspace");
  if (rqmc_status s = upload(p)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(dwork);
  for (int64_t r0 = 0; r0 < R; r0 += chunk) {
    const int n = (int)std::min<int64_t>(chunk, R - r0);
    char* dtab = w + (size_t)chunk * rep_slice_bytes(*lay);
    cudaError_t e = cudaMemcpyAsync(dtab, static_cast<const char*>(tab) + (size_t)r0 * per, (size_t)n * per,
                                    cudaMemcpyHostToDevice, st);
    if (rqmc_status s = check_cuda(p, e, "H2D batch shifts")) return s;
    RunRand rr{nullptr, nullptr, nullptr, p->s};
    if (p->kind == RQMC_LATTICE) rr.shift = reinterpret_cast<const double*>(dtab);
    else if (p->kind == RQMC_DIGITAL_NET) rr.dshift = reinterpret_cast<const uint64_t*>(dtab);
    else rr.seeds = reinterpret_cast<const uint64_t*>(dtab);
    if (rqmc_status s = run_core(p, *lay, n, w, rep_slice_bytes(*lay), rr, nullptr, dA, lda, nullptr, 0, f, fparam,
                                 d_fsum + r0, st))
      return s;
  }
  return RQMC_OK;
}

rqmc_status rqmc_plan_dispatch(rqmc_plan_t p, int R, int f, int want_y, char* buf, size_t len) {
  if (!p || !buf || len == 0 || R < 1) return RQMC_EINVAL;
  const Layout& lay = R == 1 ? p->L1 : layout_for(p, R, f);
  // placeholder addresses: 256-byte aligned, never dereferenced (only alignment and NULL-ness matter)
  char* w = reinterpret_cast<char*>(uintptr_t(1) << 20);
  double* X = reinterpret_cast<double*>(w + lay.off_x);
  const double* dA = reinterpret_cast<const double*>(w);
  double* dY = want_y ? reinterpret_cast<double*>(w) : nullptr;
  const int fk = f == RQMC_F_NONE ? -1 : f;
  const FineArgs fa = fine_args(p, lay, w, X, dA, p->tau + (p->tau & 1), dY, p->tau + (p->tau & 1), fk, nullptr,
                                (int64_t)(lay.off_fsum / sizeof(double)));
  describe_fine(fa, buf, len);
  return RQMC_OK;
}

rqmc_status rqmc_points(rqmc_plan_t p, int idx, int64_t r0, int64_t count, uint64_t* d_words, double* d_vals,
                        void* stream) {
  if (!p || idx < 0 || idx >= (int)p->lv.size() || r0 < 0 || count < 0 || r0 + count > p->lv[idx].Ml)
    return fail(p, RQMC_EINVAL, "bad level / row range");
  if (rqmc_status s = upload(p)) return s;
  // the plan's own levels (no merged coordinates, no workspace)
  GenArgs g = gen_args(p, p->L1, nullptr);
  for (size_t i = 0; i < p->lv.size(); ++i) {
    const Level& L = p->lv[i];
    g.lv[i] = GenLevel{L.M, L.Ml, 0, L.j_lo, L.s_w, L.s_w, 0, std::ldexp(1.0, -(p->m - L.w)), 0};
  }
  return check_cuda(p, launch_points(g, idx, r0, count, d_words, d_vals, static_cast<cudaStream_t>(stream)),
                    "k_points");
}

rqmc_status rqmc_profile_enable(rqmc_plan_t p, int max_runs) {
  if (!p || max_runs < 0) return RQMC_EINVAL;
  for (auto e : p->prof_ev) cudaEventDestroy(e);
  p->prof_ev.clear();
  p->prof_runs = 0;
  p->prof_max = 0;
  if (max_runs == 0) return RQMC_OK;
  p->prof_ev.resize((size_t)5 * max_runs);
  for (auto& e : p->prof_ev)
    if (cudaEventCreate(&e) != cudaSuccess) return fail(p, RQMC_ECUDA, "cudaEventCreate");
  p->prof_max = max_runs;
  return RQMC_OK;
}

rqmc_status rqmc_profile_read(rqmc_plan_t p, int* runs, double* ms_gen, double* ms_coarse, double* ms_fine,
                              double* ms_reduce) {
  if (!p) return RQMC_EINVAL;
  double acc[4] = {0, 0, 0, 0};
  for (int r = 0; r < p->prof_runs; ++r) {
    cudaEvent_t* ev = &p->prof_ev[5 * r];
    if (cudaEventSynchronize(ev[4]) != cudaSuccess) return fail(p, RQMC_ECUDA, "cudaEventSynchronize");
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev[i], ev[i + 1]) != cudaSuccess) return fail(p, RQMC_ECUDA, "elapsed");
      acc[i] += ms;
    }
  }
  if (runs) *runs = p->prof_runs;
  if (ms_gen) *ms_gen = acc[0];
  if (ms_coarse) *ms_coarse = acc[1];
  if (ms_fine) *ms_fine = acc[2];
  if (ms_reduce) *ms_reduce = acc[3];
  return RQMC_OK;
}

}  // extern "C"
