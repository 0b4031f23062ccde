/*
 * rqmc.h -- C ABI of the B200-native reduced QMC matrix product.
 *
 * Computes, for the N = b^m points x_k of a reduced rank-1 lattice or a column-reduced base-2
 * digital net (optionally randomly / digitally shifted and mapped to N(0,1)) and any dense s x tau
 * matrix A:
 *     Y = X A                      (X never materialised, only X^red per level)
 *     Q_N = N^-1 sum_k f(x_k^T A)
 * by the paper's Algorithm 2 with dense per-level products: the coordinates are grouped
 * into levels w = min(w_j, m) (tau_I), each level is one dense product
 * P_w = X^red_w (b^{m-w} x s_w) A_w (s_w x tau), and the rows are rebuilt by the periodic
 * tile-accumulate R_w[r] = P_w[r] + R_w'[r mod b^{m-w'}], Y = R_0.
 * P:n = /root/reference/PAPER.md line n;  S:n = SPEC.md line n.
 *
 * Conventions
 *  - All host arrays passed to rqmc_plan_create are COPIED; the caller keeps ownership.
 *  - Device buffers (A, Y, d_fsum, workspace) are owned by the caller (e.g. torch tensors).
 *  - fparam is a HOST pointer to 2 doubles (may be NULL when f does not use it).
 *  - stream is a cudaStream_t passed as void* (NULL = legacy default stream).  Run calls are
 *    asynchronous on it; device faults surface at the caller's next synchronisation.
 *  - Validation errors are returned synchronously; rqmc_plan_last_error() names the offending
 *    coordinate / level.  A plan is immutable after creation (device tables are uploaded on the
 *    first run call, thread-safely): concurrent runs on distinct streams with distinct outputs and
 *    workspaces are safe.
 *  - Layouts: A row-major s x tau, row j = a_j, leading dimension lda >= tau (elements).
 *    Y row-major N_local x tau, ldy >= tau.  Multi-GPU residue-class partition:
 *    the points are split into ncls classes k mod ncls and rank g owns the contiguous classes
 *    c0 .. c0+nc-1 (rqmc_plan_partition); local row i is global point
 *        k = c0 + (i mod nc) + ncls * (i div nc),      N_local = nc * N / ncls.
 *    world a power of b dividing N: ncls = world, c0 = rank, nc = 1 (k = rank + world * i), so every
 *    level with M_w >= world splits exactly.  Any other world (b = 3 on 2/4/8 GPUs, ...): ncls = b^gamma,
 *    the smallest power >= 32 world (gamma <= m), in groups of floor/ceil(ncls/world) classes (work
 *    imbalance <= 3 %).  Levels with fewer than ncls rows keep nc replicated rows per rank.
 *    world = 1 gives Y = XA.
 *  - Point kinds: RQMC_LATTICE, RQMC_DIGITAL_NET (b = 2), RQMC_REDUCED_MC and
 *    RQMC_DIGITAL_NET_ROWS (row-zeroed nets, Alg. 4) (see rqmc_kind).
 *  - Precision: fp64 throughout.  Point indices/digits are exact integers; lattice values are
 *    u = t/M (IEEE divide), shift u = u + Delta, if u >= 1 then u - 1 (no FMA contraction).
 *  - Limits: N = b^m <= 2^32; m <= 32 for nets; 1 <= world <= N.
 */
#ifndef RQMC_H
#define RQMC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rqmc_plan_s* rqmc_plan_t;

typedef enum {
  RQMC_OK = 0,
  RQMC_EINVAL = 1,       /* null pointer / bad size / bad enum / workspace too small       */
  RQMC_ENOTPRIME = 2,    /* b is not prime                                     */
  RQMC_EWORDER = 3,      /* w not nondecreasing or w_1 != 0                        */
  RQMC_EZUNIT = 4,       /* z'_j not in U_{b^{m-w_j}}                          */
  RQMC_ESHIFT = 5,       /* shift outside [0,1) or digital shift >= 2^53                   */
  RQMC_ENETMAT = 6,      /* net matrices: bad words, or reduced net not periodic    */
  RQMC_EDIM = 7,         /* dimension mismatch / lda < tau / ldy < tau                     */
  RQMC_EDOMAIN = 8,      /* Phi^-1 domain (never raised for valid plans: zero rule)        */
  RQMC_ECUDA = 9,        /* CUDA launch / copy failure, or no device                       */
  RQMC_ENOMEM = 10,      /* allocation failure                                             */
  RQMC_EUNSUPPORTED = 11 /* outside the supported envelope (N > 2^32, world, ...)          */
} rqmc_status;

/* RQMC_REDUCED_MC: reduced Monte Carlo (Sec. 5, Eq. randpts): coordinate j
 * draws only N_j = b^{m - min(w_j,m)} i.i.d. uniforms y_{j,0..N_j-1} and point n uses
 * x_{n,j} = y_{j, n mod N_j} (the truncated mixed-radix index of Eq. randpts equals n mod N_j).
 * The draws come from a counter-based generator (both the product path and the test oracle
 * implement it):  mix64(x) = SplitMix64 finaliser (x ^= x>>30; x *= 0xBF58476D1CE4E5B9;
 * x ^= x>>27; x *= 0x94D049BB133111EB; x ^= x>>31), G = 0x9E3779B97F4A7C15,
 *   key_j = mix64(seed * G + (j+1))      (j 0-based coordinate, wrapping uint64 arithmetic)
 *   word  = mix64(key_j + (r+1) * G) >> 11,  u = (word | 1) 2^-53   (exact, odd multiple of
 *   2^-53, so 0 < u < 1 and Phi^-1(u) is finite).
 * The same tree of levels, GEMMs and fused fine kernel computes the product. */
/* RQMC_DIGITAL_NET_ROWS: the paper's own reduced digital net (Alg. 3): any generating
 * matrices C^(j) (b = 2, same column-word format as RQMC_DIGITAL_NET), with the last min(w_j,m) rows
 * zeroed by the plan (Eq. reduced_genmat_net2) and no column-deletion requirement.  Coordinate j
 * then takes only 2^{m-w_j} distinct values, but their pattern in n differs per j, so no rows of
 * the product repeat: Alg. 4 saves multiplications, not additions.  On the
 * fp64 datapath an add and an FMA cost the same issue slot, so the plan computes the product as one
 * dense level of N rows and s* coordinates on the DMMA GEMM (N s* tau MACs = Alg. 4's additions).
 * Points, shifts (dshift), map, f and the multi-GPU partition are as for RQMC_DIGITAL_NET. */
typedef enum {
  RQMC_LATTICE = 0, RQMC_DIGITAL_NET = 1, RQMC_REDUCED_MC = 2, RQMC_DIGITAL_NET_ROWS = 3
} rqmc_kind;
/* Point map applied to every coordinate u in [0,1): identity; Phi^-1 (the Gaussian workloads,
 * P:59-67; u = 0 remapped, reading C-5); or the tent transformation phi(u) = 1 - |1 - 2u| (P:250-253:
 * "the random shift can be replaced by the tent transformation"; evaluated as written in fp64, 2u exact,
 * so GPU and oracle agree bit for bit).  The map commutes with the reduction: coordinate j still depends
 * on k mod M_j only. */
typedef enum { RQMC_MAP_UNIT = 0, RQMC_MAP_INVNORM = 1, RQMC_MAP_TENT = 2 } rqmc_map;

/* f(y) = F(tau^-1 sum_c g(y_c))  (SURVEY reading C-17)                                    */
typedef enum {
  RQMC_F_NONE = -1,
  RQMC_F_EXP_MEAN = 0,      /* exp(mean(y))                                  (C1, C3, C5)  */
  RQMC_F_CALL_MEAN_EXP = 1, /* max(mean(exp(p0 * y)) - p1, 0)                (C2)          *
                             * (the compile-time tree kernels evaluate exp(p0 y) by a table-driven
                             * fp64 exp (<= 2.6 ulp) with p0 y clamped to [-700, 700]: no overflow to
                             * inf / underflow to 0 beyond that; NaN propagates; the general kernel
                             * uses libdevice exp)                                               */
  RQMC_F_MEAN_SQ = 2,       /* mean(y^2)                                     (C4)          */
  RQMC_F_MEAN = 3           /* mean(y), linear                               (tests)       */
} rqmc_f;

typedef struct {
  int b, m, s, tau;         /* b prime, N = b^m, A is s x tau                                 */
  const int32_t* w;         /* s reduction indices, nondecreasing, w[0] == 0         */
  rqmc_kind kind;
  const uint64_t* z;        /* lattice: z'_j in U_{b^{m-w_j}}, s entries         */
  const uint64_t* C;        /* net (b=2): s*m column words; bit (m-1-p) of C[j*m+q] is
                               C^(j)_{p+1,q+1} (row p+1 = output digit, col q+1 = input digit,
                               LSB-first).  The plan applies the paper's row zeroing
                               (Eq. reduced_genmat_net2) and requires the result to
                               have columns q >= m - min(w_j,m) zero (column deletion),
                               which makes coordinate j periodic in k with period 2^{m-w_j}
                               (RQMC_DIGITAL_NET_ROWS: row zeroing only, any C).             */
  const double* shift;      /* lattice random shift Delta_j in [0,1), or NULL        */
  const uint64_t* dshift;   /* net digital shift sigma_j < 2^53: x = ((W << (53-m)) ^ sigma) 2^-53 */
  rqmc_map map;             /* RQMC_MAP_INVNORM: x = Phi^-1(u), u = 0 remapped (reading C-5) */
  int rank, world;          /* residue-class partition (see Layouts); (0,1) = whole problem  */
  uint64_t seed;            /* RQMC_REDUCED_MC: generator seed (z, C, shift, dshift unused)  */
} rqmc_plan_desc;

/* Level table entry (coarse -> fine), for inspection and tests. */
typedef struct {
  int w;            /* level index min(w_j, m) (m = constant level of shifted w_j >= m)        */
  int j_lo, s_w;    /* 0-based coordinates j_lo .. j_lo+s_w-1 (tau_w = s_w)             */
  int64_t M;        /* global distinct rows b^{m-w}                                            */
  int64_t M_local;  /* rows on this rank: nc M / ncls if M >= ncls, else nc (replicated)       */
  int parent;       /* index of the next coarser non-empty level, -1 for the top               */
  int coarse;       /* 1: materialised per-level GEMM pass; 0: fused into the fine kernel      */
  int fft;          /* 1: coarse level computed by the FFT product over the unit group of
                       Z / 2^k (unshifted b = 2 lattices, NEXT-4)   */
  int absorbed;     /* 1: coarse level merged into a finer coarse level's GEMM (small problems:
                       one launch for several levels; same points, P:307-309 -- unit map: the
                       merged columns generated at the absorbing level's rows; Phi^-1 map: each
                       level keeps its own reduced points, the GEMM reads level i at row r mod M_i) */
} rqmc_level_info;

typedef struct {
  int n_levels;             /* non-empty levels                                              */
  int checkpoint;           /* index of the last coarse level (root of the fine kernel)      */
  int n_fine;               /* fused fine levels below the checkpoint                        */
  int64_t n_bundles;        /* fine-kernel CTAs (bundles of residues of the checkpoint)      */
  int64_t N_local;          /* nc N / ncls (= N / world when world is a power of b)          */
  int s_star;               /* s* = max{j : w_j < m}                                 */
} rqmc_plan_summary;

rqmc_status rqmc_plan_create(const rqmc_plan_desc* desc, rqmc_plan_t* out);
void        rqmc_plan_destroy(rqmc_plan_t p);
const char* rqmc_strerror(rqmc_status s);
const char* rqmc_plan_last_error(rqmc_plan_t p);

rqmc_status rqmc_plan_summary_get(rqmc_plan_t p, rqmc_plan_summary* out);
rqmc_status rqmc_plan_level(rqmc_plan_t p, int idx, rqmc_level_info* out);
/* Global point index k of local row i (k = c0 + (i mod nc) + ncls (i div nc)); -1 if out of range. */
int64_t     rqmc_plan_global_row(rqmc_plan_t p, int64_t i);
/* Residue-class partition of this rank (see Layouts): ncls classes k mod ncls, this rank owns classes
 * first .. first+count-1.  Any output may be NULL. */
rqmc_status rqmc_plan_partition(rqmc_plan_t p, int64_t* classes, int64_t* first, int64_t* count);
/* Counter law: local rows, algorithmic MACs tau * sum_w M_w s_w and the
 * minimum HBM bytes 8 s tau (+ 8 N tau when Y is stored). */
rqmc_status rqmc_plan_stats(rqmc_plan_t p, int want_y, int64_t* local_rows, double* macs, double* min_bytes);

/* Bytes of device workspace a run needs (X^red of every level, checkpoint R buffers, partials,
 * b = 3 plans: the fine kernel's tail-split scratch and counters (zeroed by every run itself),
 * plus a staging copy of A for the *_host entry points).  Contents need no initialisation; one
 * workspace must not be shared by runs in flight concurrently. */
rqmc_status rqmc_workspace_size(rqmc_plan_t p, size_t* bytes);

/* Y = X A on this rank's rows (dY non-NULL, ldy >= tau); if f != RQMC_F_NONE and d_fsum != NULL,
 * also writes d_fsum[0] = sum over this rank's rows of f(x_k^T A) (fixed-order reduction).
 * Q_N = (all-reduce over ranks of d_fsum) / N. */
rqmc_status rqmc_xa(rqmc_plan_t p, const double* dA, int64_t lda, double* dY, int64_t ldy,
                    rqmc_f f, const double* fparam, double* d_fsum,
                    void* dwork, size_t wbytes, void* stream);

/* As rqmc_xa without storing Y (the N x tau result is consumed in registers by f). */
rqmc_status rqmc_qn(rqmc_plan_t p, const double* dA, int64_t lda, rqmc_f f, const double* fparam,
                    double* d_fsum, void* dwork, size_t wbytes, void* stream);

/* End-to-end form with HOST buffers: copies hA (pinned or pageable) into the workspace, runs
 * rqmc_qn and copies the local f-sum back into *h_fsum; synchronises the stream before returning.
 * The H2D copy of A runs on a plan-owned copy stream in the order the run reads it (each coarse
 * level's rows, coarse to fine, then the fine levels' rows), overlapped with the point generation and
 * the GEMMs before it: each GEMM waits only for its own rows.  With page-locked hA the whole sequence
 * (copies, kernels, the D2H into a plan-owned pinned slot) is captured once per (hA, lda, f, fparam,
 * dwork) as a CUDA graph and replayed; the replay reads hA's current contents.  Not reentrant per plan
 * (serialised by a plan mutex). */
rqmc_status rqmc_qn_host(rqmc_plan_t p, const double* hA, int64_t lda, rqmc_f f, const double* fparam,
                         double* h_fsum, void* dwork, size_t wbytes, void* stream);

/* rqmc_xa with A in HOST memory (pinned or pageable), the same piecewise overlapped H2D and graph
 * replay as rqmc_qn_host: Y = X A on this rank's rows into the caller's DEVICE buffer dY (ldy >= tau;
 * an N x tau result of up to tens of GB stays in HBM), and, if f != RQMC_F_NONE, the local f-sum into
 * *h_fsum (required then).  Synchronises the stream before returning.  The opt-in residue-chunk
 * pipeline (RQMC_CHUNKS) is not used here.  Errors: EINVAL (null hA / dY / dwork, f without h_fsum,
 * workspace too small), EDIM (lda or ldy < tau), ECUDA. */
rqmc_status rqmc_xa_host(rqmc_plan_t p, const double* hA, int64_t lda, double* dY, int64_t ldy,
                         rqmc_f f, const double* fparam, double* h_fsum, void* dwork, size_t wbytes,
                         void* stream);

/* Batched randomisation: R independent randomisations of
 * the SAME plan (generating vector / matrices, layout, map) and the same A, each giving its own
 * local f-sum:  d_fsum[r] = sum over this rank's rows of f(x^(r)_k^T A), r = 0..R-1 (device array).
 * Exactly the input matching the plan's kind is read (host arrays, copied by the call):
 *   lattice : hshifts  R*s doubles, row r = Delta^(r) in [0,1)^s (plan created with a shift)
 *   net     : hdshifts R*s words  < 2^53, row r = sigma^(r)        (plan created with a dshift)
 *   reduced MC: hseeds R seeds (replica r draws with seed hseeds[r]).
 * Q_N^(r) = (all-reduce of d_fsum[r]) / N; their mean and standard error over r form the RQMC
 * estimate.  Replica r computes what rqmc_qn computes for a plan holding that shift/seed -- bit for
 * bit when the batch runs with the single-run layout (same checkpoint, rqmc_plan_summary_batch),
 * else up to summation order.  Replicas run together (grid dimension) in
 * chunks of as many as the workspace holds; rqmc_workspace_size_batch(p, R) is the size for all R
 * at once (>= that of one replica).  Errors: EINVAL (missing input, unshifted plan, workspace below
 * one replica), ESHIFT (shift outside [0,1) / >= 2^53), ECUDA. */
rqmc_status rqmc_workspace_size_batch(rqmc_plan_t p, int R, size_t* bytes);
/* The layout a batch of R concurrent replicas with integrand f uses: replicas add parallelism, so
 * the checkpoint may sit coarser (more fused fine levels) than for a single run.  Fields checkpoint,
 * n_fine, n_bundles describe the batch layout; the rest as rqmc_plan_summary_get.  (f is reserved:
 * the current choice does not depend on it.) */
rqmc_status rqmc_plan_summary_batch(rqmc_plan_t p, int R, int f, rqmc_plan_summary* out);
rqmc_status rqmc_qn_batch(rqmc_plan_t p, int R, const double* hshifts, const uint64_t* hdshifts,
                          const uint64_t* hseeds, const double* dA, int64_t lda, rqmc_f f,
                          const double* fparam, double* d_fsum, void* dwork, size_t wbytes, void* stream);

/* Inspection / tests (host only, no device needed): the name of the fused fine-level kernel template
 * a run would launch for a batch of R replicas (R = 1: rqmc_xa / rqmc_qn), integrand f (RQMC_F_NONE:
 * Y only) and want_y (Y stored or not), e.g. "k_fine_tree<6,2,g=1,Y=0>" (compile-time log_b tree,
 * NF = 6 fine levels, b = 2, g = identity, Y not stored) or "k_fine<4,BotB2>" (general kernel, 4 fused
 * levels, hand-scheduled b = 2 bottom block).  Honors RQMC_NO_TREE / RQMC_CKPT_W like the run calls.
 * Writes a NUL-terminated string of at most len bytes.  Errors: EINVAL (NULL, len 0, R < 1). */
rqmc_status rqmc_plan_dispatch(rqmc_plan_t p, int R, int f, int want_y, char* buf, size_t len);

/* Debug / parity: the reduced points of level `idx` for local rows [r0, r0+count):
 * d_words[i*s_w+q] = integer word (lattice t = r z'_j mod M; net W or shifted V) and
 * d_vals[i*s_w+q] = the mapped fp64 coordinate.  Either output may be NULL. */
rqmc_status rqmc_points(rqmc_plan_t p, int idx, int64_t r0, int64_t count,
                        uint64_t* d_words, double* d_vals, void* stream);

/* Device-side phase timing for roofline reporting: while enabled (max_runs > 0) every run records
 * CUDA events on its stream around its phases (points, coarse GEMMs, fused fine kernel, reduction);
 * rqmc_profile_read synchronises those events and returns the summed milliseconds of the recorded
 * runs (and how many).  max_runs = 0 disables and frees the events.  Not thread-safe per plan. */
rqmc_status rqmc_profile_enable(rqmc_plan_t p, int max_runs);
rqmc_status rqmc_profile_read(rqmc_plan_t p, int* runs, double* ms_gen, double* ms_coarse,
                              double* ms_fine, double* ms_reduce);

#ifdef __cplusplus
}
#endif
#endif /* RQMC_H */
