/*
 * mscg.h — C ABI of the B200-native solve phase for the mini-Schur-complement
 * (MSC) domain-decomposition preconditioner (arXiv:1104.3349).
 *
 * The reference (/root/reference/proj, CPU-only C++20) has no FFI: its
 * boundary is the C++ API in proj/include/msc/.  Each entry point below is the
 * plain-pointer form of the reference call it replaces (cited per function).
 * The C++ drop-in layer (include/msc_b200/msc.hpp) re-exposes the reference
 * signatures over these calls; Python binds them with ctypes
 * (paper_1104_3349_b200/_capi.py).
 *
 * Conventions
 *   - int32 CSR (row offsets, columns strictly increasing per row), fp64
 *     values: the reference SparseMatrix layout (sparse_matrix.hpp:77-81).
 *   - Every function returns an mscg_code; on failure *status (if non-null)
 *     carries the code, the failing block and the zero-pivot index (reference
 *     SingularMatrixError{pivot_index}, sparse_matrix.hpp:23-28) and a message
 *     with the reference's wording (e.g. "build_preconditioner: (1,1) block 3:
 *     factor_ilut: zero pivot at index 2207").
 *   - Vectors passed with MSCG_MEM_HOST are host arrays (copied through
 *     pinned staging); MSCG_MEM_DEVICE are device pointers on the handle's
 *     device and stream.  There is no CPU fallback: without a CUDA device the
 *     device entry points fail with MSCG_ERR_CUDA.
 *
 * Limits the reference does not have (each fails with
 * MSCG_ERR_INVALID_ARGUMENT and a message naming it, never silently):
 *   - a factored block (interior block, Schur block, or the whole overlapped
 *     band) holds at most 65535 rows: factor columns are stored block-local
 *     as uint16;
 *   - the ILUT working row (8 B per block row) and the triangular solve's
 *     solution vector plus far-sum slots live in shared memory (227 KB per
 *     CTA): about 27 000 rows per ILUT block and 25 000 per solved block
 *     (BASELINE blocks are <= 3 400 rows; cfg3's whole S^ band is 6 360);
 *   - GMRES restart <= 500 (the Givens state is staged in shared memory);
 *   - a context drives one device; contexts on several devices may coexist
 *     in one process.
 */
#ifndef MSCG_H
#define MSCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSCG_ABI_VERSION 1

typedef enum {
  MSCG_OK = 0,
  MSCG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  MSCG_ERR_SINGULAR = 2,         /* SingularMatrixError */
  MSCG_ERR_CUDA = 3,             /* no device / CUDA runtime failure */
  MSCG_ERR_OUT_OF_MEMORY = 4,
  MSCG_ERR_RUNTIME = 5,          /* std::runtime_error */
  MSCG_ERR_IO = 6                /* msc::IoError (matrix_market.hpp:16-24) */
} mscg_code;

typedef enum { MSCG_MEM_HOST = 0, MSCG_MEM_DEVICE = 1 } mscg_mem;

typedef struct {
  int code;
  int block;        /* failing interior / Schur block, -1 if n/a */
  int pivot_index;  /* zero pivot (local row), -1 if n/a */
  char message[512];
} mscg_status;

typedef struct mscg_ctx mscg_ctx;         /* device, stream, scratch */
typedef struct mscg_csr mscg_csr;         /* device-resident sparse matrix */
typedef struct mscg_precond mscg_precond; /* device-resident MSC preconditioner */
typedef struct mscg_problem mscg_problem; /* host setup: partitioned system */
typedef struct mscg_factors mscg_factors; /* device-resident factors of one block */

int mscg_abi_version(void);

/* ---- context ------------------------------------------------------------ */
int mscg_ctx_create(int device, mscg_ctx **out, mscg_status *st);
void mscg_ctx_destroy(mscg_ctx *ctx);
/* cudaStream_t of the context (as void*), for callers that pass device ptrs. */
void *mscg_ctx_stream(mscg_ctx *ctx);
/* Order every later call of this context on `stream` (a cudaStream_t owned by
 * the caller, e.g. the stream a collective library runs on; NULL is the legacy
 * default stream); use_own != 0 restores the context's own stream. */
int mscg_ctx_set_stream(mscg_ctx *ctx, void *stream, int use_own,
                        mscg_status *st);
int mscg_ctx_synchronize(mscg_ctx *ctx, mscg_status *st);
/* Kernels launched by this library since creation (evidence counter). */
int64_t mscg_ctx_launches(mscg_ctx *ctx);
/* Interior correction of preconditioners built later on this context (no
 * reference counterpart; the result is the same operator): 0 = the
 * reference's two steps w = E z2, x1 = z1 - D^-1 w; 1 = precompute
 * W = D^-1 E per interior block at build time and apply x1 = z1 - W z2;
 * 2 = auto (1 when W is smaller than the interior factors and fits; the
 * default, overridable by MSCG_CORRECTION=off|on|auto); -1 = default. */
#define MSCG_CORRECTION_OFF 0
#define MSCG_CORRECTION_ON 1
#define MSCG_CORRECTION_AUTO 2
int mscg_ctx_set_correction(mscg_ctx *ctx, int mode, mscg_status *st);

/* ---- host problem layer (setup, once) -------------------- */
/* generate_oseen(grid_n, nu, Uniform|Stretched, Recirculating, stretch)
 * (oseen.hpp:43-44) -> scale_rows (row_scaling.hpp:23) ->
 * partition_saddle(.., nA, Interleaved) (partitioned_matrix.hpp:69-70)
 * [-> SURVEY §8(d) interface anchoring when anchored != 0]. */
int mscg_problem_oseen(int grid_n, double nu, int stretched, double stretch,
                       int n_a, int anchored, int threads, mscg_problem **out,
                       mscg_status *st);
/* PartitionedMatrix::from_split(C, p, d_ranges) (partitioned_matrix.hpp:28-29). */
/* The same with generate_oseen's assembly and scale_rows on the device
 * (oseen.cpp:108-212, row_scaling.cpp:8-31): bit-identical
 * matrix and rhs; partition and anchoring stay on the host. */
int mscg_problem_oseen_device(mscg_ctx *ctx, int grid_n, double nu, int stretched,
                              double stretch, int n_a, int anchored, int threads,
                              mscg_problem **out, mscg_status *st);
int mscg_problem_from_csr(int n, const int *rp, const int *ci, const double *v,
                          int p, int nranges, const int *ranges,
                          mscg_problem **out, mscg_status *st);
void mscg_problem_destroy(mscg_problem *pb);
/* nested_dissection(build_graph(A), target) (graph.cpp:8-30,178-230) of the
 * pattern of a square CSR matrix, on the device (ctx) or the host (ctx NULL,
 * `threads` workers): perm[n] = forward permutation (blocks in depth-first
 * leaf order, each ascending, then the ascending separator), *nblocks, and
 * ranges[2*cap] the block ranges.  Identical to the reference.  (The Oseen
 * problem builders use it inside partition_saddle; mscg_problem_oseen_device
 * runs it on the device.) */
int mscg_nested_dissection(mscg_ctx *ctx, int n, const int *rp, const int *ci, int target,
                           int threads, int *perm, int *nblocks, int *ranges, int cap,
                           mscg_status *st);
void mscg_problem_dims(const mscg_problem *pb, int *n, int *p, int *nblocks,
                       int64_t *nnz_c, int *separator_size);
/* which: 0 = C (final numbering), 5 = S^ (after mscg_problem_build_schur).
 * Pointers are borrowed (valid until the problem is destroyed). */
int mscg_problem_csr(const mscg_problem *pb, int which, int *nrows, int *ncols,
                     int64_t *nnz, const int **rp, const int **ci,
                     const double **v);
const int *mscg_problem_perm(const mscg_problem *pb);
const int *mscg_problem_d_ranges(const mscg_problem *pb);   /* 2*nblocks */
const double *mscg_problem_scaled_rhs(const mscg_problem *pb); /* or NULL */
/* build_msc (schur_approx.hpp:45-46) for variant "lum" | "mscn" | "mscnr"
 * with numbering aggregates.  mode 0: equal_sizes(n_g, sz) (sz<=0 -> n_g/8,
 * benchmark.cpp:74-77); mode 1: anchored greedy sizes;
 * mode 2: explicit sizes[nsizes]. */
int mscg_problem_build_schur(mscg_problem *pb, const char *variant, int mode,
                             int sz, int nsizes, const int *sizes, int threads,
                             mscg_status *st);
/* The same on the device (one CTA per aggregate: dense LU of D_ii, multi-RHS
 * solve, correction), S^ bit-identical to the host build and the reference
 * (schur_approx.cpp:88-161). */
int mscg_problem_build_schur_device(mscg_ctx *ctx, mscg_problem *pb, const char *variant,
                                    int mode, int sz, int nsizes, const int *sizes,
                                    mscg_status *st);
/* build_msc over OVERLAPPED numbering aggregates (aggregate_overlapped,
 * aggregates.cpp:50-85) for "omscn" | "omscnr" | "olum": owned sizes as
 * mscg_problem_build_schur (mode 0/1/2); widths[nwidths] explicit (one per
 * aggregate), or (widths NULL) `overlap` for every aggregate (< 0: sz), the last 0,
 * clipped to min(size - 1, n_g - end) (benchmark.cpp:74-88).  Each
 * aggregate's S_ii lives on its span [b, e + w); the merge writes every owned
 * column over the whole span (schur_approx.cpp:141-160), so S^ is banded and
 * a preconditioner built from this problem factors it whole (one exact LU,
 * the reference's schur_single_).  ctx NULL: host build; else on the device
 * (local blocks) with the merge on the host.  Errors as the reference
 * ("aggregate_overlapped: ...", "build_msc: variant omscn needs an
 * overlapped aggregate set"). */
int mscg_problem_build_schur_overlapped(mscg_ctx *ctx, mscg_problem *pb, const char *variant,
                                        int mode, int sz, int nsizes, const int *sizes,
                                        int overlap, int nwidths, const int *widths,
                                        int threads, mscg_status *st);
int mscg_problem_num_aggregates(const mscg_problem *pb);
const int *mscg_problem_schur_ranges(const mscg_problem *pb); /* 2*nagg */

/* ---- device sparse matrices ---------------------------------------------- */
/* Upload CSR to HBM (SELL-32 slices for the SpMV kernel). */
int mscg_csr_upload(mscg_ctx *ctx, int nrows, int ncols, const int *rp,
                    const int *ci, const double *v, mscg_csr **out,
                    mscg_status *st);
void mscg_csr_destroy(mscg_csr *a);
/* y = A x with the reference's row-sequential accumulation order
 * (matvec, sparse_matrix.cpp:110-125): bit-identical results. */
int mscg_spmv(mscg_csr *a, const double *x, double *y, int mem,
              mscg_status *st);

/* ---- MSC preconditioner ------------------------------------------------ */
/* nschur = MSCG_SCHUR_SINGLE: S^ is an overlapped band, factored whole by one
 * exact LU (preconditioner.cpp:58-67; s_ranges unused); a singular band
 * raises "build_preconditioner: overlapped Schur band: dense_lu: zero pivot
 * at index i". */
#define MSCG_SCHUR_SINGLE (-1)
/* build_preconditioner(c, schur, tolA, sA) (preconditioner.hpp:66-68) over
 * raw arrays: C (n x n, final numbering) split at p, interior block ranges,
 * block-diagonal S^ (n_g x n_g) with its owned ranges.  Interior blocks with
 * dim <= sA get the exact LU (factor_exact), the others ILUT(tolA)
 * (factor_ilut, factorization.cpp:34-127), batched on the device. */
int mscg_precond_build(mscg_ctx *ctx, int n, int p, const int *c_rp,
                       const int *c_ci, const double *c_v, int nblocks,
                       const int *d_ranges, const int *s_rp, const int *s_ci,
                       const double *s_v, int nschur, const int *s_ranges,
                       double tol_a, int s_a, mscg_precond **out,
                       mscg_status *st);
/* factor_ilut(a, tol) (kind 0, factorization.hpp:38, factorization.cpp:34-127)
 * or factor_exact(a) (kind 1, factorization.hpp:32, dense_lu with partial
 * pivoting) of one square CSR block on the device.  Errors as the reference:
 * "factor_ilut: zero pivot at index i" / "dense_lu: zero pivot at index i"
 * (MSCG_ERR_SINGULAR, pivot_index = i), "factor_ilut: negative drop
 * tolerance" (MSCG_ERR_INVALID_ARGUMENT).  Blocks up to 65535 rows. */
int mscg_factor(mscg_ctx *ctx, int n, const int *rp, const int *ci, const double *v,
                int kind, double tol, mscg_factors **out, mscg_status *st);
/* TriangularFactors in the reference CSR (factorization.hpp:18-27): L strictly
 * lower (unit diagonal implicit), U with its diagonal, row_perm.forward.
 * Call with lrp == NULL first to get the sizes. */
int mscg_factors_get(const mscg_factors *f, int *dim, int64_t *nnz_l, int64_t *nnz_u,
                     int *lrp, int *lci, double *lv, int *urp, int *uci, double *uv,
                     int *perm, mscg_status *st);
/* x = U^-1 L^-1 P b (solve, factorization.hpp:41, factorization.cpp:129-158). */
int mscg_factors_solve(mscg_factors *f, const double *b, double *x, int mem,
                       mscg_status *st);
void mscg_factors_destroy(mscg_factors *f);
int mscg_precond_build_problem(mscg_ctx *ctx, const mscg_problem *pb,
                               double tol_a, int s_a, mscg_precond **out,
                               mscg_status *st);
void mscg_precond_destroy(mscg_precond *pc);
/* ---- sharded preconditioner (no reference counterpart) ----
 * A shard owns interior blocks [block_begin, block_end) of the same split
 * (its D blocks, E rows and F columns; the Schur factors are replicated).
 * One apply across ranks, device pointers, global-length vectors:
 *   apply_shard(phase 0, y, t, -): z1_r = D_r^-1 y1_r, t = F_r z1_r   (n_g)
 *   caller:  t = sum over ranks of t                    (all-reduce)
 *   apply_shard(phase 1, y, t, x): x2 = S^-1 (y2 - t), x1_r = z1_r - D_r^-1 E_r x2
 * Each rank's x holds its interior rows [row_lo, row_hi) and all of x2.
 * spmv_shard: y1_r = C[rows_r, :] x and y2part = F_r x1_r (+ C22 x2 when
 * with_interface_block, on exactly one rank); sum y2part over ranks for the
 * interface rows of C x. */
int mscg_precond_build_shard(mscg_ctx *ctx, int n, int p, const int *c_rp,
                             const int *c_ci, const double *c_v, int nblocks,
                             const int *d_ranges, const int *s_rp,
                             const int *s_ci, const double *s_v, int nschur,
                             const int *s_ranges, double tol_a, int s_a,
                             int block_begin, int block_end, mscg_precond **out,
                             mscg_status *st);
int mscg_precond_build_problem_shard(mscg_ctx *ctx, const mscg_problem *pb,
                                     double tol_a, int s_a, int block_begin,
                                     int block_end, mscg_precond **out,
                                     mscg_status *st);
int mscg_precond_shard_rows(const mscg_precond *pc, int *row_lo, int *row_hi);
int mscg_precond_apply_shard(mscg_precond *pc, int phase, const double *y_dev,
                             double *t_dev, double *x_dev, mscg_status *st);
int mscg_precond_spmv_shard(mscg_precond *pc, const double *x_dev,
                            double *y_dev, double *y2part_dev,
                            int with_interface_block, mscg_status *st);

/* MscPreconditioner::apply (preconditioner.cpp:85-114): x = B^-1 y. */
int mscg_precond_apply(mscg_precond *pc, const double *y, double *x, int mem,
                       mscg_status *st);
/* stored_nnz (preconditioner.cpp:116-121): factor nnz + nnz(E) + nnz(F). */
/* x = B^-1 y with device vectors, enqueued on `stream` (NULL = legacy
 * default stream) instead of the context's.  Applies on different streams,
 * from any threads, run concurrently: each stream gets its own scratch
 * (the reference promises apply is safe from several threads,
 * preconditioner.hpp:17-18). */
int mscg_precond_apply_stream(mscg_precond *pc, const double *y_dev, double *x_dev,
                              void *stream, mscg_status *st);
int64_t mscg_precond_stored_nnz(const mscg_precond *pc);
int mscg_precond_dims(const mscg_precond *pc, int *n, int *p, int *nblocks,
                      int *nschur);
/* Factor download for the d_factors()/schur_factors() accessors
 * (preconditioner.hpp:41-44): kind 0 = interior blocks, 1 = Schur blocks.
 * Reference layout: L strict lower, U with its diagonal first in each row,
 * row_perm forward map.  Pass NULL arrays to query sizes only. */
int mscg_precond_factor(const mscg_precond *pc, int kind, int idx, int *dim,
                        int64_t *nnz_l, int64_t *nnz_u, int *lrp, int *lci,
                        double *lv, int *urp, int *uci, double *uv, int *perm,
                        mscg_status *st);
/* Timing breakdown of the last build (seconds). */
int mscg_precond_build_times(const mscg_precond *pc, double *ilut_s,
                             double *schur_lu_s, double *pack_s);
/* Interior correction of this preconditioner: *on = 1 when W = D^-1 E is
 * in use, *entries = its fp64 entries, *kmax = most interface columns of a
 * block, *build_s = seconds spent building it. */
int mscg_precond_correction(const mscg_precond *pc, int *on, int64_t *entries,
                            int *kmax, double *build_s);
/* The operator matrix C of the preconditioner, resident on the device. */
mscg_csr *mscg_precond_matrix(mscg_precond *pc);

/* Stored-entry counts for roofline bookkeeping: interior-block L and U
 * (U without its diagonal), Schur-block L and U, E, F and C. */
int mscg_precond_nnz(const mscg_precond *pc, int64_t counts[7]);
/* Select, per preconditioner, whether applies use the explicit correction
 * panels when they were built (1, default) or the reference's E SpMV +
 * second interior solve (0).  Same operator; used by the bench to report
 * both apply rates.  Not synchronised with in-flight applies. */
int mscg_precond_use_correction(mscg_precond *pc, int on);
/* Bytes of the device layout one apply streams (what the kernels move, as
 * opposed to the reference-CSR "algorithmic" count): [0] one interior
 * solve pass, [1] one Schur solve pass, [2] correction panels + z1/x1,
 * [3] E and F (SELL), [4] C (SELL), [5] vectors; breakdown of [0]: [6] near
 * tiles (copied prefixes, both triangles), [7] far entries, [8] work items,
 * [9] number of near tiles kept dense. */
int mscg_precond_layout_bytes(const mscg_precond *pc, int64_t out[10]);

/* ---- measurement helpers ------------------------------------------------ */
/* oracle::random_vector (proj/tests/oracles.hpp:92-98): std::mt19937(seed)
 * + std::uniform_real_distribution<double>(-1, 1), the reference's seeded
 * right-hand-side convention. */
void mscg_random_vector(int n, unsigned seed, double *out);
/* `steps` back-to-back [apply(y) -> x; C x -> w] (with_spmv) on device
 * vectors, timed with CUDA events on the context stream.  total_ms: first to
 * last event; stage_ms[6]: summed per stage (D-solve, F-SpMV, S-solve,
 * E-SpMV, D-solve+sub, C-SpMV); launches: kernels enqueued. */
int mscg_bench_apply(mscg_precond *pc, const double *y_dev, double *x_dev,
                     double *w_dev, int steps, int with_spmv, double *total_ms,
                     double *stage_ms, int64_t *launches, mscg_status *st);

/* Tracing (diagnostics): one interior-block solve pass with SM clock stamps
 * for block 0 — per tile (data landed, far sums in, tile solved) and per far
 * work item (start, dot done, published, id); see tools/trace_*.py.
 * cap >= 32 * dim(block 0) int64.
 * Returns dim(block 0). */
int mscg_debug_trace_dsolve(mscg_precond *pc, const double *y_dev, double *x_dev,
                            int64_t *out, int cap, mscg_status *st);

/* ---- restarted GMRES (gmres.hpp:44-47, gmres.cpp:35-191) -------------- */
typedef struct {
  int restart;      /* default 300 */
  int max_iters;    /* default 3000 */
  double rel_tol;   /* default 1e-9 */
  int side;         /* 0 = right (default), 1 = left */
  int orth;         /* 0 = MGS (reference order), 1 = CGS2 (three basis sweeps),
                       2 = DCGS2 (two basis sweeps, delayed reorthogonalisation) */
} mscg_gmres_config;

typedef struct {
  int iterations;
  int converged;
  int history_len;  /* residual_history entries written (<= hist_cap) */
  int history_total;
  double solve_seconds;
  double final_true_residual;
} mscg_gmres_report;

/* A = operator on the device (usually mscg_precond_matrix(pc)); pc may be
 * NULL for an unpreconditioned solve. */
int mscg_gmres(mscg_ctx *ctx, mscg_csr *a, mscg_precond *pc, const double *b,
               double *x, int mem, const mscg_gmres_config *cfg,
               mscg_gmres_report *rep, double *history, int hist_cap,
               mscg_status *st);

/* Distributed right-preconditioned GMRES (DCGS2) over preconditioner shards
 * (no reference counterpart): one process per GPU, each with its
 * shard (mscg_precond_build_shard).  b, x are global-length vectors (x gets
 * the rank's interior rows and the interface, other rows zero).  Krylov
 * vectors are compact per rank ([own interior rows | interface], the
 * interface replicated); the exchanges per iteration are two n_g all-reduces
 * (preconditioner, matvec) and two short ones (the 2j+2 sweep-1 dots and one
 * norm).  allreduce(count, user) must replace comm_buf[0:count] (device,
 * comm_cap >= max(2*restart+4, n_g) doubles) by its sum over the ranks, in
 * stream order on the context stream (NCCL on that stream, or gloo on CUDA
 * tensors).  cfg->side must be right and cfg->orth DCGS2. */
typedef void (*mscg_allreduce_fn)(int count, void *user);
int mscg_gmres_shard(mscg_ctx *ctx, mscg_precond *shard, int rank, int world,
                     const double *b, double *x, int mem, const mscg_gmres_config *cfg,
                     double *comm_buf, int comm_cap, mscg_allreduce_fn allreduce,
                     void *user, mscg_gmres_report *rep, double *history, int hist_cap,
                     mscg_status *st);
/* true_residual (gmres.cpp:26-33). */
int mscg_true_residual(mscg_ctx *ctx, mscg_csr *a, const double *x,
                       const double *b, int mem, double *out, mscg_status *st);

/* ---- Matrix Market coordinate I/O (host) -------------------------------
 * Replaces load_matrix_market / write_matrix_market / load_vector_market /
 * write_vector_market (proj/include/msc/matrix_market.hpp:26-36,
 * proj/src/matrix_market.cpp:20-142).  mscg_mm_read with rp == NULL only
 * reports the sizes; call again with rp[nrows+1], ci[nnz], v[nnz].  Failures
 * return MSCG_ERR_IO with the reference's message ("... (line N)"). */
int mscg_mm_read(const char *path, int *nrows, int *ncols, int64_t *nnz, int *rp,
                 int *ci, double *v, mscg_status *st);
int mscg_mm_write(const char *path, int nrows, int ncols, const int *rp, const int *ci,
                  const double *v, mscg_status *st);
/* n x 1 coordinate files; v == NULL only reports n */
int mscg_mm_read_vector(const char *path, int *n, double *v, mscg_status *st);
int mscg_mm_write_vector(const char *path, int n, const double *v, mscg_status *st);

#ifdef __cplusplus
}
#endif
#endif /* MSCG_H */
