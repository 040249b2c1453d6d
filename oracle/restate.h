/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the hot path.
 *
 * Plain-C restatement of the reference's solve-phase algorithms (each
 * function cites the reference file:line it follows).  Built by
 * oracle/Makefile into oracle/_build/liborestate.so with -ffp-contract=off so
 * its arithmetic is bit-identical to the reference compiled for x86-64
 * (which has no FMA).  Pinned against the compiled reference
 * (oracle/_ref/libmscref.so) and the committed fixtures in tests/golden/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 */
#ifndef MSC_ORACLE_RESTATE_H
#define MSC_ORACLE_RESTATE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CSR with int32 offsets (reference SparseMatrix, sparse_matrix.hpp:77-81). */
typedef struct {
  int n;
  int *rp, *ci;
  double *v;
} rs_csr;

typedef struct {
  int n;
  rs_csr L, U;   /* L strict lower (unit diag implicit), U with diagonal */
  int *perm;     /* row_perm.forward */
} rs_factors;

void rs_matvec(int nrows, const int *rp, const int *ci, const double *v,
               const double *x, double *y);

/* Returns 0, or -1 - pivot on a zero pivot (SingularMatrixError). */
int rs_ilut(int n, const int *rp, const int *ci, const double *v, double tol,
            rs_factors **out);
int rs_exact(int n, const int *rp, const int *ci, const double *v,
             rs_factors **out);
void rs_factors_free(rs_factors *f);
void rs_factors_dims(const rs_factors *f, int *n, int64_t *nnz_l, int64_t *nnz_u);
void rs_factors_get(const rs_factors *f, int *lrp, int *lci, double *lv,
                    int *urp, int *uci, double *uv, int *perm);
void rs_solve(const rs_factors *f, const double *b, double *x);

/* MSC preconditioner apply (preconditioner.cpp:85-114) over given factors. */
typedef struct {
  int n, p;
  int nd, ns;
  const int *d_ranges, *s_ranges;   /* [begin,end) pairs */
  rs_factors **dfac, **sfac;
  int e_nrows; const int *e_rp, *e_ci; const double *e_v;   /* E: p x n_g */
  int f_nrows; const int *f_rp, *f_ci; const double *f_v;   /* F: n_g x p */
} rs_msc;

void rs_msc_apply(const rs_msc *m, const double *y, double *x);

/* Restarted GMRES (gmres.cpp:35-191).  side: 0 none, 1 right, 2 left.
 * hist capacity *nhist on input, count on output. */
int rs_gmres(int n, const int *rp, const int *ci, const double *v,
             const rs_msc *m, int side, const double *b, int restart,
             int max_iters, double rel_tol, double *x, int *iters,
             int *converged, double *hist, int *nhist);

#ifdef __cplusplus
}
#endif
#endif
