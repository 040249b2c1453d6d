/* TEST INFRASTRUCTURE ONLY — see restate.h.
 *
 * Plain-C restatement of the reference hot path.  Compiled with
 * -ffp-contract=off: every product/sum below is a separately rounded IEEE
 * operation in the same order as the reference, so results are bit-identical
 * to /root/reference/proj built for x86-64 (no FMA).
 */
#include "restate.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static void *xmalloc(size_t n) {
  void *p = malloc(n ? n : 1);
  if (!p) abort();
  return p;
}

typedef struct {
  int *c;
  double *v;
  int64_t n, cap;
} vec_cv;

static void cv_push(vec_cv *a, int c, double v) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 64;
    a->c = realloc(a->c, sizeof(int) * a->cap);
    a->v = realloc(a->v, sizeof(double) * a->cap);
    if (!a->c || !a->v) abort();
  }
  a->c[a->n] = c;
  a->v[a->n] = v;
  a->n++;
}

/* y = A x, row-major sequential accumulation: sparse_matrix.cpp:110-125. */
void rs_matvec(int nrows, const int *rp, const int *ci, const double *v,
               const double *x, double *y) {
  for (int i = 0; i < nrows; ++i) {
    double acc = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) acc += v[k] * x[ci[k]];
    y[i] = acc;
  }
}

static int cmp_int(const void *a, const void *b) {
  int x = *(const int *)a, y = *(const int *)b;
  return (x > y) - (x < y);
}

/* Row-wise IKJ ILUT with dropping: factorization.cpp:34-127.
 *  - tau = tol * ||original row i||_2 (:55-58)
 *  - pending pivots k < i taken in ascending order (std::set, :64-94); fills
 *    from U rows only add indices > k, so a forward scan reproduces the order
 *  - multiplier dropped when |m| < tau or m == 0 (:77-80)
 *  - L keeps nonzero multipliers, U keeps |v| >= tau && v != 0 off-diagonal,
 *    the diagonal always, zero diagonal -> SingularMatrixError(i) (:97-116). */
int rs_ilut(int n, const int *rp, const int *ci, const double *v, double tol,
            rs_factors **out) {
  double *work = xmalloc(sizeof(double) * n);
  char *present = xmalloc(n);
  char *pending = xmalloc(n);
  int *touched = xmalloc(sizeof(int) * n);
  double *udiag = xmalloc(sizeof(double) * n);
  int64_t *ustart = xmalloc(sizeof(int64_t) * (n + 1));
  memset(work, 0, sizeof(double) * n);
  memset(present, 0, n);
  memset(pending, 0, n);
  vec_cv L = {0}, U = {0};      /* U without diagonal (the replay rows) */
  int *lrp = xmalloc(sizeof(int) * (n + 1));
  lrp[0] = 0;
  ustart[0] = 0;
  int rc = 0;

  for (int i = 0; i < n; ++i) {
    double row_norm = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) row_norm += v[k] * v[k];
    row_norm = sqrt(row_norm);
    const double tau = tol * row_norm;
    int nt = 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      work[ci[k]] = v[k];
      present[ci[k]] = 1;
      touched[nt++] = ci[k];
      if (ci[k] < i) pending[ci[k]] = 1;
    }
    for (int k = 0; k < i; ++k) {
      if (!pending[k]) continue;
      pending[k] = 0;
      const double mult = work[k] / udiag[k];
      if (fabs(mult) < tau || mult == 0.0) {
        work[k] = 0.0;
        continue;
      }
      work[k] = mult;
      for (int64_t t = ustart[k]; t < ustart[k + 1]; ++t) {
        const int j = U.c[t];
        if (!present[j]) {
          present[j] = 1;
          work[j] = 0.0;
          touched[nt++] = j;
          if (j < i) pending[j] = 1;
        }
        work[j] -= mult * U.v[t];
      }
    }
    qsort(touched, nt, sizeof(int), cmp_int);
    double diag = 0.0;
    for (int t = 0; t < nt; ++t) {
      const int j = touched[t];
      const double val = work[j];
      if (j < i) {
        if (val != 0.0) cv_push(&L, j, val);
      } else if (j == i) {
        diag = val;
      } else if (fabs(val) >= tau && val != 0.0) {
        cv_push(&U, j, val);
      }
      work[j] = 0.0;
      present[j] = 0;
    }
    lrp[i + 1] = (int)L.n;
    ustart[i + 1] = U.n;
    if (diag == 0.0) {
      rc = -1 - i;
      break;
    }
    udiag[i] = diag;
  }

  if (rc == 0) {
    rs_factors *f = xmalloc(sizeof(rs_factors));
    f->n = n;
    f->L.n = n;
    f->L.rp = lrp;
    f->L.ci = xmalloc(sizeof(int) * L.n);
    f->L.v = xmalloc(sizeof(double) * L.n);
    memcpy(f->L.ci, L.c, sizeof(int) * L.n);
    memcpy(f->L.v, L.v, sizeof(double) * L.n);
    /* U rows: diagonal first (smallest column), then the kept entries. */
    const int64_t unnz = U.n + n;
    f->U.n = n;
    f->U.rp = xmalloc(sizeof(int) * (n + 1));
    f->U.ci = xmalloc(sizeof(int) * unnz);
    f->U.v = xmalloc(sizeof(double) * unnz);
    int64_t w = 0;
    f->U.rp[0] = 0;
    for (int i = 0; i < n; ++i) {
      f->U.ci[w] = i;
      f->U.v[w++] = udiag[i];
      for (int64_t t = ustart[i]; t < ustart[i + 1]; ++t) {
        f->U.ci[w] = U.c[t];
        f->U.v[w++] = U.v[t];
      }
      f->U.rp[i + 1] = (int)w;
    }
    f->perm = xmalloc(sizeof(int) * n);
    for (int i = 0; i < n; ++i) f->perm[i] = i;
    *out = f;
  } else {
    free(lrp);
  }
  free(L.c); free(L.v); free(U.c); free(U.v);
  free(work); free(present); free(pending); free(touched); free(udiag);
  free(ustart);
  return rc;
}

/* LU with partial pivoting (dense_matrix.cpp:85-123, first max wins ties,
 * exactly-zero pivot column throws) re-stored sparse (factorization.cpp:11-32). */
int rs_exact(int n, const int *rp, const int *ci, const double *v,
             rs_factors **out) {
  double *a = xmalloc(sizeof(double) * (size_t)n * n);
  memset(a, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k) a[(size_t)i * n + ci[k]] = v[k];
  int *perm = xmalloc(sizeof(int) * n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = fabs(a[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      if (fabs(a[(size_t)i * n + k]) > best) {
        best = fabs(a[(size_t)i * n + k]);
        piv = i;
      }
    }
    if (best == 0.0) {
      free(a);
      free(perm);
      return -1 - k;
    }
    if (piv != k) {
      for (int j = 0; j < n; ++j) {
        double t = a[(size_t)k * n + j];
        a[(size_t)k * n + j] = a[(size_t)piv * n + j];
        a[(size_t)piv * n + j] = t;
      }
      int t = perm[k]; perm[k] = perm[piv]; perm[piv] = t;
    }
    const double pivot = a[(size_t)k * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double lik = a[(size_t)i * n + k] / pivot;
      a[(size_t)i * n + k] = lik;
      if (lik == 0.0) continue;
      for (int j = k + 1; j < n; ++j)
        a[(size_t)i * n + j] -= lik * a[(size_t)k * n + j];
    }
  }
  vec_cv L = {0}, U = {0};
  rs_factors *f = xmalloc(sizeof(rs_factors));
  f->n = n;
  f->L.n = f->U.n = n;
  f->L.rp = xmalloc(sizeof(int) * (n + 1));
  f->U.rp = xmalloc(sizeof(int) * (n + 1));
  f->L.rp[0] = f->U.rp[0] = 0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < i; ++j)
      if (a[(size_t)i * n + j] != 0.0) cv_push(&L, j, a[(size_t)i * n + j]);
    for (int j = i; j < n; ++j)
      if (a[(size_t)i * n + j] != 0.0) cv_push(&U, j, a[(size_t)i * n + j]);
    f->L.rp[i + 1] = (int)L.n;
    f->U.rp[i + 1] = (int)U.n;
  }
  f->L.ci = L.c ? L.c : xmalloc(sizeof(int));
  f->L.v = L.v ? L.v : xmalloc(sizeof(double));
  f->U.ci = U.c;
  f->U.v = U.v;
  f->perm = perm;
  free(a);
  *out = f;
  return 0;
}

void rs_factors_free(rs_factors *f) {
  if (!f) return;
  free(f->L.rp); free(f->L.ci); free(f->L.v);
  free(f->U.rp); free(f->U.ci); free(f->U.v);
  free(f->perm);
  free(f);
}

void rs_factors_dims(const rs_factors *f, int *n, int64_t *nnz_l, int64_t *nnz_u) {
  *n = f->n;
  *nnz_l = f->L.rp[f->n];
  *nnz_u = f->U.rp[f->n];
}

void rs_factors_get(const rs_factors *f, int *lrp, int *lci, double *lv,
                    int *urp, int *uci, double *uv, int *perm) {
  const int n = f->n;
  memcpy(lrp, f->L.rp, sizeof(int) * (n + 1));
  memcpy(lci, f->L.ci, sizeof(int) * f->L.rp[n]);
  memcpy(lv, f->L.v, sizeof(double) * f->L.rp[n]);
  memcpy(urp, f->U.rp, sizeof(int) * (n + 1));
  memcpy(uci, f->U.ci, sizeof(int) * f->U.rp[n]);
  memcpy(uv, f->U.v, sizeof(double) * f->U.rp[n]);
  if (perm) memcpy(perm, f->perm, sizeof(int) * n);
}

/* x = U^-1 L^-1 P b: factorization.cpp:129-158. */
void rs_solve(const rs_factors *f, const double *b, double *x) {
  const int n = f->n;
  for (int i = 0; i < n; ++i) x[i] = b[f->perm[i]];
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int k = f->L.rp[i]; k < f->L.rp[i + 1]; ++k) s -= f->L.v[k] * x[f->L.ci[k]];
    x[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    double diag = 0.0;
    for (int k = f->U.rp[i]; k < f->U.rp[i + 1]; ++k) {
      if (f->U.ci[k] == i) diag = f->U.v[k];
      else s -= f->U.v[k] * x[f->U.ci[k]];
    }
    x[i] = s / diag;
  }
}

/* block_solve: preconditioner.cpp:13-22. */
static void block_solve(int nb, const int *ranges, rs_factors **fac,
                        const double *y, double *z) {
  for (int b = 0; b < nb; ++b) {
    const int beg = ranges[2 * b];
    rs_solve(fac[b], y + beg, z + beg);
  }
}

/* MscPreconditioner::apply: preconditioner.cpp:85-114 (block-diagonal S^). */
void rs_msc_apply(const rs_msc *m, const double *y, double *x) {
  const int p = m->p, ng = m->n - m->p;
  double *z1 = xmalloc(sizeof(double) * (p + 1));
  double *t = xmalloc(sizeof(double) * (ng + 1));
  double *z2 = xmalloc(sizeof(double) * (ng + 1));
  double *w = xmalloc(sizeof(double) * (p + 1));
  double *corr = xmalloc(sizeof(double) * (p + 1));
  block_solve(m->nd, m->d_ranges, m->dfac, y, z1);
  rs_matvec(m->f_nrows, m->f_rp, m->f_ci, m->f_v, z1, t);
  for (int i = 0; i < ng; ++i) t[i] = y[p + i] - t[i];
  block_solve(m->ns, m->s_ranges, m->sfac, t, z2);
  rs_matvec(m->e_nrows, m->e_rp, m->e_ci, m->e_v, z2, w);
  block_solve(m->nd, m->d_ranges, m->dfac, w, corr);
  for (int i = 0; i < p; ++i) x[i] = z1[i] - corr[i];
  for (int i = 0; i < ng; ++i) x[p + i] = z2[i];
  free(z1); free(t); free(z2); free(w); free(corr);
}

static double norm2(int n, const double *v) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

static double dotp(int n, const double *a, const double *b) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* true_residual: gmres.cpp:26-33. */
static double true_res(int n, const int *rp, const int *ci, const double *v,
                       const double *x, const double *b, double *tmp) {
  rs_matvec(n, rp, ci, v, x, tmp);
  for (int i = 0; i < n; ++i) tmp[i] = b[i] - tmp[i];
  const double bn = norm2(n, b), rn = norm2(n, tmp);
  return bn == 0.0 ? rn : rn / bn;
}

/* Restarted GMRES with MGS + Givens: gmres.cpp:35-191. */
int rs_gmres(int n, const int *rp, const int *ci, const double *v,
             const rs_msc *m, int side, const double *b, int restart,
             int max_iters, double rel_tol, double *x, int *iters,
             int *converged, double *hist, int *nhist) {
  const int cap = *nhist;
  int nh = 0;
#define PUSH(val) do { if (nh < cap) hist[nh] = (val); nh++; } while (0)
  if (restart < 1 || !(rel_tol > 0.0) || max_iters < 1) return -1;
  const int left = m && side == 2, right = m && side == 1;
  for (int i = 0; i < n; ++i) x[i] = 0.0;
  *iters = 0;
  *converged = 0;
  const double norm_b = norm2(n, b);
  if (norm_b == 0.0) {
    *converged = 1;
    PUSH(0.0);
    *nhist = nh;
    return 0;
  }
  double *tmp = xmalloc(sizeof(double) * n);
  double *tmp2 = xmalloc(sizeof(double) * n);
  double denom = norm_b;
  if (left) {
    rs_msc_apply(m, b, tmp);
    denom = norm2(n, tmp);
  }
  if (denom == 0.0) denom = norm_b;
  const int mm = restart;
  double *V = xmalloc(sizeof(double) * (size_t)n * (mm + 1));
  double *H = calloc((size_t)(mm + 1) * mm, sizeof(double));
  double *cs = xmalloc(sizeof(double) * mm), *sn = xmalloc(sizeof(double) * mm);
  double *g = xmalloc(sizeof(double) * (mm + 1));
  double *y = xmalloc(sizeof(double) * mm);
  double *w = xmalloc(sizeof(double) * n);
#define HH(i, j) H[(size_t)(j) * (mm + 1) + (i)]
  double last_true = 1.0, prev_cycle_true = -1.0;
  int done = 0;
  while (!done) {
    double *r = tmp;
    rs_matvec(n, rp, ci, v, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    if (left) {
      rs_msc_apply(m, r, tmp2);
      memcpy(r, tmp2, sizeof(double) * n);
    }
    const double beta = norm2(n, r);
    const double rel0 = beta / denom;
    if (nh == 0) PUSH(rel0);
    if (rel0 <= rel_tol) {
      last_true = true_res(n, rp, ci, v, x, b, tmp2);
      *converged = last_true <= rel_tol;
      break;
    }
    for (int i = 0; i < n; ++i) V[i] = r[i] / beta;
    for (int i = 0; i <= mm; ++i) g[i] = 0.0;
    g[0] = beta;
    int mcount = 0, breakdown = 0, inner_conv = 0;
    for (int j = 0; j < mm && *iters < max_iters; ++j) {
      const double *vj = V + (size_t)j * n;
      if (right) {
        rs_msc_apply(m, vj, tmp2);
        rs_matvec(n, rp, ci, v, tmp2, w);
      } else if (left) {
        rs_matvec(n, rp, ci, v, vj, tmp2);
        rs_msc_apply(m, tmp2, w);
      } else {
        rs_matvec(n, rp, ci, v, vj, w);
      }
      for (int i = 0; i <= j; ++i) {
        const double *vi = V + (size_t)i * n;
        const double hij = dotp(n, vi, w);
        HH(i, j) = hij;
        for (int t = 0; t < n; ++t) w[t] -= hij * vi[t];
      }
      const double hnext = norm2(n, w);
      HH(j + 1, j) = hnext;
      if (hnext >= 1e-14) {
        double *vn = V + (size_t)(j + 1) * n;
        for (int t = 0; t < n; ++t) vn[t] = w[t] / hnext;
      } else {
        breakdown = 1;
      }
      for (int i = 0; i < j; ++i) {
        const double t1 = cs[i] * HH(i, j) + sn[i] * HH(i + 1, j);
        const double t2 = -sn[i] * HH(i, j) + cs[i] * HH(i + 1, j);
        HH(i, j) = t1;
        HH(i + 1, j) = t2;
      }
      const double dr = hypot(HH(j, j), HH(j + 1, j));
      cs[j] = dr == 0.0 ? 1.0 : HH(j, j) / dr;
      sn[j] = dr == 0.0 ? 0.0 : HH(j + 1, j) / dr;
      HH(j, j) = dr;
      HH(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++*iters;
      mcount = j + 1;
      const double rel = fabs(g[j + 1]) / denom;
      PUSH(rel);
      if (breakdown || rel <= rel_tol) {
        inner_conv = rel <= rel_tol;
        break;
      }
    }
    for (int i = mcount - 1; i >= 0; --i) {
      double s = g[i];
      for (int j = i + 1; j < mcount; ++j) s -= HH(i, j) * y[j];
      y[i] = s / HH(i, i);
    }
    double *z = tmp;
    for (int t = 0; t < n; ++t) z[t] = 0.0;
    for (int j = 0; j < mcount; ++j) {
      const double *vj = V + (size_t)j * n;
      for (int t = 0; t < n; ++t) z[t] += y[j] * vj[t];
    }
    if (right) {
      rs_msc_apply(m, z, tmp2);
      memcpy(z, tmp2, sizeof(double) * n);
    }
    for (int t = 0; t < n; ++t) x[t] += z[t];
    last_true = true_res(n, rp, ci, v, x, b, tmp2);
    if (last_true <= rel_tol) {
      *converged = 1;
      done = 1;
    } else if (breakdown) {
      *converged = 0;
      done = 1;
    } else if (*iters >= max_iters) {
      *converged = 0;
      done = 1;
    } else if (inner_conv) {
      if (prev_cycle_true >= 0.0 && last_true >= 0.999 * prev_cycle_true) {
        *converged = 0;
        done = 1;
      }
    }
    prev_cycle_true = last_true;
  }
  PUSH(last_true);
  *nhist = nh;
#undef HH
#undef PUSH
  free(tmp); free(tmp2); free(V); free(H); free(cs); free(sn); free(g);
  free(y); free(w);
  return 0;
}
