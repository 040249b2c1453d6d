// Mini-Schur-complement construction S^ on the device (reference build_msc,
// proj/src/schur_approx.cpp:88-161, numbering aggregates), one CTA per
// aggregate [sb, se) of the interface:
//   LUM:   S_ii = G_ii
//   MSCN:  S_ii = G_ii - F_ii D_ii^-1 E_ii
//   MSCNR: S_ii = G_ii - F_ii D_ii^-1 diag(E_ii 1)
// where for numbering aggregates the D-side set is the same index range
// (D_ii = D[sb:se, sb:se]).  Every step replays the reference's operation
// order with separately rounded multiply / add (no FMA), so S^ is
// bit-identical to the host build and to the reference:
//   dense_lu          dense_matrix.cpp:85-123  (first maximum wins, zero
//                     pivot column -> SingularMatrixError, whole-row swaps)
//   factor_exact      factorization.cpp:11-32  (L / U re-stored sparse: the
//                     solve skips exact zeros)
//   solve (multi-RHS) factorization.cpp:160-199
//   multiply          dense_matrix.cpp:62-77,  subtract  dense_matrix.cpp:55-60
// The LU runs block-wide on an L2-resident dense copy; the multi-RHS solve
// and the correction put one thread on each right-hand-side column.
#include <algorithm>
#include <string>

#include "common.cuh"
#include "internal.hpp"
#include "host/setup.hpp"

namespace mscg {

namespace {

constexpr int kMscThreads = 256;

__global__ void __launch_bounds__(kMscThreads) msc_block_kernel(
    int p, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ cv,
    const int* __restrict__ ranges, int variant, const long long* __restrict__ soff,
    double* __restrict__ scratch, int* __restrict__ perm_all, unsigned long long* err,
    int* __restrict__ row_nnz, const int* __restrict__ roff) {
  const int agg = blockIdx.x;
  const int sb = ranges[2 * agg], se = ranges[2 * agg + 1], m = se - sb;
  // per-aggregate row storage (perm, row counts): spans of overlapped
  // aggregates share rows, so each aggregate has its own slice
  const int r0 = roff[agg];
  const long long mm = static_cast<long long>(m) * m;
  const bool lum = variant == kMscLum;
  double* S = scratch + soff[agg];
  double* A = S + mm;   // D_ii, then its LU
  double* B = A + mm;   // right-hand sides (E_ii or diag(E_ii 1))
  double* X = B + mm;   // D_ii^-1 B
  int* perm = perm_all + r0;
  const int tid = threadIdx.x;
  __shared__ double red_v[kMscThreads / 32];
  __shared__ int red_i[kMscThreads / 32];
  __shared__ int s_piv;
  __shared__ double s_best;

  for (long long t = tid; t < (lum ? mm : 3 * mm); t += blockDim.x) S[t] = 0.0;
  __syncthreads();
  // S = G_ii; A = D_ii; B = E_ii (MSCN) or diag(E_ii 1) (MSCNR)
  for (int r = tid; r < m; r += blockDim.x) {
    for (int k = rp[p + sb + r]; k < rp[p + sb + r + 1]; ++k) {
      const int c = ci[k] - (p + sb);
      if (c >= 0 && c < m) S[static_cast<long long>(r) * m + c] = cv[k];
    }
    if (lum) continue;
    perm[r] = r;
    double rowsum = 0.0;
    for (int k = rp[sb + r]; k < rp[sb + r + 1]; ++k) {
      const int c = ci[k];
      if (c >= sb && c < se) A[static_cast<long long>(r) * m + (c - sb)] = cv[k];
      if (c >= p + sb && c < p + se) {
        if (variant == kMscMscn)
          B[static_cast<long long>(r) * m + (c - p - sb)] = cv[k];
        else  // matvec(e_ii, ones): row order, v * 1.0
          rowsum = __dadd_rn(rowsum, __dmul_rn(cv[k], 1.0));
      }
    }
    if (variant == kMscMscnr) B[static_cast<long long>(r) * m + r] = rowsum;
  }
  __syncthreads();

  if (!lum) {
    // ---- dense_lu(D_ii) with partial pivoting
    for (int k = 0; k < m; ++k) {
      double bv = -1.0;
      int bi = m;
      for (int i = k + tid; i < m; i += blockDim.x) {
        const double v = fabs(A[static_cast<long long>(i) * m + k]);
        if (v > bv) {
          bv = v;
          bi = i;
        }
      }
      for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, bv, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if ((tid & 31) == 0) {
        red_v[tid >> 5] = bv;
        red_i[tid >> 5] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double v = red_v[0];
        int idx = red_i[0];
        for (int w = 1; w < kMscThreads / 32; ++w)
          if (red_v[w] > v || (red_v[w] == v && red_i[w] < idx)) {
            v = red_v[w];
            idx = red_i[w];
          }
        s_best = v;
        s_piv = idx;
      }
      __syncthreads();
      if (s_piv < m && s_best == 0.0) {  // exactly zero pivot column
        if (tid == 0)
          atomicMin(err, (static_cast<unsigned long long>(agg) << 32) | static_cast<unsigned>(k));
        return;
      }
      const int piv = s_piv < m ? s_piv : k;  // all-NaN column: keep k
      if (piv != k) {
        for (int j = tid; j < m; j += blockDim.x) {
          const double t1 = A[static_cast<long long>(k) * m + j];
          A[static_cast<long long>(k) * m + j] = A[static_cast<long long>(piv) * m + j];
          A[static_cast<long long>(piv) * m + j] = t1;
        }
        if (tid == 0) {
          const int t2 = perm[k];
          perm[k] = perm[piv];
          perm[piv] = t2;
        }
      }
      __syncthreads();
      const double pivot = A[static_cast<long long>(k) * m + k];
      for (int i = k + 1 + tid; i < m; i += blockDim.x) {
        double* ai = A + static_cast<long long>(i) * m;
        ai[k] = __ddiv_rn(ai[k], pivot);
      }
      __syncthreads();
      const int w = m - k - 1;
      const long long work = static_cast<long long>(w) * w;
      for (long long t = tid; t < work; t += blockDim.x) {
        const int i = k + 1 + static_cast<int>(t / w);
        const int j = k + 1 + static_cast<int>(t % w);
        const double lik = A[static_cast<long long>(i) * m + k];
        if (lik != 0.0) {
          double* aij = A + static_cast<long long>(i) * m + j;
          *aij = __dsub_rn(*aij, __dmul_rn(lik, A[static_cast<long long>(k) * m + j]));
        }
      }
      __syncthreads();
    }
    // ---- X = solve(LU, B): one thread per right-hand-side column
    for (int j = tid; j < m; j += blockDim.x) {
      for (int i = 0; i < m; ++i)
        X[static_cast<long long>(i) * m + j] = B[static_cast<long long>(perm[i]) * m + j];
      for (int i = 0; i < m; ++i) {
        const double* li = A + static_cast<long long>(i) * m;
        double xi = X[static_cast<long long>(i) * m + j];
        for (int c = 0; c < i; ++c) {
          const double lik = li[c];
          if (lik != 0.0) xi = __dsub_rn(xi, __dmul_rn(lik, X[static_cast<long long>(c) * m + j]));
        }
        X[static_cast<long long>(i) * m + j] = xi;
      }
      for (int i = m - 1; i >= 0; --i) {
        const double* ui = A + static_cast<long long>(i) * m;
        double xi = X[static_cast<long long>(i) * m + j];
        for (int c = i + 1; c < m; ++c) {
          const double uik = ui[c];
          if (uik != 0.0) xi = __dsub_rn(xi, __dmul_rn(uik, X[static_cast<long long>(c) * m + j]));
        }
        X[static_cast<long long>(i) * m + j] = __ddiv_rn(xi, ui[i]);
      }
    }
    __syncthreads();
    // ---- S -= F_ii X (multiply: row order from 0.0, then subtract)
    for (int j = tid; j < m; j += blockDim.x)
      for (int r = 0; r < m; ++r) {
        double corr = 0.0;
        for (int k = rp[p + sb + r]; k < rp[p + sb + r + 1]; ++k) {
          const int c = ci[k];
          if (c >= sb && c < se)
            corr = __dadd_rn(corr, __dmul_rn(cv[k], X[static_cast<long long>(c - sb) * m + j]));
        }
        double* s = S + static_cast<long long>(r) * m + j;
        *s = __dsub_rn(*s, corr);
      }
    __syncthreads();
  }
  for (int r = tid; r < m; r += blockDim.x) {
    int cnt = 0;
    for (int c = 0; c < m; ++c) cnt += S[static_cast<long long>(r) * m + c] != 0.0;
    row_nnz[r0 + r] = cnt;
  }
}

// The block-diagonal S^ CSR: row sb + r holds the nonzeros of S_ii row r
// in column order (the reference's merge, schur_approx.cpp:141-160).
__global__ void __launch_bounds__(kMscThreads) msc_fill_kernel(
    const int* __restrict__ ranges, const long long* __restrict__ soff,
    const double* __restrict__ scratch, const int* __restrict__ srp, int* __restrict__ sci,
    double* __restrict__ sv) {
  const int agg = blockIdx.x;
  const int sb = ranges[2 * agg], se = ranges[2 * agg + 1], m = se - sb;
  const double* S = scratch + soff[agg];
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    int o = srp[sb + r];
    for (int c = 0; c < m; ++c) {
      const double v = S[static_cast<long long>(r) * m + c];
      if (v != 0.0) {
        sci[o] = sb + c;
        sv[o] = v;
        ++o;
      }
    }
  }
}

}  // namespace

void build_msc_device(Ctx* ctx, int n, int p, const int* c_rp, const int* c_ci, const double* c_v,
                      const std::vector<std::pair<int, int>>& ranges,
                      const std::vector<std::pair<int, int>>& spans, int variant,
                      std::vector<int>& s_rp, std::vector<int>& s_ci, std::vector<double>& s_v) {
  cudaStream_t s = ctx->stream;
  const int k = static_cast<int>(ranges.size());
  const int ng = n - p;
  const bool overlapped = spans != ranges;
  s_rp.assign(ng + 1, 0);
  s_ci.clear();
  s_v.clear();
  if (k == 0) return;
  const int64_t nnz = c_rp[n];
  // each CTA works on its aggregate's span (= its owned range unless the
  // aggregates overlap)
  std::vector<int> hr(2 * k), hro(k + 1, 0);
  std::vector<long long> hoff(k + 1, 0);
  for (int i = 0; i < k; ++i) {
    hr[2 * i] = spans[i].first;
    hr[2 * i + 1] = spans[i].second;
    const long long m = spans[i].second - spans[i].first;
    hoff[i + 1] = hoff[i] + (variant == kMscLum ? 1 : 4) * m * m;
    hro[i + 1] = hro[i] + static_cast<int>(m);
  }
  if (!overlapped)
    for (int i = 0; i < k; ++i) hro[i] = ranges[i].first;  // = the running sum
  DevBuf d_rp(sizeof(int) * (n + 1)), d_ci(sizeof(int) * std::max<int64_t>(1, nnz)),
      d_v(sizeof(double) * std::max<int64_t>(1, nnz));
  MSCG_CUDA(cudaMemcpyAsync(d_rp.p, c_rp, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s));
  if (nnz) {
    MSCG_CUDA(cudaMemcpyAsync(d_ci.p, c_ci, sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
    MSCG_CUDA(cudaMemcpyAsync(d_v.p, c_v, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
  }
  DevBuf d_r(sizeof(int) * hr.size()), d_off(sizeof(long long) * hoff.size()),
      d_ro(sizeof(int) * hro.size());
  MSCG_CUDA(cudaMemcpyAsync(d_r.p, hr.data(), sizeof(int) * hr.size(), cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaMemcpyAsync(d_off.p, hoff.data(), sizeof(long long) * hoff.size(),
                            cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaMemcpyAsync(d_ro.p, hro.data(), sizeof(int) * hro.size(), cudaMemcpyHostToDevice, s));
  const int rows_total = std::max(ng, hro[k]);
  DevBuf scratch(sizeof(double) * std::max<long long>(1, hoff[k]));
  DevBuf perm(sizeof(int) * std::max(1, rows_total)), nnzr(sizeof(int) * std::max(1, rows_total));
  DevBuf err(sizeof(unsigned long long));
  const unsigned long long none = ~0ull;
  MSCG_CUDA(cudaMemcpyAsync(err.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
  msc_block_kernel<<<k, kMscThreads, 0, s>>>(p, d_rp.as<int>(), d_ci.as<int>(), d_v.as<double>(),
                                             d_r.as<int>(), variant, d_off.as<long long>(),
                                             scratch.as<double>(), perm.as<int>(),
                                             err.as<unsigned long long>(), nnzr.as<int>(),
                                             d_ro.as<int>());
  MSCG_CUDA(cudaGetLastError());
  ctx->launches++;
  unsigned long long herr = none;
  std::vector<int> hn(ng);
  MSCG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(herr), cudaMemcpyDeviceToHost, s));
  if (ng && !overlapped)
    MSCG_CUDA(cudaMemcpyAsync(hn.data(), nnzr.p, sizeof(int) * ng, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  if (herr != none) {
    const int agg = static_cast<int>(herr >> 32), piv = static_cast<int>(herr & 0xffffffffu);
    throw Error(2, "build_msc: singular D block of aggregate " + std::to_string(agg) +
                       " (dense_lu: zero pivot at index " + std::to_string(piv) + ")",
                -1, piv);
  }
  if (overlapped) {
    // banded S^: the local blocks come back and are merged in the
    // reference's order (owned columns over whole spans, host::merge_msc)
    std::vector<std::vector<double>> loc(k);
    std::vector<const double*> lp(k);
    for (int i = 0; i < k; ++i) {
      const size_t m = spans[i].second - spans[i].first;
      loc[i].resize(m * m);
      MSCG_CUDA(cudaMemcpyAsync(loc[i].data(), scratch.as<double>() + hoff[i], sizeof(double) * m * m,
                                cudaMemcpyDeviceToHost, s));
      lp[i] = loc[i].data();
    }
    MSCG_CUDA(cudaStreamSynchronize(s));
    host::Csr out = host::merge_msc(ng, ranges, spans, lp);
    s_rp = std::move(out.rp);
    s_ci = std::move(out.ci);
    s_v = std::move(out.v);
    return;
  }
  for (int r = 0; r < ng; ++r) s_rp[r + 1] = s_rp[r] + hn[r];
  const int snnz = s_rp[ng];
  DevBuf d_srp(sizeof(int) * (ng + 1)), d_sci(sizeof(int) * std::max(1, snnz)),
      d_sv(sizeof(double) * std::max(1, snnz));
  MSCG_CUDA(cudaMemcpyAsync(d_srp.p, s_rp.data(), sizeof(int) * (ng + 1), cudaMemcpyHostToDevice, s));
  msc_fill_kernel<<<k, kMscThreads, 0, s>>>(d_r.as<int>(), d_off.as<long long>(),
                                            scratch.as<double>(), d_srp.as<int>(), d_sci.as<int>(),
                                            d_sv.as<double>());
  MSCG_CUDA(cudaGetLastError());
  ctx->launches++;
  s_ci.resize(snnz);
  s_v.resize(snnz);
  if (snnz) {
    MSCG_CUDA(cudaMemcpyAsync(s_ci.data(), d_sci.p, sizeof(int) * snnz, cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaMemcpyAsync(s_v.data(), d_sv.p, sizeof(double) * snnz, cudaMemcpyDeviceToHost, s));
  }
  MSCG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mscg
