// Explicit interior correction W = D^-1 E (second half of
// MscPreconditioner::apply, proj/src/preconditioner.cpp:105-111).
//
// The reference finishes an apply with w = E z2 and x1 = z1 - D^-1 w: a
// second full pass of the interior-block triangular solves, i.e. a second
// stream of every ILUT factor (>45 % of an apply's bytes) through the
// latency-bound tile chain.  E couples a block only to the interface
// unknowns on its boundary (k_b ≈ 210 columns for a 32x32-cell block of
// ~3100 rows), so the block's D_b^-1 E_b is a dense dim_b x k_b panel that
// is smaller than the block's factors (cfg5: 20 GB against 40 GB of factor
// stream) and is applied as a streaming GEMV with no dependency chain:
//
//   x1_b = z1_b - W_b z2[cols_b],   W_b = U_b^-1 L_b^-1 E_b[:, cols_b]
//
// Mathematically identical to the reference; rounding differs at the level
// of the solve's own (≈1e-15 relative, tests check 1e-10 against the
// reference apply).  W is built once at setup with the same trisolve_kernel
// the apply uses: launch k solves column k of every block with k_b > k
// (blocks sorted by k_b, so the launch is a prefix of that order).
//
// Layout: per block, W_b column-major (column k = dim_b consecutive fp64),
// blocks back to back; cols_b ascending interface columns (int32).  A work
// item is (block, 512-row slice; 256 or 128 when there are too few blocks to
// fill the GPU; 64 rows split four ways over k — correct_split_kernel —
// when even 128 leaves fewer than 4 items per SM, cfg2 22 -> 16 us); a CTA
// of 256 threads owns one item, stages
// z2[cols_b] in shared memory and each thread accumulates rows i and i+256
// over k in ascending order (one fma per entry, deterministic).  Roofline:
// HBM, 8 B per W entry (read once per apply, streaming loads so W does not
// evict the vectors from L2) + 24 B per row (z1 in, x1 out, W column reuse
// of z2 from shared memory).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include <cstdio>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kCorrThreads = 256;
constexpr int kCorrSlice = 2 * kCorrThreads;

// Rows wa (and wb) of a panel with leading dimension d, summed over k in
// ascending order; loads are issued kBatch columns at a time so that every
// thread keeps kBatch (2 kBatch) streaming loads in flight.
template <bool kTwo>
__device__ __forceinline__ void corr_rows(const double* __restrict__ wa,
                                          const double* __restrict__ wb, int d, int kb,
                                          const double* zs, double& a0, double& a1) {
  constexpr int kBatch = 8;
  int k = 0;
  for (; k + kBatch <= kb; k += kBatch) {
    double va[kBatch], vb[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      va[j] = __ldcs(wa + static_cast<size_t>(k + j) * d);
      if (kTwo) vb[j] = __ldcs(wb + static_cast<size_t>(k + j) * d);
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const double z = zs[k + j];
      a0 = fma(va[j], z, a0);
      if (kTwo) a1 = fma(vb[j], z, a1);
    }
  }
  for (; k < kb; ++k) {
    const double z = zs[k];
    a0 = fma(__ldcs(wa + static_cast<size_t>(k) * d), z, a0);
    if (kTwo) a1 = fma(__ldcs(wb + static_cast<size_t>(k) * d), z, a1);
  }
}

__global__ void __launch_bounds__(kCorrThreads) correct_kernel(
    const int2* __restrict__ items, int item0, const int* __restrict__ row0,
    const int* __restrict__ dim, const long long* __restrict__ woff,
    const int* __restrict__ wcoff, const int* __restrict__ wcols,
    const double* __restrict__ W, const double* __restrict__ x2,
    const double* __restrict__ z1, double* __restrict__ out, int slice) {
  extern __shared__ double zs[];
  const int2 it = items[item0 + blockIdx.x];
  const int b = it.x, i0 = it.y;
  const int c0 = wcoff[b], kb = wcoff[b + 1] - c0;
  for (int k = threadIdx.x; k < kb; k += kCorrThreads) zs[k] = __ldg(x2 + __ldg(wcols + c0 + k));
  __syncthreads();
  const int r0 = row0[b];
  const int d = dim[b], de = min(d, i0 + slice);  // rows [i0, de) of this item
  if (static_cast<int>(threadIdx.x) >= slice) return;
  const int ia = i0 + threadIdx.x, ib = ia + kCorrThreads;
  // rows past the block read a valid row (clamped, same sectors as their
  // neighbours) and are not written; the second row is walked only by warps
  // that own at least one of them, so the branch is warp-uniform
  const double* wbase = W + woff[b];
  const double* wa = wbase + min(ia, d - 1);
  const double* wb = wbase + min(ib, d - 1);
  double a0 = 0.0, a1 = 0.0;
  if (i0 + kCorrThreads + static_cast<int>(threadIdx.x & ~31u) < de)
    corr_rows<true>(wa, wb, d, kb, zs, a0, a1);
  else
    corr_rows<false>(wa, wb, d, kb, zs, a0, a1);
  if (ia < de) out[r0 + ia] = __dsub_rn(z1[r0 + ia], a0);
  if (ib < de) out[r0 + ib] = __dsub_rn(z1[r0 + ib], a1);
}

// Few rows (cfg1 / cfg2): one row per kSplit threads, each summing a
// contiguous quarter of the columns (ascending), the quarters then added in
// order — deterministic; kSplit times the loads in flight of the one-thread
// rows, whose k_b-long chains left the GPU latency-bound (cfg2 22 us).
constexpr int kSplit = 4;
constexpr int kSplitRows = kCorrThreads / kSplit;  // rows per CTA

__global__ void __launch_bounds__(kCorrThreads) correct_split_kernel(
    const int2* __restrict__ items, int item0, const int* __restrict__ row0,
    const int* __restrict__ dim, const long long* __restrict__ woff,
    const int* __restrict__ wcoff, const int* __restrict__ wcols,
    const double* __restrict__ W, const double* __restrict__ x2,
    const double* __restrict__ z1, double* __restrict__ out) {
  extern __shared__ double zs[];
  __shared__ double part[kSplit][kSplitRows];
  const int2 it = items[item0 + blockIdx.x];
  const int b = it.x, i0 = it.y;
  const int c0 = wcoff[b], kb = wcoff[b + 1] - c0;
  for (int k = threadIdx.x; k < kb; k += kCorrThreads) zs[k] = __ldg(x2 + __ldg(wcols + c0 + k));
  __syncthreads();
  const int d = dim[b];
  const int r = threadIdx.x % kSplitRows, q = threadIdx.x / kSplitRows;  // row, quarter
  const int i = i0 + r;
  const int k0 = kb * q / kSplit, k1 = kb * (q + 1) / kSplit;
  const double* wr = W + woff[b] + min(i, d - 1);
  double a = 0.0, a2 = 0.0;
  int k = k0;
  for (; k + 8 <= k1; k += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(wr + static_cast<size_t>(k + j) * d);
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      a = fma(v[j], zs[k + j], a);
      a2 = fma(v[j + 1], zs[k + j + 1], a2);
    }
  }
  for (; k < k1; ++k) a = fma(__ldcs(wr + static_cast<size_t>(k) * d), zs[k], a);
  part[q][r] = a + a2;
  __syncthreads();
  if (q == 0 && i < d && i < i0 + kSplitRows) {
    double t = part[0][r];
#pragma unroll
    for (int qq = 1; qq < kSplit; ++qq) t += part[qq][r];
    const int r0 = row0[b];
    out[r0 + i] = __dsub_rn(z1[r0 + i], t);
  }
}

// Setup: r[row0_b + rows of column k of E_b] = values (or 0 when clearing).
__global__ void corr_scatter_kernel(const int* __restrict__ order, int k,
                                    const int* __restrict__ row0, const int* __restrict__ wcoff,
                                    const int* __restrict__ ecp, const int* __restrict__ erow,
                                    const double* __restrict__ eval, double* __restrict__ r,
                                    int clear) {
  const int b = order[blockIdx.x];
  const int c = wcoff[b] + k;
  const int r0 = row0[b];
  for (int e = ecp[c] + threadIdx.x; e < ecp[c + 1]; e += blockDim.x)
    r[r0 + erow[e]] = clear ? 0.0 : eval[e];
}

// Setup: W_b[:, k] = o[row0_b .. row0_b + dim_b).
__global__ void corr_gather_kernel(const int* __restrict__ order, int k,
                                   const int* __restrict__ row0, const int* __restrict__ dim,
                                   const long long* __restrict__ woff,
                                   const double* __restrict__ o, double* __restrict__ W) {
  const int b = order[blockIdx.x];
  const int d = dim[b], r0 = row0[b];
  double* col = W + woff[b] + static_cast<size_t>(k) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) col[i] = o[r0 + i];
}

template <class T>
DevBuf upload(const std::vector<T>& h, cudaStream_t s) {
  DevBuf d(sizeof(T) * std::max<size_t>(1, h.size()));
  if (!h.empty()) MSCG_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(),
                                            cudaMemcpyHostToDevice, s));
  return d;
}

}  // namespace

int correction_mode_default() {
  static const int m = [] {
    const char* e = getenv("MSCG_CORRECTION");
    if (!e) return kCorrAuto;
    if (!strcmp(e, "off") || !strcmp(e, "0")) return kCorrOff;
    if (!strcmp(e, "on") || !strcmp(e, "1")) return kCorrOn;
    return kCorrAuto;
  }();
  return m;
}

std::unique_ptr<Correction> build_correction(Ctx* ctx, const FactorSet& D, const int* e_rp,
                                             const int* e_ci, const double* e_v, int mode,
                                             double* r_scratch, double* o_scratch) {
  if (mode == kCorrOff || D.nblocks == 0) return nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  const int nb = D.nblocks;
  auto c = std::make_unique<Correction>();
  c->nblocks = nb;
  // interface columns of each block (ascending) and E_b by column
  std::vector<int> wcoff(nb + 1, 0), wcols, ecp(1, 0), erow;
  std::vector<double> eval;
  std::vector<long long> woff(nb + 1, 0);
  std::vector<int> kb(nb);
  {
    std::vector<std::vector<std::pair<int, double>>> bycol;
    for (int b = 0; b < nb; ++b) {
      const int r0 = D.h_row0[b], d = D.h_dim[b];
      std::vector<int> cols;
      for (int i = r0; i < r0 + d; ++i)
        for (int e = e_rp[i]; e < e_rp[i + 1]; ++e) cols.push_back(e_ci[e]);
      std::sort(cols.begin(), cols.end());
      cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
      kb[b] = static_cast<int>(cols.size());
      bycol.assign(cols.size(), {});
      for (int i = r0; i < r0 + d; ++i)
        for (int e = e_rp[i]; e < e_rp[i + 1]; ++e) {
          const int k = static_cast<int>(std::lower_bound(cols.begin(), cols.end(), e_ci[e]) -
                                         cols.begin());
          bycol[k].push_back({i - r0, e_v[e]});
        }
      for (size_t k = 0; k < cols.size(); ++k) {
        wcols.push_back(cols[k]);
        for (auto [row, v] : bycol[k]) {
          erow.push_back(row);
          eval.push_back(v);
        }
        ecp.push_back(static_cast<int>(erow.size()));
      }
      wcoff[b + 1] = wcoff[b] + kb[b];
      woff[b + 1] = woff[b] + static_cast<long long>(d) * kb[b];
      c->kmax = std::max(c->kmax, kb[b]);
    }
  }
  c->entries = woff[nb];
  const int64_t w_bytes = 8 * c->entries;
  if (static_cast<size_t>(c->kmax) * 8 > 200 * 1024) {
    if (mode == kCorrOn)
      throw Error(1, "build_preconditioner: interior correction needs more than 200 KB of "
                     "interface values per block");
    return nullptr;
  }
  if (mode == kCorrAuto) {
    // decided by the byte counts alone: worth it when the panels move fewer
    // bytes than a pass over the factors (12 B per stored entry incl. the U
    // diagonal).  Free memory is only an out-of-memory guard, and a skip for
    // that reason is logged (the apply path, and so its rounding, is then
    // the reference's two interior passes; mscg_precond_correction reports
    // which path a preconditioner uses).
    const int64_t factor_bytes = 12 * (D.nnz_l() + D.nnz_u() + D.total_rows);
    if (w_bytes > factor_bytes) return nullptr;
    size_t free_b = 0, total_b = 0;
    MSCG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (static_cast<size_t>(w_bytes) + (size_t(4) << 30) > free_b) {
      fprintf(stderr,
              "mscg: interior correction skipped: its %.2f GB of panels do not fit in %.2f GB "
              "of free device memory (applies use the two interior passes)\n",
              w_bytes / 1e9, free_b / 1e9);
      return nullptr;
    }
  }
  cudaStream_t s = ctx->stream;
  c->row0 = D.row0.as<int>();
  c->dim = D.dim.as<int>();
  c->woff = upload(woff, s);
  c->wcoff = upload(wcoff, s);
  c->wcols = upload(wcols, s);
  c->wval = DevBuf(sizeof(double) * std::max<int64_t>(1, c->entries));
  // work items (block, slice) in block order; chunk c = blocks h_chunk[c]..
  // slices of 512 rows (two per thread); fewer blocks than fill the GPU
  // (cfg1/cfg2) get slices of 256 or 128 rows so every SM has items
  int sms = 148, dev = 0;
  MSCG_CUDA(cudaGetDevice(&dev));
  MSCG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  c->slice = kCorrSlice;
  while (c->slice > 128 && static_cast<int64_t>(D.total_rows) / c->slice < 4 * sms) c->slice /= 2;
  // still too few items for the GPU: rows of kSplit threads (MSCG_CORR_SPLIT=0|1)
  {
    const char* e = getenv("MSCG_CORR_SPLIT");
    c->split = e ? e[0] == '1' : static_cast<int64_t>(D.total_rows) / c->slice < 4 * sms;
    if (c->split) c->slice = kSplitRows;
  }
  std::vector<int2> items;
  c->h_item_chunk.assign(kSolveChunks + 1, 0);
  for (int ch = 0; ch < kSolveChunks; ++ch) {
    c->h_item_chunk[ch] = static_cast<int>(items.size());
    for (int b = D.h_chunk[ch]; b < D.h_chunk[ch + 1]; ++b)
      for (int i = 0; i < D.h_dim[b]; i += c->slice) items.push_back(make_int2(b, i));
  }
  c->h_item_chunk[kSolveChunks] = static_cast<int>(items.size());
  c->items = upload(items, s);
  {
    // build: launch k solves column k of the blocks with k_b > k
    std::vector<int> order(nb);
    for (int b = 0; b < nb; ++b) order[b] = b;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return kb[a] > kb[b]; });
    DevBuf d_order = upload(order, s);
    DevBuf d_ecp = upload(ecp, s), d_erow = upload(erow, s), d_eval = upload(eval, s);
    MSCG_CUDA(cudaMemsetAsync(r_scratch, 0, sizeof(double) * D.total_rows, s));
    int npos = nb;
    for (int k = 0; k < c->kmax; ++k) {
      while (npos > 0 && kb[order[npos - 1]] <= k) --npos;
      corr_scatter_kernel<<<npos, 32, 0, s>>>(d_order.as<int>(), k, c->row0, c->wcoff.as<int>(),
                                              d_ecp.as<int>(), d_erow.as<int>(),
                                              d_eval.as<double>(), r_scratch, 0);
      MSCG_CUDA(cudaGetLastError());
      block_trisolve(D, r_scratch, o_scratch, nullptr, s, nullptr, -1, d_order.as<int>(), npos);
      corr_gather_kernel<<<npos, 256, 0, s>>>(d_order.as<int>(), k, c->row0, c->dim,
                                              c->woff.as<long long>(), o_scratch,
                                              c->wval.as<double>());
      MSCG_CUDA(cudaGetLastError());
      corr_scatter_kernel<<<npos, 32, 0, s>>>(d_order.as<int>(), k, c->row0, c->wcoff.as<int>(),
                                              d_ecp.as<int>(), d_erow.as<int>(),
                                              d_eval.as<double>(), r_scratch, 1);
      MSCG_CUDA(cudaGetLastError());
    }
    MSCG_CUDA(cudaStreamSynchronize(s));
  }
  c->build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return c;
}

void apply_correction(const Correction& c, const double* x2, const double* z1, double* out,
                      int chunk, cudaStream_t s) {
  const int i0 = chunk < 0 ? 0 : c.h_item_chunk[chunk];
  const int i1 = chunk < 0 ? c.h_item_chunk[kSolveChunks] : c.h_item_chunk[chunk + 1];
  if (i1 <= i0) return;
  const size_t smem = sizeof(double) * std::max(1, c.kmax);
  if (c.split) {
    ensure_smem(reinterpret_cast<const void*>(correct_split_kernel), smem);
    correct_split_kernel<<<i1 - i0, kCorrThreads, smem, s>>>(
        c.items.as<int2>(), i0, c.row0, c.dim, c.woff.as<long long>(), c.wcoff.as<int>(),
        c.wcols.as<int>(), c.wval.as<double>(), x2, z1, out);
  } else {
    ensure_smem(reinterpret_cast<const void*>(correct_kernel), smem);
    correct_kernel<<<i1 - i0, kCorrThreads, smem, s>>>(
        c.items.as<int2>(), i0, c.row0, c.dim, c.woff.as<long long>(), c.wcoff.as<int>(),
        c.wcols.as<int>(), c.wval.as<double>(), x2, z1, out, c.slice);
  }
  MSCG_CUDA(cudaGetLastError());
}

}  // namespace mscg
