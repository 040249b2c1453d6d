// SpMV y = A x for C, E and F (reference matvec, sparse_matrix.cpp:110-125).
//
// Layout: SELL-32 (sigma = 1): 32 consecutive rows form a slice stored
// column-major, so lane r of a warp owns row r of the slice and the warp
// reads 32 consecutive (value, column) pairs per step — fully coalesced
// 256 B + 128 B transactions.  Each lane accumulates its row in the
// reference's order with separately rounded multiply and add
// (__dmul_rn/__dadd_rn, no FMA contraction), so y is bit-identical to the
// reference's x86 result.  Roofline: HBM, 12 B/nnz + 8 B/row (x gathers hit
// L2: x is <= 100 MB at cfg5).
#include <algorithm>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

// Rows [row_lo, row_hi) are written; slices from row_lo / 32 are walked
// (a slice straddling the range computes rows it does not write).
__global__ void __launch_bounds__(256) sell_spmv_kernel(
    int row_lo, int row_hi, int nslices, const int64_t* __restrict__ sptr,
    const int* __restrict__ swidth, const int* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ x,
    double* __restrict__ y, const double* base, int mode) {
  const int slice = (row_lo >> 5) + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (slice >= nslices) return;
  const int row = slice * 32 + lane;
  const int64_t p0 = sptr[slice] + lane;
  const int w = swidth[slice];
  double acc = 0.0;
#pragma unroll 4
  for (int k = 0; k < w; ++k) {
    const int c = __ldg(col + p0 + 32 * k);
    const double v = __ldg(val + p0 + 32 * k);
    if (c >= 0) acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + c)));
  }
  if (row >= row_lo && row < row_hi)
    y[row] = mode == 0 ? acc : (mode == 1 ? __dsub_rn(base[row], acc) : __dadd_rn(base[row], acc));
}

}  // namespace

std::unique_ptr<DevCsr> upload_csr(Ctx* ctx, int nrows, int ncols, const int* rp,
                                   const int* ci, const double* v) {
  auto a = std::make_unique<DevCsr>();
  a->ctx = ctx;
  a->nrows = nrows;
  a->ncols = ncols;
  a->nnz = rp[nrows];
  a->nslices = (nrows + 31) / 32;
  std::vector<int64_t> sptr(a->nslices + 1, 0);
  std::vector<int> swidth(a->nslices, 0);
  for (int s = 0; s < a->nslices; ++s) {
    int w = 0;
    for (int r = s * 32; r < std::min(nrows, s * 32 + 32); ++r) w = std::max(w, rp[r + 1] - rp[r]);
    swidth[s] = w;
    sptr[s + 1] = sptr[s] + 32LL * w;
  }
  a->padded = sptr[a->nslices];
  std::vector<int> hcol(std::max<int64_t>(1, a->padded), -1);
  std::vector<double> hval(std::max<int64_t>(1, a->padded), 0.0);
  for (int s = 0; s < a->nslices; ++s)
    for (int r = s * 32; r < std::min(nrows, s * 32 + 32); ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) {
        const int64_t pos = sptr[s] + 32LL * (k - rp[r]) + (r - s * 32);
        hcol[pos] = ci[k];
        hval[pos] = v[k];
      }
  a->slice_ptr = DevBuf(sizeof(int64_t) * sptr.size());
  a->slice_width = DevBuf(sizeof(int) * std::max<size_t>(1, swidth.size()));
  a->col = DevBuf(sizeof(int) * hcol.size());
  a->val = DevBuf(sizeof(double) * hval.size());
  cudaStream_t s = ctx->stream;
  MSCG_CUDA(cudaMemcpyAsync(a->slice_ptr.p, sptr.data(), a->slice_ptr.bytes, cudaMemcpyHostToDevice, s));
  if (!swidth.empty())
    MSCG_CUDA(cudaMemcpyAsync(a->slice_width.p, swidth.data(), sizeof(int) * swidth.size(),
                              cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaMemcpyAsync(a->col.p, hcol.data(), a->col.bytes, cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaMemcpyAsync(a->val.p, hval.data(), a->val.bytes, cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  return a;
}

void spmv_rows(const DevCsr& a, const double* x, double* y, const double* base, int mode,
               int row_lo, int row_hi, cudaStream_t s) {
  if (a.nslices == 0 || row_hi <= row_lo) return;
  const int threads = 256;
  const int nsl = ((row_hi + 31) >> 5) - (row_lo >> 5);
  const int blocks = (nsl * 32 + threads - 1) / threads;
  sell_spmv_kernel<<<blocks, threads, 0, s>>>(row_lo, row_hi, a.nslices, a.slice_ptr.as<int64_t>(),
                                              a.slice_width.as<int>(), a.col.as<int>(),
                                              a.val.as<double>(), x, y, base, mode);
  MSCG_CUDA(cudaGetLastError());
  a.ctx->launches++;
}

void spmv(const DevCsr& a, const double* x, double* y, const double* base, int mode,
          cudaStream_t s) {
  spmv_rows(a, x, y, base, mode, 0, a.nrows, s);
}

}  // namespace mscg
