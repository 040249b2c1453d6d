// SpMV y = A x for C, E and F (reference matvec, sparse_matrix.cpp:110-125).
//
// Layout: SELL-64 (sigma = 1): 64 consecutive rows form a slice stored
// column-major, and lane r of a warp owns rows 2r and 2r + 1 of the slice,
// so entry k of both rows is one 16-byte load (double2) with its two columns
// one 8-byte load (int2): a warp reads 512 B of values + 256 B of columns per
// step, fully coalesced, 128-bit vectorised.  Each row is accumulated in the
// reference's order with separately rounded multiply and add
// (__dmul_rn/__dadd_rn, no FMA contraction), so y is bit-identical to the
// reference's x86 result.  Roofline: HBM, 12 B/nnz + 8 B/row (x gathers hit
// L2: x is <= 100 MB at cfg5).
#include <algorithm>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kSlice = 64;

// Rows [row_lo, row_hi) are written; slices from row_lo / 64 are walked
// (a slice straddling the range computes rows it does not write).
__global__ void __launch_bounds__(256) sell_spmv_kernel(
    int row_lo, int row_hi, int nslices, const int64_t* __restrict__ sptr,
    const int* __restrict__ swidth, const int* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ x,
    double* __restrict__ y, const double* base, int mode) {
  const int slice = (row_lo / kSlice) + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (slice >= nslices) return;
  const int row = slice * kSlice + 2 * lane;
  // sptr is a multiple of 64 entries: the pair loads are 16 / 8-byte aligned
  const double2* v2 = reinterpret_cast<const double2*>(val + sptr[slice]) + lane;
  const int2* c2 = reinterpret_cast<const int2*>(col + sptr[slice]) + lane;
  const int w = swidth[slice];
  double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
  for (int k = 0; k < w; ++k) {
    const int2 c = __ldg(c2 + 32 * k);
    const double2 v = __ldg(v2 + 32 * k);
    if (c.x >= 0) a0 = __dadd_rn(a0, __dmul_rn(v.x, __ldg(x + c.x)));
    if (c.y >= 0) a1 = __dadd_rn(a1, __dmul_rn(v.y, __ldg(x + c.y)));
  }
  auto put = [&](int r, double acc) {
    if (r >= row_lo && r < row_hi)
      y[r] = mode == 0 ? acc : (mode == 1 ? __dsub_rn(base[r], acc) : __dadd_rn(base[r], acc));
  };
  put(row, a0);
  put(row + 1, a1);
}

}  // namespace

std::unique_ptr<DevCsr> upload_csr(Ctx* ctx, int nrows, int ncols, const int* rp,
                                   const int* ci, const double* v) {
  auto a = std::make_unique<DevCsr>();
  a->ctx = ctx;
  a->nrows = nrows;
  a->ncols = ncols;
  a->nnz = rp[nrows];
  a->nslices = (nrows + kSlice - 1) / kSlice;
  std::vector<int64_t> sptr(a->nslices + 1, 0);
  std::vector<int> swidth(a->nslices, 0);
  for (int s = 0; s < a->nslices; ++s) {
    int w = 0;
    for (int r = s * kSlice; r < std::min(nrows, s * kSlice + kSlice); ++r)
      w = std::max(w, rp[r + 1] - rp[r]);
    swidth[s] = w;
    sptr[s + 1] = sptr[s] + static_cast<int64_t>(kSlice) * w;
  }
  a->padded = sptr[a->nslices];
  std::vector<int> hcol(std::max<int64_t>(1, a->padded), -1);
  std::vector<double> hval(std::max<int64_t>(1, a->padded), 0.0);
  for (int s = 0; s < a->nslices; ++s)
    for (int r = s * kSlice; r < std::min(nrows, s * kSlice + kSlice); ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) {
        const int64_t pos = sptr[s] + static_cast<int64_t>(kSlice) * (k - rp[r]) + (r - s * kSlice);
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
  const int nsl = (row_hi + kSlice - 1) / kSlice - row_lo / kSlice;
  const int blocks = (nsl * 32 + threads - 1) / threads;  // one warp per slice
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
