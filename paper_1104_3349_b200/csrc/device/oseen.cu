// Oseen saddle-point assembly and row equilibration on the device (SURVEY
// 8(f) row 3): the MAC-grid matrix of generate_oseen (proj/src/oseen.cpp:
// 108-212, Recirculating wind, pinned last pressure) followed by scale_rows
// (proj/src/row_scaling.cpp:8-31), one thread per row.
//
// Bit-identical to the reference: this file is compiled with --fmad=false so
// every expression below rounds exactly as the host code (the reference's
// order, -ffp-contract=off) does; the grid coordinates (std::pow for the
// stretched grid) come from the host; a row's at most 7 stencil entries are
// sorted and duplicates summed from 0.0 as from_triplets does, exact zeros
// pruned.  Rows land in fixed 8-entry slots, then are compacted.
#include <string>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kRowSlots = 8;

struct DevGrid {
  int n;
  const double *x, *y, *xc, *yc;
  __device__ int nu_per_comp() const { return n * (n - 1); }
  __device__ int iu(int i, int j) const { return (i - 1) + j * (n - 1); }
  __device__ int iv(int i, int j) const { return nu_per_comp() + i + (j - 1) * n; }
  __device__ int ip(int i, int j) const { return i + j * n; }
};

struct Row {
  int c[kRowSlots * 2];
  double v[kRowSlots * 2];
  int m = 0;
  double rhs = 0.0, diag = 0.0;
  __device__ void push(int col, double val) {
    c[m] = col;
    v[m] = val;
    ++m;
  }
};

struct Nb {
  int col;
  double value, dist, face;
};

__device__ __forceinline__ void diffusion(Row& r, double nu, const Nb& nb) {
  const double t = nu * nb.face / nb.dist;
  r.diag += t;
  if (nb.col >= 0) r.push(nb.col, -t);
  else r.rhs += t * nb.value;
}

__device__ __forceinline__ void convection(Row& r, double speed, double vol, const Nb& up,
                                           bool upstream_is_low) {
  if (speed == 0.0) return;
  const bool use_low = speed > 0.0;
  if (use_low != upstream_is_low) return;
  const double c = fabs(speed) * vol / up.dist;
  r.diag += c;
  if (up.col >= 0) r.push(up.col, -c);
  else r.rhs += c * up.value;
}

__device__ __forceinline__ void wind(double x, double y, double& w1, double& w2) {
  const double xh = 2.0 * x - 1.0;
  const double yh = 2.0 * y - 1.0;
  w1 = 2.0 * yh * (1.0 - xh * xh);
  w2 = -2.0 * xh * (1.0 - yh * yh);
}

// Sort by column, sum duplicates from 0.0, drop exact zeros, then divide by
// the signed entry of largest magnitude (first maximum wins).
__device__ void finish_row(Row& r, int row, int* oc, double* ov, int* olen, double* rhs,
                           double rhs_in) {
  for (int a = 1; a < r.m; ++a) {
    const int c = r.c[a];
    const double v = r.v[a];
    int b = a - 1;
    while (b >= 0 && r.c[b] > c) {
      r.c[b + 1] = r.c[b];
      r.v[b + 1] = r.v[b];
      --b;
    }
    r.c[b + 1] = c;
    r.v[b + 1] = v;
  }
  int len = 0;
  int* cs = oc + static_cast<long long>(row) * kRowSlots;
  double* vs = ov + static_cast<long long>(row) * kRowSlots;
  for (int k = 0; k < r.m;) {
    const int c = r.c[k];
    double sum = 0.0;
    while (k < r.m && r.c[k] == c) sum += r.v[k++];
    if (sum != 0.0) {
      cs[len] = c;
      vs[len] = sum;
      ++len;
    }
  }
  olen[row] = len;
  if (len == 0) {  // scale_rows rejects it; the host raises the error
    rhs[row] = rhs_in;
    return;
  }
  double pivot = vs[0];
  for (int k = 0; k < len; ++k)
    if (fabs(vs[k]) > fabs(pivot)) pivot = vs[k];
  for (int k = 0; k < len; ++k) vs[k] /= pivot;
  rhs[row] = rhs_in / pivot;
}

__global__ void __launch_bounds__(256) oseen_rows_kernel(DevGrid g, double nu, int p, int pin,
                                                         int nrows, int* __restrict__ oc,
                                                         double* __restrict__ ov,
                                                         int* __restrict__ olen,
                                                         double* __restrict__ rhs) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  const int n = g.n, nuc = g.nu_per_comp();
  Row r;
  if (row < nuc) {  // u-momentum (oseen.cpp:115-149)
    const int j = row / (n - 1), i = row % (n - 1) + 1;
    const double wx = g.xc[i] - g.xc[i - 1];
    const double hy = g.y[j + 1] - g.y[j];
    const double vol = wx * hy;
    double w1, w2;
    wind(g.x[i], g.yc[j], w1, w2);
    const Nb west{i - 1 >= 1 ? g.iu(i - 1, j) : -1, 0.0, g.x[i] - g.x[i - 1], hy};
    const Nb east{i + 1 <= n - 1 ? g.iu(i + 1, j) : -1, 0.0, g.x[i + 1] - g.x[i], hy};
    const Nb south{j - 1 >= 0 ? g.iu(i, j - 1) : -1, 0.0,
                   j - 1 >= 0 ? g.yc[j] - g.yc[j - 1] : g.yc[j], wx};
    const Nb north{j + 1 <= n - 1 ? g.iu(i, j + 1) : -1, 1.0,
                   j + 1 <= n - 1 ? g.yc[j + 1] - g.yc[j] : 1.0 - g.yc[n - 1], wx};
    diffusion(r, nu, west);
    diffusion(r, nu, east);
    diffusion(r, nu, south);
    diffusion(r, nu, north);
    convection(r, w1, vol, west, true);
    convection(r, w1, vol, east, false);
    convection(r, w2, vol, south, true);
    convection(r, w2, vol, north, false);
    r.push(row, r.diag);
    if (g.ip(i, j) != pin) r.push(p + g.ip(i, j), hy);
    if (g.ip(i - 1, j) != pin) r.push(p + g.ip(i - 1, j), -hy);
    finish_row(r, row, oc, ov, olen, rhs, r.rhs);
  } else if (row < p) {  // v-momentum (oseen.cpp:151-181)
    const int q = row - nuc;
    const int j = q / n + 1, i = q % n;
    const double wx = g.x[i + 1] - g.x[i];
    const double hy = g.yc[j] - g.yc[j - 1];
    const double vol = wx * hy;
    double w1, w2;
    wind(g.xc[i], g.y[j], w1, w2);
    const Nb west{i - 1 >= 0 ? g.iv(i - 1, j) : -1, 0.0,
                  i - 1 >= 0 ? g.xc[i] - g.xc[i - 1] : g.xc[0], hy};
    const Nb east{i + 1 <= n - 1 ? g.iv(i + 1, j) : -1, 0.0,
                  i + 1 <= n - 1 ? g.xc[i + 1] - g.xc[i] : 1.0 - g.xc[n - 1], hy};
    const Nb south{j - 1 >= 1 ? g.iv(i, j - 1) : -1, 0.0, g.y[j] - g.y[j - 1], wx};
    const Nb north{j + 1 <= n - 1 ? g.iv(i, j + 1) : -1, 0.0, g.y[j + 1] - g.y[j], wx};
    diffusion(r, nu, west);
    diffusion(r, nu, east);
    diffusion(r, nu, south);
    diffusion(r, nu, north);
    convection(r, w1, vol, west, true);
    convection(r, w1, vol, east, false);
    convection(r, w2, vol, south, true);
    convection(r, w2, vol, north, false);
    r.push(row, r.diag);
    if (g.ip(i, j) != pin) r.push(p + g.ip(i, j), wx);
    if (g.ip(i, j - 1) != pin) r.push(p + g.ip(i, j - 1), -wx);
    finish_row(r, row, oc, ov, olen, rhs, r.rhs);
  } else {  // continuity in flux form (oseen.cpp:183-193), pinned last pressure
    const int q = row - p;
    const int j = q / n, i = q % n;
    if (q == pin) {
      r.push(p + pin, 1.0);
    } else {
      const double dx = g.x[i + 1] - g.x[i];
      const double dy = g.y[j + 1] - g.y[j];
      if (i + 1 <= n - 1) r.push(g.iu(i + 1, j), dy);
      if (i >= 1) r.push(g.iu(i, j), -dy);
      if (j + 1 <= n - 1) r.push(g.iv(i, j + 1), dx);
      if (j >= 1) r.push(g.iv(i, j), -dx);
    }
    finish_row(r, row, oc, ov, olen, rhs, 0.0);
  }
}

__global__ void __launch_bounds__(256) compact_rows_kernel(int nrows, const int* __restrict__ oc,
                                                           const double* __restrict__ ov,
                                                           const int* __restrict__ rp,
                                                           int* __restrict__ ci,
                                                           double* __restrict__ v) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  for (int k = rp[row]; k < rp[row + 1]; ++k) {
    ci[k] = oc[static_cast<long long>(row) * kRowSlots + (k - rp[row])];
    v[k] = ov[static_cast<long long>(row) * kRowSlots + (k - rp[row])];
  }
}

}  // namespace

void oseen_assemble_device(Ctx* ctx, int n, const std::vector<double>& x,
                           const std::vector<double>& y, const std::vector<double>& xc,
                           const std::vector<double>& yc, double nu, std::vector<int>& rp,
                           std::vector<int>& ci, std::vector<double>& v,
                           std::vector<double>& rhs, int& p_out) {
  cudaStream_t s = ctx->stream;
  const int nuc = n * (n - 1), p = 2 * nuc, np = n * n, nrows = p + np;
  p_out = p;
  DevBuf dx(sizeof(double) * x.size()), dy(sizeof(double) * y.size()),
      dxc(sizeof(double) * xc.size()), dyc(sizeof(double) * yc.size());
  MSCG_CUDA(cudaMemcpyAsync(dx.p, x.data(), dx.bytes, cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaMemcpyAsync(dy.p, y.data(), dy.bytes, cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaMemcpyAsync(dxc.p, xc.data(), dxc.bytes, cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaMemcpyAsync(dyc.p, yc.data(), dyc.bytes, cudaMemcpyHostToDevice, s));
  DevBuf oc(sizeof(int) * kRowSlots * static_cast<size_t>(nrows)),
      ov(sizeof(double) * kRowSlots * static_cast<size_t>(nrows)), olen(sizeof(int) * nrows),
      drhs(sizeof(double) * nrows);
  DevGrid g{n, dx.as<double>(), dy.as<double>(), dxc.as<double>(), dyc.as<double>()};
  const int threads = 256, blocks = (nrows + threads - 1) / threads;
  oseen_rows_kernel<<<blocks, threads, 0, s>>>(g, nu, p, np - 1, nrows, oc.as<int>(),
                                               ov.as<double>(), olen.as<int>(), drhs.as<double>());
  MSCG_CUDA(cudaGetLastError());
  ctx->launches++;
  std::vector<int> len(nrows);
  rhs.resize(nrows);
  MSCG_CUDA(cudaMemcpyAsync(len.data(), olen.p, sizeof(int) * nrows, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaMemcpyAsync(rhs.data(), drhs.p, sizeof(double) * nrows, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  rp.assign(nrows + 1, 0);
  for (int r = 0; r < nrows; ++r) {
    if (len[r] == 0)
      throw Error(1, "scale_rows: row " + std::to_string(r) + " is identically zero");
    rp[r + 1] = rp[r] + len[r];
  }
  const int nnz = rp[nrows];
  DevBuf drp(sizeof(int) * (nrows + 1)), dci(sizeof(int) * nnz), dv(sizeof(double) * nnz);
  MSCG_CUDA(cudaMemcpyAsync(drp.p, rp.data(), drp.bytes, cudaMemcpyHostToDevice, s));
  compact_rows_kernel<<<blocks, threads, 0, s>>>(nrows, oc.as<int>(), ov.as<double>(),
                                                 drp.as<int>(), dci.as<int>(), dv.as<double>());
  MSCG_CUDA(cudaGetLastError());
  ctx->launches++;
  ci.resize(nnz);
  v.resize(nnz);
  MSCG_CUDA(cudaMemcpyAsync(ci.data(), dci.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaMemcpyAsync(v.data(), dv.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mscg
