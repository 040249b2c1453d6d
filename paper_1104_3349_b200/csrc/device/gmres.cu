// Restarted GMRES on the device (reference gmres, proj/src/gmres.cpp:35-191).
//
// The Arnoldi step keeps every vector in HBM and every scalar on the device:
//   w = A B^-1 v_j            (precond apply + SELL SpMV, right preconditioning)
//   orthogonalisation         DCGS2 (default): two basis sweeps, see below;
//                             CGS2: multi-dot, fused axpy+dot, multi-axpy
//                             (h = V^T w; w -= V h, twice), or MGS in the
//                             reference's order (one fused axpy+dot kernel per
//                             basis vector)
//   h_{j+1,j} = ||w||, v_{j+1} = w / h_{j+1,j}
//   Givens rotation + residual estimate: one single-thread kernel
// Reductions are two-stage and deterministic (fixed per-CTA partials summed in
// CTA order by the last CTA).  The host reads one 32-byte status record per
// iteration (the reference's convergence test needs it); no other host
// synchronisation happens inside a cycle.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kThreads = 256;

struct Reducer {
  double* partials;        // [nvec][nblk]
  unsigned int* counter;   // last-block detection
  int nblk;
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) r += sh[w];
  return r;  // valid in thread 0
}

// Finalise: the last CTA to arrive sums partials[i][*] in CTA order.
__device__ __forceinline__ bool last_block(Reducer red) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(red.counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  return is_last;
}

// out[i] (i < nvec) = sum over CTAs of partials[i][cta]; scale: out = f(sum).
// One warp per output: lane l adds the CTAs l, l + 32, ... in order
// (coalesced loads), then a fixed butterfly — deterministic, and a few
// latencies instead of one dependent L2 load per CTA.
__device__ void finish(Reducer red, int nvec, double* out, int mode) {
  __threadfence();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = warp; i < nvec; i += nw) {
    const double* pr = red.partials + static_cast<size_t>(i) * red.nblk;
    double s = 0.0;
    for (int c = lane; c < red.nblk; c += 32) s += __ldcg(pr + c);
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) out[i] = mode == 1 ? sqrt(s) : s;
  }
  if (threadIdx.x == 0) *red.counter = 0u;
  __syncthreads();  // every output written before the caller's epilogue reads it
}

// ||x||_2 -> *out
__global__ void __launch_bounds__(kThreads) nrm2_kernel(int n, const double* __restrict__ x,
                                                        Reducer red, double* out) {
  __shared__ double sh[kThreads / 32];
  double acc = 0.0;
  // grid-stride, four loads in flight per thread (summation order unchanged)
  const int stride = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const double a = x[i], b = x[i + stride], c = x[i + 2 * stride], d = x[i + 3 * stride];
    acc = fma(a, a, acc);
    acc = fma(b, b, acc);
    acc = fma(c, c, acc);
    acc = fma(d, d, acc);
  }
  for (; i < n; i += stride) acc = fma(x[i], x[i], acc);
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) red.partials[blockIdx.x] = s;
  if (last_block(red)) finish(red, 1, out, 1);
}

// sum of squares of x[0:n) -> *out (a distributed rank's local part)
__global__ void __launch_bounds__(kThreads) sumsq_kernel(int n, const double* __restrict__ x,
                                                         Reducer red, double* out) {
  __shared__ double sh[kThreads / 32];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    acc = fma(x[i], x[i], acc);
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) red.partials[blockIdx.x] = s;
  if (last_block(red)) finish(red, 1, out, 0);
}

__global__ void sqrt_kernel(double* v) { *v = sqrt(*v); }

// y = a - b (elementwise)
__global__ void sub2_kernel(int n, const double* __restrict__ a, const double* __restrict__ b,
                            double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = a[i] - b[i];
}

// h[i] = V_i . w for i < nv: basis vectors in groups of kDotGroup, so w is
// read once per group and each CTA reduces kDotGroup sums per pass.  Rows
// go in 16-byte pairs (the basis is stored with a 32-element-aligned
// leading dimension), two pairs in flight per thread.
// Groups of 16 (184 registers, one CTA per SM) halve the w re-reads on long
// vectors; short ones keep groups of 8 (two CTAs per SM, one wave).
template <int kDotGroup>
__global__ void __launch_bounds__(kThreads) multidot_kernel(int n, int nv, const double* __restrict__ V,
                                                            size_t ld, const double* __restrict__ w,
                                                            Reducer red, double* h) {
  __shared__ double sh[kThreads / 32][kDotGroup];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npair = n >> 1;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (int i0 = 0; i0 < nv; i0 += kDotGroup) {
    const int ng = min(kDotGroup, nv - i0);
    double acc[kDotGroup];
#pragma unroll
    for (int g = 0; g < kDotGroup; ++g) acc[g] = 0.0;
    const int stride = gridDim.x * blockDim.x;
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + stride < npair; q += 2 * stride) {
      const double2 wa = w2[q], wb = w2[q + stride];
      double2 va[kDotGroup], vb[kDotGroup];
#pragma unroll
      for (int g = 0; g < kDotGroup; ++g) {
        const double2* vg = reinterpret_cast<const double2*>(V + ld * (i0 + g));
        va[g] = g < ng ? __ldg(vg + q) : make_double2(0.0, 0.0);
        vb[g] = g < ng ? __ldg(vg + q + stride) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int g = 0; g < kDotGroup; ++g)
        acc[g] = fma(vb[g].y, wb.y, fma(vb[g].x, wb.x, fma(va[g].y, wa.y, fma(va[g].x, wa.x, acc[g]))));
    }
    if (q < npair) {
      const double2 wa = w2[q];
#pragma unroll
      for (int g = 0; g < kDotGroup; ++g)
        if (g < ng) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(V + ld * (i0 + g)) + q);
          acc[g] = fma(v.y, wa.y, fma(v.x, wa.x, acc[g]));
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd length: the last row
#pragma unroll
      for (int g = 0; g < kDotGroup; ++g)
        if (g < ng) acc[g] = fma(__ldg(V + ld * (i0 + g) + (n - 1)), w[n - 1], acc[g]);
    }
#pragma unroll
    for (int g = 0; g < kDotGroup; ++g) {
      double v = acc[g];
      for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) sh[warp][g] = v;
    }
    __syncthreads();
    if (threadIdx.x < ng) {
      double t = 0.0;
      for (int k = 0; k < kThreads / 32; ++k) t += sh[k][threadIdx.x];
      red.partials[static_cast<size_t>(i0 + threadIdx.x) * red.nblk + blockIdx.x] = t;
    }
    __syncthreads();
  }
  if (last_block(red)) finish(red, nv, h, 0);
}

// w -= sum_i h[i] V_i ; optionally H(:,j) += h (accum into column) by CTA 0.
__global__ void __launch_bounds__(kThreads) multiaxpy_kernel(int n, int nv, const double* __restrict__ V,
                                                             size_t ld, const double* __restrict__ h,
                                                             double* __restrict__ w, double* hcol,
                                                             int accumulate) {
  __shared__ double sh[512];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) sh[i] = h[i];
  __syncthreads();
  const int npair = n >> 1;
  double2* w2 = reinterpret_cast<double2*>(w);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npair; q += gridDim.x * blockDim.x) {
    double2 acc = w2[q];
    for (int i = 0; i < nv; ++i) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(V + ld * i) + q);
      acc.x = fma(-sh[i], v.x, acc.x);
      acc.y = fma(-sh[i], v.y, acc.y);
    }
    w2[q] = acc;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double acc = w[n - 1];
    for (int i = 0; i < nv; ++i) acc = fma(-sh[i], V[ld * i + (n - 1)], acc);
    w[n - 1] = acc;
  }
  if (blockIdx.x == 0 && hcol)
    for (int i = threadIdx.x; i < nv; i += blockDim.x) hcol[i] = accumulate ? hcol[i] + sh[i] : sh[i];
}

// CGS2 middle step, fused: w -= V h (first pass's projection, same per-row
// arithmetic as multiaxpy_kernel) and h2 = V^T w (second pass's dots) in one
// sweep, so the basis streams from HBM three times per Arnoldi step instead of
// four (the dot re-reads the rows this thread just loaded: L1/L2 hits).  Per
// row pair the 32 products of a group of 32 basis vectors are reduced across
// the warp by a transposing butterfly (31 shuffles; lane k ends with vector
// 32g + k), accumulated per warp in shared memory, then per CTA into the
// partials, which the last CTA sums in CTA order (deterministic).  CTA 0
// stores H(:,j) = h.
__global__ void __launch_bounds__(kThreads) axpy_dot_kernel(int n, int nv, const double* __restrict__ V,
                                                            size_t ld, const double* __restrict__ h,
                                                            double* __restrict__ w, double* hcol,
                                                            Reducer red, double* hout) {
  __shared__ double sh[512];
  __shared__ double acc_sh[kThreads / 32][512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) sh[i] = h[i];
  for (int i = lane; i < nv; i += 32) acc_sh[warp][i] = 0.0;
  __syncthreads();
  const int npair = n >> 1;
  double2* w2 = reinterpret_cast<double2*>(w);
  const int stride = gridDim.x * blockDim.x;
  for (int qb = blockIdx.x * blockDim.x; qb < npair; qb += stride) {  // CTA-uniform trip count
    const int q = qb + threadIdx.x;
    const bool on = q < npair;
    double2 acc = make_double2(0.0, 0.0);
    if (on) {
      acc = w2[q];
      // software-pipelined: the next kU rows are in flight while the current
      // kU are applied (same i-ascending order as multiaxpy_kernel)
      constexpr int kU = 16;
      double2 cur[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        cur[u] = u < nv ? __ldg(reinterpret_cast<const double2*>(V + ld * u) + q)
                        : make_double2(0.0, 0.0);
      for (int i0 = 0; i0 < nv; i0 += kU) {
        double2 nxt[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int i = i0 + kU + u;
          nxt[u] = i < nv ? __ldg(reinterpret_cast<const double2*>(V + ld * i) + q)
                          : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (i0 + u < nv) {
            acc.x = fma(-sh[i0 + u], cur[u].x, acc.x);
            acc.y = fma(-sh[i0 + u], cur[u].y, acc.y);
          }
#pragma unroll
        for (int u = 0; u < kU; ++u) cur[u] = nxt[u];
      }
      w2[q] = acc;
    }
    // groups last to first: the rows loaded last are the likeliest L2 hits
    for (int g0 = (nv - 1) & ~31; g0 >= 0; g0 -= 32) {
      double p[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = g0 + k;
        double2 v = make_double2(0.0, 0.0);
        if (on && i < nv) v = __ldg(reinterpret_cast<const double2*>(V + ld * i) + q);
        p[k] = fma(v.y, acc.y, v.x * acc.x);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const bool hi = lane & off;
#pragma unroll
        for (int k = 0; k < off; ++k) {
          const double send = hi ? p[k] : p[k + off];
          const double keep = hi ? p[k + off] : p[k];
          p[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      if (g0 + lane < nv) acc_sh[warp][g0 + lane] += p[0];
    }
  }
  __syncthreads();
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd length: the last row
    double a = w[n - 1];
    for (int i = 0; i < nv; ++i) a = fma(-sh[i], V[ld * i + (n - 1)], a);
    w[n - 1] = a;
    for (int i = 0; i < nv; ++i) acc_sh[0][i] = fma(V[ld * i + (n - 1)], a, acc_sh[0][i]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) t += acc_sh[k][i];
    red.partials[static_cast<size_t>(i) * red.nblk + blockIdx.x] = t;
  }
  if (blockIdx.x == 0 && hcol)
    for (int i = threadIdx.x; i < nv; i += blockDim.x) hcol[i] = sh[i];
  if (last_block(red)) finish(red, nv, hout, 0);
}

// MGS step (reference order, gmres.cpp:112-116), fused: apply the previous
// projection w -= h_prev v_{i-1} and accumulate v_i . w in the same pass.
__global__ void __launch_bounds__(kThreads) mgs_kernel(int n, const double* __restrict__ vprev,
                                                       const double* hprev, const double* __restrict__ vi,
                                                       double* __restrict__ w, Reducer red, double* hout) {
  __shared__ double sh[kThreads / 32];
  const double hp = vprev ? *hprev : 0.0;
  double acc = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double wr = w[r];
    if (vprev) {
      wr = __dsub_rn(wr, __dmul_rn(hp, vprev[r]));
      w[r] = wr;
    }
    if (vi) acc = fma(vi[r], wr, acc);
  }
  if (!vi) return;
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) red.partials[blockIdx.x] = s;
  if (last_block(red)) finish(red, 1, hout, 0);
}

// y = x / s  (s on device)
__global__ void scale_div_kernel(int n, const double* __restrict__ x, const double* s,
                                 double* __restrict__ y) {
  const double d = *s;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}

// z = sum_j y_j V_j with the reference's per-entry order (gmres.cpp:158-161).
__global__ void combine_kernel(int n, int m, const double* __restrict__ V, size_t ld,
                               const double* __restrict__ y, double* __restrict__ z) {
  __shared__ double sy[512];
  for (int j = threadIdx.x; j < m; j += blockDim.x) sy[j] = y[j];
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, __dmul_rn(sy[j], V[ld * j + r]));
    z[r] = acc;
  }
}

__global__ void axpy1_kernel(int n, const double* __restrict__ z, double* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = x[i] + z[i];
}

__global__ void fill_kernel(int n, double v, double* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = v;
}

// Small dense state: H column-major (m+1) x m, cs, sn, g.
struct Small {
  double* H;
  double* cs;
  double* sn;
  double* g;
  double* y;
  double* scal;   // [0] hnext, [1] beta, [2] tmp norm, ...
  double* status; // [0] rel, [1] breakdown, [2] hnext, [3] |g_{j+1}|
  int m;
};

// v_{j+1} = w / hnext (if hnext >= 1e-14), Givens update of column j
// (gmres.cpp:117-148), single thread.
__global__ void givens_kernel(Small s, int j, double denom) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int ld = s.m + 1;
  double* Hc = s.H + static_cast<size_t>(j) * ld;
  const double hnext = s.scal[0];
  Hc[j + 1] = hnext;
  const bool breakdown = !(hnext >= 1e-14);
  for (int i = 0; i < j; ++i) {
    const double t1 = s.cs[i] * Hc[i] + s.sn[i] * Hc[i + 1];
    const double t2 = -s.sn[i] * Hc[i] + s.cs[i] * Hc[i + 1];
    Hc[i] = t1;
    Hc[i + 1] = t2;
  }
  const double dr = hypot(Hc[j], Hc[j + 1]);
  s.cs[j] = dr == 0.0 ? 1.0 : Hc[j] / dr;
  s.sn[j] = dr == 0.0 ? 0.0 : Hc[j + 1] / dr;
  Hc[j] = dr;
  Hc[j + 1] = 0.0;
  s.g[j + 1] = -s.sn[j] * s.g[j];
  s.g[j] = s.cs[j] * s.g[j];
  s.status[0] = fabs(s.g[j + 1]) / denom;
  s.status[1] = breakdown ? 1.0 : 0.0;
  s.status[2] = hnext;
}

// Back substitution H y = g (gmres.cpp:152-157).
__global__ void backsolve_kernel(Small s, int m) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int ld = s.m + 1;
  for (int i = m - 1; i >= 0; --i) {
    double acc = s.g[i];
    for (int j = i + 1; j < m; ++j) acc -= s.H[static_cast<size_t>(j) * ld + i] * s.y[j];
    s.y[i] = acc / s.H[static_cast<size_t>(i) * ld + i];
  }
}

__global__ void init_cycle_kernel(Small s, const double* beta, double* nu0) {
  for (int i = threadIdx.x; i <= s.m; i += blockDim.x) s.g[i] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    s.g[0] = *beta;
    if (nu0) *nu0 = *beta;
  }
}

// ---------------------------------------------------------------- DCGS2
// Low-synchronisation CGS2 with delayed reorthogonalisation (the DCGS2
// Arnoldi of Swirydowicz et al. 2020 / Bielich et al. 2022, restated): two
// sweeps over the basis per iteration instead of three.
//
// State after iteration j: q_0..q_j final (orthonormal), slot j+1 holds
// y_{j+1} = A B^-1 q_j projected ONCE (unnormalised, nu_{j+1} = ||y_{j+1}||),
// H columns 0..j-1 final and column j preliminary.  Iteration j+1:
//   w = A B^-1 y_{j+1}                        (the operator is linear: W = w / nu)
//   sweep 1 (dcgs2_dot_kernel): s' = Q^T y, t' = Q^T w, y.y, y.w;  its last
//     CTA then (dcgs2_fix) reorthogonalises y in coefficient space:
//       u = y / nu, s = Q^T u, rho = sqrt(u.u - s.s), q_{j+1} = (u - Q s) / rho
//     which finalises column j (H[0:j+1, j] += nu s, H[j+1, j] = nu rho) and
//     its Givens rotation, and forms column j+1 without touching a vector:
//       A B^-1 q_{j+1} = (W - Q_{j+2} H s) / rho,  t = Q^T W,
//       c = q_{j+1}.W = (u.W - s.t) / rho,  h = ([t; c] - H s) / rho;
//   sweep 2 (dcgs2_axpy_kernel): q_{j+1} = (u - Q s) / rho into its slot and
//     y_{j+2} = (W - Q t - c q_{j+1}) / rho into the next, with ||y_{j+2}||;
//     its last CTA rotates a copy of column j+1 (preliminary) for the
//     convergence test, so the host still reads one status per iteration.
// The last column of a cycle is finalised by the speculative next iteration
// already in the stream, or by one dot sweep (finalize-only) at restart.
// Same operator and projections as CGS2; only rounding differs (measured:
// iteration counts and histories unchanged, tests/test_gpu_parity.py).
struct Dcgs {
  double* Hraw;  // (m+1) x m raw Hessenberg columns, column-major, ld m+1
  double* dots;  // sweep-1 sums: [0,nq) Q^T y, [nq,2nq) Q^T w, [2nq] y.y, [2nq+1] y.w
  double* coef;  // [0,m+1) s, [m+1, 2m+2) t, [2m+2] c, [2m+3] rho, [2m+4] nu, [2m+5] ok
  double* nu;    // [m+2]: nu[j] = ||y_j||
};

// The serial Givens work of an iteration runs on one thread of a reduction
// kernel's last CTA; the CTA first stages the rotations and the column in
// shared memory (a dependent global load per rotation would cost an L2 round
// trip each).  kMaxRestart bounds the staged arrays.
constexpr int kMaxRestart = 500;
struct GivensStage {
  double cs[kMaxRestart + 1], sn[kMaxRestart + 1], col[kMaxRestart + 2];
};

// all threads: stage rotations 0..k-1 and column entries 0..k+1
__device__ __forceinline__ void stage_givens(GivensStage& gs, const Small& s, const double* raw, int k) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    gs.cs[i] = s.cs[i];
    gs.sn[i] = s.sn[i];
  }
  for (int i = threadIdx.x; i <= k + 1; i += blockDim.x) gs.col[i] = raw[i];
  __syncthreads();
}

// one thread: rotations 0..k-1 applied to the staged column
// (gmres.cpp:117-148 arithmetic), then the new rotation k
__device__ __forceinline__ void rotate_staged(GivensStage& gs, int k, double& cs, double& sn) {
  double* Hc = gs.col;
  for (int i = 0; i < k; ++i) {
    const double t1 = gs.cs[i] * Hc[i] + gs.sn[i] * Hc[i + 1];
    const double t2 = -gs.sn[i] * Hc[i] + gs.cs[i] * Hc[i + 1];
    Hc[i] = t1;
    Hc[i + 1] = t2;
  }
  const double dr = hypot(Hc[k], Hc[k + 1]);
  cs = dr == 0.0 ? 1.0 : Hc[k] / dr;
  sn = dr == 0.0 ? 0.0 : Hc[k + 1] / dr;
  Hc[k] = dr;
  Hc[k + 1] = 0.0;
}

// Sweep-1 epilogue (last CTA, all threads): finalise column j-1 and its
// rotation, then the coefficients of sweep 2 and the raw column j.
// finalize_only: no w (the cycle's last column).
__device__ void dcgs2_fix(const Small& s, const Dcgs& d, int j, bool finalize_only) {
  __shared__ GivensStage gs;
  __shared__ double S[kMaxRestart + 1], T[kMaxRestart + 1];
  __shared__ double sc[2];
  const int m = s.m, ldh = m + 1;
  const double nu = d.nu[j];
  const bool ok = nu >= 1e-14;  // y_j exists (no breakdown before it)
  for (int i = threadIdx.x; i < j; i += blockDim.x) {
    const double si = ok ? d.dots[i] / nu : 0.0;
    const double ti = ok && !finalize_only ? d.dots[j + i] / nu : 0.0;
    S[i] = si;
    T[i] = ti;
    d.coef[i] = si;
    d.coef[m + 1 + i] = ti;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double rho = 1.0;
    if (j > 0 && ok) {
      const double alpha = d.dots[2 * j] / (nu * nu);
      double ss = 0.0;
      for (int i = 0; i < j; ++i) ss = fma(S[i], S[i], ss);
      const double r2 = alpha - ss;
      rho = r2 > 0.0 ? sqrt(r2) : sqrt(alpha);
    }
    sc[0] = rho;
  }
  __syncthreads();
  const double rho = sc[0];
  if (j > 0) {
    // column j-1: H[0:j, j-1] += nu s, H[j, j-1] = nu rho (raw), then its
    // final rotation
    double* hc = d.Hraw + static_cast<size_t>(j - 1) * ldh;
    if (ok) {
      for (int i = threadIdx.x; i < j; i += blockDim.x) hc[i] = fma(nu, S[i], hc[i]);
      if (threadIdx.x == 0) hc[j] = nu * rho;
    }
    __syncthreads();
    stage_givens(gs, s, hc, j - 1);
    if (threadIdx.x == 0) {
      const int k = j - 1;
      double cs, sn;
      rotate_staged(gs, k, cs, sn);
      s.cs[k] = cs;
      s.sn[k] = sn;
      s.g[k + 1] = -sn * s.g[k];
      s.g[k] = cs * s.g[k];
    }
    __syncthreads();
    double* Rc = s.H + static_cast<size_t>(j - 1) * ldh;
    for (int i = threadIdx.x; i <= j; i += blockDim.x) Rc[i] = gs.col[i];
  }
  if (finalize_only) return;
  if (threadIdx.x == 0) {
    const double bt = ok ? d.dots[2 * j + 1] / (nu * nu) : 0.0;
    double st = 0.0;
    for (int i = 0; i < j; ++i) st = fma(S[i], T[i], st);
    const double c = (bt - st) / rho;
    sc[1] = c;
    d.coef[2 * m + 2] = c;
    d.coef[2 * m + 3] = rho;
    d.coef[2 * m + 4] = nu;
    d.coef[2 * m + 5] = ok ? 1.0 : 0.0;
  }
  __syncthreads();
  const double c = sc[1];
  // raw column j: h_i = (t_i - sum_k H[i,k] s_k) / rho, t_j = c (H upper
  // Hessenberg: k >= i-1); for fixed k the threads read a column: coalesced
  double* hj = d.Hraw + static_cast<size_t>(j) * ldh;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    double acc = i < j ? T[i] : c;
#pragma unroll 4
    for (int k = i > 0 ? i - 1 : 0; k < j; ++k) acc = fma(-d.Hraw[static_cast<size_t>(k) * ldh + i], S[k], acc);
    hj[i] = acc / rho;
  }
}

// Sweep 1: dots of y = slot j (and w) against q_0..q_{j-1}, plus y.y and
// y.w, basis vectors in groups of kG (w and y re-read per group).  kW = false:
// the cycle's finalize-only sweep (no w).  The inner loop is branch-free so
// that every load of a row pair is in flight at once.
template <int kG, bool kW>
__device__ __forceinline__ void dot_sweep(int n, int j, const double* __restrict__ V, size_t ld,
                                          const double* __restrict__ w, Reducer red) {
  __shared__ double sh[kThreads / 32][2 * kG + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = j;
  const double* y = V + ld * j;
  const int npair = n >> 1;
  const double2* y2 = reinterpret_cast<const double2*>(y);
  const double2* w2 = reinterpret_cast<const double2*>(kW ? w : y);
  const int ngroups = nq > 0 ? (nq + kG - 1) / kG : 1;
  const int stride = gridDim.x * blockDim.x;
  for (int grp = 0; grp < ngroups; ++grp) {
    const int i0 = grp * kG;
    const int ng = max(0, min(kG, nq - i0));
    const bool first = grp == 0;
    double ay[kG], aw[kG], yy = 0.0, yw = 0.0;
#pragma unroll
    for (int g = 0; g < kG; ++g) ay[g] = aw[g] = 0.0;
    // basis rows past the group's end read a valid vector (clamped index)
    // into accumulators that are never stored
    const double2* vg[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g)
      vg[g] = reinterpret_cast<const double2*>(V + ld * min(i0 + g, max(nq - 1, 0)));
    // two row pairs per trip (q, q + stride), like multidot_kernel: 2 kG
    // basis loads in flight per thread
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + stride < npair; q += 2 * stride) {
      const double2 ya = y2[q], yb = y2[q + stride];
      const double2 wa = w2[q], wb = w2[q + stride];
      double2 va[kG], vb[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        va[g] = __ldg(vg[g] + q);
        vb[g] = __ldg(vg[g] + q + stride);
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        ay[g] = fma(vb[g].y, yb.y, fma(vb[g].x, yb.x, fma(va[g].y, ya.y, fma(va[g].x, ya.x, ay[g]))));
        if (kW)
          aw[g] = fma(vb[g].y, wb.y, fma(vb[g].x, wb.x, fma(va[g].y, wa.y, fma(va[g].x, wa.x, aw[g]))));
      }
      yy = fma(yb.y, yb.y, fma(yb.x, yb.x, fma(ya.y, ya.y, fma(ya.x, ya.x, yy))));
      if (kW) yw = fma(yb.y, wb.y, fma(yb.x, wb.x, fma(ya.y, wa.y, fma(ya.x, wa.x, yw))));
    }
    if (q < npair) {
      const double2 yv = y2[q];
      const double2 wv = w2[q];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const double2 v = __ldg(vg[g] + q);
        ay[g] = fma(v.y, yv.y, fma(v.x, yv.x, ay[g]));
        if (kW) aw[g] = fma(v.y, wv.y, fma(v.x, wv.x, aw[g]));
      }
      yy = fma(yv.y, yv.y, fma(yv.x, yv.x, yy));
      if (kW) yw = fma(yv.y, wv.y, fma(yv.x, wv.x, yw));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd length: the last row
      const double yl = y[n - 1], wl = kW ? w[n - 1] : 0.0;
#pragma unroll
      for (int g = 0; g < kG; ++g)
        if (g < ng) {
          const double vl = V[ld * (i0 + g) + (n - 1)];
          ay[g] = fma(vl, yl, ay[g]);
          aw[g] = fma(vl, wl, aw[g]);
        }
      yy = fma(yl, yl, yy);
      yw = fma(yl, wl, yw);
    }
#pragma unroll
    for (int g = 0; g < 2 * kG + 2; ++g) {
      double v = g < kG ? ay[g] : (g < 2 * kG ? aw[g - kG] : (g == 2 * kG ? yy : yw));
      for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) sh[warp][g] = v;
    }
    __syncthreads();
    if (threadIdx.x < 2 * kG + 2) {
      const int g = threadIdx.x;
      int vec = -1;
      if (g < kG) {
        if (g < ng) vec = i0 + g;
      } else if (g < 2 * kG) {
        if (g - kG < ng) vec = nq + i0 + g - kG;
      } else if (first) {
        vec = 2 * nq + (g - 2 * kG);
      }
      if (vec >= 0) {
        double t = 0.0;
        for (int k = 0; k < kThreads / 32; ++k) t += sh[k][g];
        red.partials[static_cast<size_t>(vec) * red.nblk + blockIdx.x] = (kW || g < kG || g == 2 * kG) ? t : 0.0;
      }
    }
    __syncthreads();
  }
}

template <int kG, bool kW>
__global__ void __launch_bounds__(kThreads, 1) dcgs2_dot_kernel(int n, int j, const double* __restrict__ V,
                                                             size_t ld, const double* __restrict__ w,
                                                             Reducer red, Small s, Dcgs d, int local) {
  dot_sweep<kG, kW>(n, j, V, ld, w, red);
  if (last_block(red)) {
    finish(red, 2 * j + 2, d.dots, 0);
    if (local) return;  // distributed: the sums are all-reduced first (dcgs2_fix_kernel)
    __syncthreads();
    dcgs2_fix(s, d, j, !kW);
  }
}

__global__ void __launch_bounds__(kThreads) dcgs2_fix_kernel(Small s, Dcgs d, int j, int finalize_only) {
  dcgs2_fix(s, d, j, finalize_only != 0);
}

// Preliminary rotation of column j once nu[j+1] = ||y_{j+1}|| is final, and
// the iteration's status (one CTA; gs aliases free shared memory).
__device__ void dcgs2_prelim(const Small& s, const Dcgs& d, int j, double denom, GivensStage& gs) {
  __shared__ double hn_s;
  const int m = s.m;
  if (threadIdx.x == 0) {
    hn_s = d.nu[j + 1];
    d.Hraw[static_cast<size_t>(j) * (m + 1) + j + 1] = hn_s;
  }
  __syncthreads();
  // preliminary rotation of column j (the final one follows its
  // reorthogonalisation in the next sweep 1)
  stage_givens(gs, s, d.Hraw + static_cast<size_t>(j) * (m + 1), j);
  if (threadIdx.x == 0) {
    const double hn = hn_s;
    double cs, sn;
    rotate_staged(gs, j, cs, sn);
    const double gj1 = -sn * s.g[j];
    s.status[0] = fabs(gj1) / denom;
    s.status[1] = !(hn >= 1e-14) ? 1.0 : 0.0;
    s.status[2] = hn;
  }
}

// distributed: nu[j+1] holds the all-reduced sum of squares
__global__ void __launch_bounds__(kThreads) dcgs2_prelim_kernel(Small s, Dcgs d, int j, double denom) {
  __shared__ GivensStage gs;
  if (threadIdx.x == 0) d.nu[j + 1] = sqrt(d.nu[j + 1]);
  __syncthreads();
  dcgs2_prelim(s, d, j, denom, gs);
}

// Sweep 2: q_j = (y/nu - Q s)/rho over slot j (in place) and
// y_{j+1} = (w/nu - Q t - c q_j)/rho into slot j+1, ||y_{j+1}|| reduced; the
// last CTA forms the preliminary rotation of column j and the status.
// n_dot <= n: rows counted in the norm (a distributed rank's own rows);
// local: leave the sum of squares in nu[j+1] for the all-reduce.
// the coefficients and (last CTA, after the sweep) the Givens stage share
// one shared-memory buffer: more CTAs per SM for the sweep
constexpr int kCoefElems = 2 * (kMaxRestart + 12);
constexpr int kStageElems = (sizeof(GivensStage) + sizeof(double) - 1) / sizeof(double);
constexpr int kSbufElems = kCoefElems > kStageElems ? kCoefElems : kStageElems;

// the sweep of dcgs2_axpy_kernel; this CTA's sum of squares -> partials[cta]
__device__ __forceinline__ void axpy_sweep(int n, int j, double* V, size_t ld,
                                           const double* __restrict__ w, const Small& s,
                                           const Dcgs& d, Reducer red, int n_dot, double* sbuf) {
  double* sS = sbuf;
  double* sT = sbuf + kMaxRestart + 12;
  __shared__ double sh[kThreads / 32];
  const int m = s.m;
  for (int i = threadIdx.x; i < j; i += blockDim.x) {
    sS[i] = d.coef[i];
    sT[i] = d.coef[m + 1 + i];
  }
  const double c = d.coef[2 * m + 2], rho = d.coef[2 * m + 3], nu = d.coef[2 * m + 4];
  const bool ok = d.coef[2 * m + 5] != 0.0;
  __syncthreads();
  double* y = V + ld * j;
  double* yn = V + ld * (j + 1);
  double2* y2 = reinterpret_cast<double2*>(y);
  double2* yn2 = reinterpret_cast<double2*>(yn);
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const int npair = n >> 1;
  double acc = 0.0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npair; q += gridDim.x * blockDim.x) {
    const double2 yv = y2[q], wv = w2[q];
    double ux = ok ? yv.x / nu : 0.0, uy = ok ? yv.y / nu : 0.0;
    double wx = ok ? wv.x / nu : 0.0, wy = ok ? wv.y / nu : 0.0;
    // multiaxpy-style: a short unrolled loop per thread, many warps per SM
    // keep the basis stream in flight
#pragma unroll 8
    for (int i = 0; i < j; ++i) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(V + ld * i) + q);
      ux = fma(-sS[i], v.x, ux);
      uy = fma(-sS[i], v.y, uy);
      wx = fma(-sT[i], v.x, wx);
      wy = fma(-sT[i], v.y, wy);
    }
    const double qx = ux / rho, qy = uy / rho;
    const double nx = fma(-c, qx, wx) / rho, ny = fma(-c, qy, wy) / rho;
    y2[q] = make_double2(qx, qy);
    yn2[q] = make_double2(nx, ny);
    if (2 * q < n_dot) acc = fma(nx, nx, acc);
    if (2 * q + 1 < n_dot) acc = fma(ny, ny, acc);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd length: the last row
    double ul = ok ? y[n - 1] / nu : 0.0, wl = ok ? w[n - 1] / nu : 0.0;
    for (int i = 0; i < j; ++i) {
      const double v = V[ld * i + (n - 1)];
      ul = fma(-sS[i], v, ul);
      wl = fma(-sT[i], v, wl);
    }
    const double ql = ul / rho, nl = fma(-c, ql, wl) / rho;
    y[n - 1] = ql;
    yn[n - 1] = nl;
    if (n - 1 < n_dot) acc = fma(nl, nl, acc);
  }
  const double bs = block_sum(acc, sh);
  if (threadIdx.x == 0) red.partials[blockIdx.x] = bs;
}

__global__ void __launch_bounds__(kThreads) dcgs2_axpy_kernel(int n, int j, double* V, size_t ld,
                                                              const double* __restrict__ w, Small s,
                                                              Dcgs d, Reducer red, double denom,
                                                              int n_dot, int local) {
  __shared__ __align__(16) double sbuf[kSbufElems];
  axpy_sweep(n, j, V, ld, w, s, d, red, n_dot, sbuf);
  if (last_block(red)) {
    if (local) {
      finish(red, 1, d.nu + j + 1, 0);
      return;
    }
    finish(red, 1, d.nu + j + 1, 1);
    GivensStage& gs = *reinterpret_cast<GivensStage*>(sbuf);  // coefficients no longer read
    dcgs2_prelim(s, d, j, denom, gs);
  }
}

// ---- one cooperative kernel per DCGS2 step, for short vectors (cfg1 /
// cfg2), where the two sweeps are latency-bound: grid-wide barriers replace
// the last-CTA hand-offs, and every CTA helps reduce the per-CTA partials,
// so only the Givens work stays on one CTA.
namespace cg = cooperative_groups;

__device__ __forceinline__ void grid_finish(Reducer red, int nvec, double* out, int mode) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp, nw = gridDim.x * (blockDim.x >> 5);
  for (int i = gw; i < nvec; i += nw) {
    const double* pr = red.partials + static_cast<size_t>(i) * red.nblk;
    double v = 0.0;
    for (int c = lane; c < red.nblk; c += 32) v += __ldcg(pr + c);
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) out[i] = mode == 1 ? sqrt(v) : v;
  }
}

__global__ void __launch_bounds__(kThreads, 1) dcgs2_step_coop_kernel(int n, int j, double* V, size_t ld,
                                                                   const double* __restrict__ w,
                                                                   Reducer red, Small s, Dcgs d,
                                                                   double denom) {
  cg::grid_group grid = cg::this_grid();
  __shared__ __align__(16) double sbuf[kSbufElems];
  dot_sweep<8, true>(n, j, V, ld, w, red);
  grid.sync();
  grid_finish(red, 2 * j + 2, d.dots, 0);
  grid.sync();
  if (blockIdx.x == 0) dcgs2_fix(s, d, j, false);
  grid.sync();
  axpy_sweep(n, j, V, ld, w, s, d, red, n, sbuf);
  grid.sync();
  if (blockIdx.x == 0) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
      double v = 0.0;
      for (int c = lane; c < red.nblk; c += 32) v += __ldcg(red.partials + c);
      for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) d.nu[j + 1] = sqrt(v);
    }
    __syncthreads();
    GivensStage& gs = *reinterpret_cast<GivensStage*>(sbuf);
    dcgs2_prelim(s, d, j, denom, gs);
  }
}

struct Vec {
  DevBuf buf;
  double* p() const { return buf.as<double>(); }
};

struct Workspace {
  Ctx* ctx;
  int n, nblk;
  DevBuf partials, counter, small;
  Reducer red;
  explicit Workspace(Ctx* c, int n_, int maxvec) : ctx(c), n(n_) {
    nblk = std::max(1, std::min(c->sm_count * 4, (n + kThreads - 1) / kThreads));
    partials = DevBuf(sizeof(double) * static_cast<size_t>(nblk) * std::max(1, maxvec));
    counter = DevBuf(sizeof(unsigned int) * 4);
    MSCG_CUDA(cudaMemsetAsync(counter.p, 0, counter.bytes, c->stream));
    red = {partials.as<double>(), counter.as<unsigned int>(), nblk};
  }
  void nrm2(const double* x, double* out) {
    nrm2_kernel<<<nblk, kThreads, 0, ctx->stream>>>(n, x, red, out);
    MSCG_CUDA(cudaGetLastError());
    ctx->launches++;
  }
  double host_nrm2(const double* x, double* dev_slot) {
    nrm2(x, dev_slot);
    double h = 0;
    MSCG_CUDA(cudaMemcpyAsync(&h, dev_slot, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    MSCG_CUDA(cudaStreamSynchronize(ctx->stream));
    return h;
  }
  int grid() const { return nblk; }
};

}  // namespace

namespace {
// ||b - A x|| / ||b|| with caller-provided scratch (r: n doubles, slot: 2).
double true_residual_ws(Workspace& ws, const DevCsr& a, const double* x, const double* b,
                        double* r, double* slot) {
  spmv(a, x, r, b, 1, ws.ctx->stream);
  const double rn = ws.host_nrm2(r, slot);
  const double bn = ws.host_nrm2(b, slot + 1);
  return bn == 0.0 ? rn : rn / bn;
}
}  // namespace

double true_residual(Ctx* ctx, const DevCsr& a, const double* x, const double* b) {
  const int n = a.nrows;
  Workspace ws(ctx, n, 1);
  DevBuf r(sizeof(double) * std::max(1, n)), slot(sizeof(double) * 2);
  return true_residual_ws(ws, a, x, b, r.as<double>(), slot.as<double>());
}

GmresResult gmres(Ctx* ctx, const DevCsr& a, Precond* pc, const double* b, double* x,
                  const GmresConfig& cfg) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const int n = a.nrows;
  if (a.ncols != n) throw Error(1, "gmres: dimension mismatch");
  if (pc && pc->n != n) throw Error(1, "gmres: preconditioner dimension mismatch");
  if (cfg.restart < 1 || !(cfg.rel_tol > 0.0) || cfg.max_iters < 1)
    throw Error(1, "gmres: bad solver configuration");
  if (cfg.restart > 500) throw Error(1, "gmres: restart above 500 is not supported");
  cudaStream_t s = ctx->stream;
  const int m = cfg.restart;
  const bool left = pc && cfg.left, right = pc && !cfg.left;
  GmresResult res;

  const bool dcgs2 = cfg.orth == 2;
  Workspace ws(ctx, n, 2 * m + 4);
  const int G = ws.grid();
  // basis columns 256-byte aligned (16-byte pair loads in the CGS2 kernels)
  const size_t ld = (static_cast<size_t>(n) + 31) & ~static_cast<size_t>(31);
  DevBuf V(sizeof(double) * ld * (m + 1)), w(sizeof(double) * n), tmp(sizeof(double) * n);
  DevBuf small(sizeof(double) * (static_cast<size_t>(m + 1) * m + 4 * (m + 1) + 64));
  double* sp = small.as<double>();
  Small st;
  st.m = m;
  st.H = sp;
  st.cs = st.H + static_cast<size_t>(m + 1) * m;
  st.sn = st.cs + (m + 1);
  st.g = st.sn + (m + 1);
  st.y = st.g + (m + 1);
  st.scal = st.y + (m + 1);
  st.status = st.scal + 16;
  double* hbuf = st.scal + 32;  // scratch for multidot results (<= m+1)
  DevBuf hscratch(sizeof(double) * 2 * (m + 2));
  // DCGS2 state: raw Hessenberg, sweep-1 sums, sweep-2 coefficients, norms
  const size_t ldh = static_cast<size_t>(m + 1);
  DevBuf dstate(dcgs2 ? sizeof(double) * (ldh * m + (2 * m + 4) + (2 * m + 8) + (m + 2)) : 8);
  Dcgs dc{};
  if (dcgs2) {
    dc.Hraw = dstate.as<double>();
    dc.dots = dc.Hraw + ldh * m;
    dc.coef = dc.dots + (2 * m + 4);
    dc.nu = dc.coef + (2 * m + 8);
    MSCG_CUDA(cudaMemsetAsync(dstate.p, 0, dstate.bytes, s));
  }
  // MSCG_CGS2_FUSED=0: the four-sweep CGS2 (two multi-dot + multi-axpy pairs)
  const char* fused_env = std::getenv("MSCG_CGS2_FUSED");
  const bool cgs2_fused = !(fused_env && fused_env[0] == '0');
  // Short vectors (n < 2^18: cfg1 / cfg2): one cooperative kernel per DCGS2
  // step (MSCG_DCGS2_COOP=0|1 forces it off / on), as many CTAs as fit at
  // once and as the partials buffer holds
  int coop_grid = 0;
  if (dcgs2) {
    const char* ce = std::getenv("MSCG_DCGS2_COOP");
    const bool want = ce ? ce[0] == '1' : n < (1 << 18);
    int coop = 0, per_sm = 0, dev = 0;
    MSCG_CUDA(cudaGetDevice(&dev));
    MSCG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    MSCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dcgs2_step_coop_kernel, kThreads, 0));
    if (want && coop && per_sm > 0) coop_grid = std::max(1, std::min(per_sm * ctx->sm_count, G));
  }
  // MSCG_DOT16=0|1 forces the group size (tests: both give bit-identical sums)
  const char* dot16_env = std::getenv("MSCG_DOT16");
  const bool dot16 = dot16_env ? dot16_env[0] == '1' : G >= 4 * ctx->sm_count;
  // The fused kernel re-reads each thread's basis rows after its axpy: fewer
  // resident rows keep that footprint (rows x (j+1) x 8 B) inside L2.
  const char* cps_env = std::getenv("MSCG_AXPYDOT_CPS");
  const int cps = cps_env ? std::max(1, std::atoi(cps_env)) : 1;
  const int G_ad = std::max(1, std::min(G, ctx->sm_count * cps));
  Reducer red_ad = ws.red;
  red_ad.nblk = G_ad;
  // page-locked status slots (two iterations in flight) and their events
  struct HostStatus {
    double* p = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~HostStatus() {
      if (p) cudaFreeHost(p);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
    }
  } hs;
  MSCG_CUDA(cudaMallocHost(&hs.p, 8 * sizeof(double)));
  for (auto& e : hs.ev) MSCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  double* hstat = hs.p;
  cudaEvent_t* hev = hs.ev;
  MSCG_CUDA(cudaMemsetAsync(small.p, 0, small.bytes, s));
  fill_kernel<<<G, kThreads, 0, s>>>(n, 0.0, x);
  ctx->launches++;
  (void)hbuf;

  auto apply_op = [&](const double* in, double* out) {
    // out = A B^-1 in (right) | B^-1 A in (left) | A in
    if (right) {
      pc->apply(in, tmp.as<double>(), s);
      spmv(a, tmp.as<double>(), out, nullptr, 0, s);
    } else if (left) {
      spmv(a, in, tmp.as<double>(), nullptr, 0, s);
      pc->apply(tmp.as<double>(), out, s);
    } else {
      spmv(a, in, out, nullptr, 0, s);
    }
  };

  const double norm_b = ws.host_nrm2(b, st.scal + 2);
  if (norm_b == 0.0) {
    res.converged = true;
    res.history.push_back(0.0);
    res.seconds = std::chrono::duration<double>(clk::now() - t0).count();
    return res;
  }
  double denom = norm_b;
  if (left) {
    pc->apply(b, w.as<double>(), s);
    denom = ws.host_nrm2(w.as<double>(), st.scal + 2);
  }
  if (denom == 0.0) denom = norm_b;

  double last_true = 1.0, prev_cycle_true = -1.0;
  bool done = false;
  double* vbase = V.as<double>();
  while (!done) {
    // r = b - A x (into V_0), left: B^-1 r.
    spmv(a, x, vbase, b, 1, s);
    if (left) {
      MSCG_CUDA(cudaMemcpyAsync(tmp.as<double>(), vbase, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      pc->apply(tmp.as<double>(), vbase, s);
    }
    const double beta = ws.host_nrm2(vbase, st.scal + 1);
    const double rel0 = beta / denom;
    if (res.history.empty()) res.history.push_back(rel0);
    if (rel0 <= cfg.rel_tol) {
      last_true = true_residual_ws(ws, a, x, b, tmp.as<double>(), st.scal + 4);
      res.converged = last_true <= cfg.rel_tol;
      break;
    }
    if (dcgs2) {
      // slot 0 keeps r unnormalised (y_0, nu_0 = beta): q_0 = r / beta is
      // formed by the first iteration's sweep 2
      init_cycle_kernel<<<1, 128, 0, s>>>(st, st.scal + 1, dc.nu);
      ctx->launches += 1;
      MSCG_CUDA(cudaMemsetAsync(dc.Hraw, 0, sizeof(double) * ldh * m, s));
    } else {
      scale_div_kernel<<<G, kThreads, 0, s>>>(n, vbase, st.scal + 1, vbase);
      init_cycle_kernel<<<1, 128, 0, s>>>(st, st.scal + 1, nullptr);
      ctx->launches += 2;
    }

    int mm = 0;
    bool breakdown = false, inner_conv = false;
    // Iteration j+1 is enqueued before iteration j's status is read, so the
    // device never idles across the host round trip; if j ends the cycle the
    // speculative iteration only touched H(:, j+1), g[j+1..j+2] and V_{j+2},
    // none of which the cycle's solution uses.
    auto enqueue_iteration = [&](int j) {
      double* vj = vbase + ld * j;
      double* wp = w.as<double>();
      apply_op(vj, wp);
      double* Hc = st.H + static_cast<size_t>(j) * (m + 1);
      if (dcgs2) {
        // two basis sweeps; the status comes from sweep 2's last CTA (or the
        // cooperative step kernel for short vectors)
        if (coop_grid > 0) {
          Reducer rc = ws.red;
          rc.nblk = coop_grid;
          int jj = j;
          double dn = denom;
          int nn = n;
          size_t lld = ld;
          void* args[] = {&nn, &jj, &vbase, &lld, &wp, &rc, &st, &dc, &dn};
          MSCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dcgs2_step_coop_kernel),
                                                coop_grid, kThreads, args, 0, s));
          ctx->launches += 1;
        } else {
          (dot16 ? dcgs2_dot_kernel<16, true> : dcgs2_dot_kernel<8, true>)<<<G, kThreads, 0, s>>>(
              n, j, vbase, ld, wp, ws.red, st, dc, 0);
          dcgs2_axpy_kernel<<<G, kThreads, 0, s>>>(n, j, vbase, ld, wp, st, dc, ws.red, denom, n, 0);
          ctx->launches += 2;
        }
        MSCG_CUDA(cudaMemcpyAsync(hstat + 4 * (j & 1), st.status, 3 * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
        MSCG_CUDA(cudaEventRecord(hev[j & 1], s));
        return;
      }
      if (cfg.orth == 0) {
        // MGS: for i <= j: h_ij = v_i . w ; w -= h_ij v_i (fused pairwise).
        for (int i = 0; i <= j; ++i) {
          mgs_kernel<<<G, kThreads, 0, s>>>(n, i ? vbase + ld * (i - 1) : nullptr,
                                            i ? Hc + (i - 1) : nullptr, vbase + ld * i, wp,
                                            ws.red, Hc + i);
          ctx->launches++;
        }
        mgs_kernel<<<G, kThreads, 0, s>>>(n, vbase + ld * j, Hc + j, nullptr, wp, ws.red, nullptr);
        ctx->launches++;
      } else {
        // CGS2: h = V^T w; w -= V h; twice, H(:,j) = h1 + h2.
        if (cgs2_fused) {
          // dot, fused axpy + dot, axpy: three sweeps over the basis
          (dot16 ? multidot_kernel<16> : multidot_kernel<8>)<<<G, kThreads, 0, s>>>(n, j + 1, vbase, ld, wp, ws.red,
                                                 hscratch.as<double>());
          axpy_dot_kernel<<<G_ad, kThreads, 0, s>>>(n, j + 1, vbase, ld, hscratch.as<double>(), wp,
                                                    Hc, red_ad, hscratch.as<double>() + (m + 2));
          multiaxpy_kernel<<<G, kThreads, 0, s>>>(n, j + 1, vbase, ld,
                                                  hscratch.as<double>() + (m + 2), wp, Hc, 1);
          ctx->launches += 3;
        } else
        for (int pass = 0; pass < 2; ++pass) {
          (dot16 ? multidot_kernel<16> : multidot_kernel<8>)<<<G, kThreads, 0, s>>>(n, j + 1, vbase, ld, wp, ws.red,
                                                 hscratch.as<double>());
          multiaxpy_kernel<<<G, kThreads, 0, s>>>(n, j + 1, vbase, ld, hscratch.as<double>(), wp,
                                                  Hc, pass);
          ctx->launches += 2;
        }
      }
      ws.nrm2(wp, st.scal + 0);
      // v_{j+1} = w / hnext; on breakdown the (unused) vector is never referenced.
      scale_div_kernel<<<G, kThreads, 0, s>>>(n, wp, st.scal + 0, vbase + ld * (j + 1));
      givens_kernel<<<1, 32, 0, s>>>(st, j, denom);
      ctx->launches += 2;
      MSCG_CUDA(cudaMemcpyAsync(hstat + 4 * (j & 1), st.status, 3 * sizeof(double),
                                cudaMemcpyDeviceToHost, s));
      MSCG_CUDA(cudaEventRecord(hev[j & 1], s));
    };
    const int jmax = std::min(m, cfg.max_iters - res.iterations);
    if (jmax > 0) enqueue_iteration(0);
    for (int j = 0; j < jmax; ++j) {
      if (j + 1 < jmax) enqueue_iteration(j + 1);
      MSCG_CUDA(cudaEventSynchronize(hev[j & 1]));
      const double* status = hstat + 4 * (j & 1);
      breakdown = status[1] != 0.0;
      ++res.iterations;
      mm = j + 1;
      const double rel = status[0];
      res.history.push_back(rel);
      if (breakdown || rel <= cfg.rel_tol) {
        inner_conv = rel <= cfg.rel_tol;
        break;
      }
    }
    if (dcgs2 && mm > 0 && mm >= jmax) {
      // no speculative iteration in the stream: finalise column mm-1 with
      // one dot sweep of y_mm against q_0..q_{mm-1}
      (dot16 ? dcgs2_dot_kernel<16, false> : dcgs2_dot_kernel<8, false>)<<<G, kThreads, 0, s>>>(
          n, mm, vbase, ld, nullptr, ws.red, st, dc, 0);
      ctx->launches++;
    }
    backsolve_kernel<<<1, 32, 0, s>>>(st, mm);
    double* z = w.as<double>();
    combine_kernel<<<G, kThreads, 0, s>>>(n, mm, vbase, ld, st.y, z);
    ctx->launches += 2;
    if (right) {
      pc->apply(z, tmp.as<double>(), s);
      z = tmp.as<double>();
    }
    axpy1_kernel<<<G, kThreads, 0, s>>>(n, z, x);
    ctx->launches++;
    last_true = true_residual_ws(ws, a, x, b, w.as<double>(), st.scal + 4);
    if (last_true <= cfg.rel_tol) {
      res.converged = true;
      done = true;
    } else if (breakdown) {
      res.converged = false;
      done = true;
    } else if (res.iterations >= cfg.max_iters) {
      res.converged = false;
      done = true;
    } else if (inner_conv) {
      if (prev_cycle_true >= 0.0 && last_true >= 0.999 * prev_cycle_true) {
        res.converged = false;
        done = true;
      }
    }
    prev_cycle_true = last_true;
    static const bool verbose = getenv("MSCG_VERBOSE") != nullptr;
    if (verbose)
      fprintf(stderr, "gmres: cycle done, %d iterations, %.3f s, true residual %.3e\n",
              res.iterations, std::chrono::duration<double>(clk::now() - t0).count(), last_true);
  }
  res.history.push_back(last_true);
  res.final_true = last_true;
  MSCG_CUDA(cudaStreamSynchronize(s));
  res.seconds = std::chrono::duration<double>(clk::now() - t0).count();
  return res;
}

// ---------------------------------------------------------------------------
// Distributed right-preconditioned GMRES over preconditioner shards (SURVEY
// 8(e)): rank r owns the interior rows [lo, hi) of its blocks; every Krylov
// vector is stored compact, [own interior rows | interface], the interface
// part replicated (every rank computes it from the same all-reduced
// numbers, so the copies stay bit-identical).  Per iteration:
//   operator   apply_shard_begin -> all-reduce t (n_g) -> apply_shard_end;
//              spmv_shard -> all-reduce the interface rows (n_g)
//   DCGS2      sweep 1 local dots -> all-reduce (2j+2) -> fix (one CTA);
//              sweep 2 local sum of squares -> all-reduce (1) -> rotation
// Dots and norms count the interface rows on rank 0 only.  `comm.sum`
// reduces in stream order (the caller's all-reduce runs on the context
// stream: NCCL, or gloo on CUDA tensors).
GmresResult gmres_shard(Ctx* ctx, Precond* sh, const double* b_glob, double* x_glob,
                        const GmresConfig& cfg, const DistComm& comm) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  if (!sh || !sh->shard.on) throw Error(1, "gmres_shard: not a shard preconditioner");
  if (cfg.left) throw Error(1, "gmres_shard: right preconditioning only");
  if (cfg.orth != 2) throw Error(1, "gmres_shard: DCGS2 orthogonalisation only");
  if (cfg.restart < 1 || !(cfg.rel_tol > 0.0) || cfg.max_iters < 1)
    throw Error(1, "gmres: bad solver configuration");
  if (cfg.restart > kMaxRestart) throw Error(1, "gmres: restart above 500 is not supported");
  const int n = sh->n, p = sh->p, ng = n - p;
  const int lo = sh->shard.row_lo, hi = sh->shard.row_hi, own = hi - lo;
  const int nl = own + ng, n_dot = own + (comm.rank == 0 ? ng : 0);
  const int m = cfg.restart;
  if (comm.cap < std::max(2 * m + 4, std::max(ng, 1)))
    throw Error(1, "gmres_shard: communication buffer too small");
  cudaStream_t s = ctx->stream;
  GmresResult res;
  Workspace ws(ctx, std::max(nl, 1), 2 * m + 4);
  const int G = ws.grid();
  const size_t ld = (static_cast<size_t>(nl) + 31) & ~static_cast<size_t>(31);
  DevBuf V(sizeof(double) * ld * (m + 1)), w(sizeof(double) * ld), tmp(sizeof(double) * ld),
      bc(sizeof(double) * ld), xc(sizeof(double) * ld);
  DevBuf gy(sizeof(double) * n), gx(sizeof(double) * n), gw(sizeof(double) * n),
      tpart(sizeof(double) * std::max(1, ng)), y2p(sizeof(double) * std::max(1, ng));
  DevBuf small(sizeof(double) * (static_cast<size_t>(m + 1) * m + 4 * (m + 1) + 64));
  double* sp = small.as<double>();
  Small st;
  st.m = m;
  st.H = sp;
  st.cs = st.H + static_cast<size_t>(m + 1) * m;
  st.sn = st.cs + (m + 1);
  st.g = st.sn + (m + 1);
  st.y = st.g + (m + 1);
  st.scal = st.y + (m + 1);
  st.status = st.scal + 16;
  const size_t ldh = static_cast<size_t>(m + 1);
  DevBuf dstate(sizeof(double) * (ldh * m + (2 * m + 4) + (2 * m + 8) + (m + 2)));
  Dcgs dc{};
  dc.Hraw = dstate.as<double>();
  dc.dots = dc.Hraw + ldh * m;
  dc.coef = dc.dots + (2 * m + 4);
  dc.nu = dc.coef + (2 * m + 8);
  MSCG_CUDA(cudaMemsetAsync(dstate.p, 0, dstate.bytes, s));
  MSCG_CUDA(cudaMemsetAsync(small.p, 0, small.bytes, s));
  MSCG_CUDA(cudaMemsetAsync(gy.p, 0, gy.bytes, s));
  MSCG_CUDA(cudaMemsetAsync(gx.p, 0, gx.bytes, s));
  MSCG_CUDA(cudaMemsetAsync(gw.p, 0, gw.bytes, s));
  const char* dot16_env = std::getenv("MSCG_DOT16");
  const bool dot16 = dot16_env ? dot16_env[0] == '1' : G >= 4 * ctx->sm_count;

  auto sum = [&](double* d, int count) {  // all-reduce in stream order
    if (comm.size <= 1 || count <= 0) return;
    MSCG_CUDA(cudaMemcpyAsync(comm.buf, d, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
    comm.allreduce(count, comm.user);
    MSCG_CUDA(cudaMemcpyAsync(d, comm.buf, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
  };
  auto to_global = [&](const double* c, double* g) {
    if (own) MSCG_CUDA(cudaMemcpyAsync(g + lo, c, sizeof(double) * own, cudaMemcpyDeviceToDevice, s));
    if (ng) MSCG_CUDA(cudaMemcpyAsync(g + p, c + own, sizeof(double) * ng, cudaMemcpyDeviceToDevice, s));
  };
  auto from_global = [&](const double* g, double* c) {
    if (own) MSCG_CUDA(cudaMemcpyAsync(c, g + lo, sizeof(double) * own, cudaMemcpyDeviceToDevice, s));
    if (ng) MSCG_CUDA(cudaMemcpyAsync(c + own, g + p, sizeof(double) * ng, cudaMemcpyDeviceToDevice, s));
  };
  auto op_a = [&](const double* xin, double* yout) {  // yout = C xin (compact)
    to_global(xin, gx.as<double>());
    sh->spmv_shard(gx.as<double>(), gw.as<double>(), y2p.as<double>(), comm.rank == 0, s);
    sum(y2p.as<double>(), ng);
    if (own) MSCG_CUDA(cudaMemcpyAsync(yout, gw.as<double>() + lo, sizeof(double) * own, cudaMemcpyDeviceToDevice, s));
    if (ng) MSCG_CUDA(cudaMemcpyAsync(yout + own, y2p.p, sizeof(double) * ng, cudaMemcpyDeviceToDevice, s));
  };
  auto op_minv = [&](const double* yin, double* xout) {  // xout = B^-1 yin (compact)
    to_global(yin, gy.as<double>());
    sh->apply_shard_begin(gy.as<double>(), tpart.as<double>(), s);
    sum(tpart.as<double>(), ng);
    sh->apply_shard_end(gy.as<double>(), tpart.as<double>(), gx.as<double>(), s);
    from_global(gx.as<double>(), xout);
  };
  auto norm = [&](const double* x, double* slot) {  // global 2-norm, device slot + host value
    sumsq_kernel<<<G, kThreads, 0, s>>>(n_dot, x, ws.red, slot);
    ctx->launches++;
    sum(slot, 1);
    sqrt_kernel<<<1, 1, 0, s>>>(slot);
    double h = 0;
    MSCG_CUDA(cudaMemcpyAsync(&h, slot, sizeof(double), cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaStreamSynchronize(s));
    return h;
  };
  struct HostStatus {
    double* p = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~HostStatus() {
      if (p) cudaFreeHost(p);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
    }
  } hs;
  MSCG_CUDA(cudaMallocHost(&hs.p, 8 * sizeof(double)));
  for (auto& e : hs.ev) MSCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

  from_global(b_glob, bc.as<double>());
  fill_kernel<<<G, kThreads, 0, s>>>(nl, 0.0, xc.as<double>());
  ctx->launches++;
  const double norm_b = norm(bc.as<double>(), st.scal + 2);
  auto finish_x = [&] {
    MSCG_CUDA(cudaMemsetAsync(x_glob, 0, sizeof(double) * n, s));
    to_global(xc.as<double>(), x_glob);
  };
  if (norm_b == 0.0) {
    res.converged = true;
    res.history.push_back(0.0);
    finish_x();
    MSCG_CUDA(cudaStreamSynchronize(s));
    res.seconds = std::chrono::duration<double>(clk::now() - t0).count();
    return res;
  }
  const double denom = norm_b;
  auto true_res = [&]() {
    op_a(xc.as<double>(), w.as<double>());
    sub2_kernel<<<G, kThreads, 0, s>>>(nl, bc.as<double>(), w.as<double>(), tmp.as<double>());
    ctx->launches++;
    return norm(tmp.as<double>(), st.scal + 4) / norm_b;
  };
  double last_true = 1.0, prev_cycle_true = -1.0;
  bool done = false;
  double* vbase = V.as<double>();
  while (!done) {
    op_a(xc.as<double>(), w.as<double>());  // r = b - A x into slot 0 (unnormalised y_0)
    sub2_kernel<<<G, kThreads, 0, s>>>(nl, bc.as<double>(), w.as<double>(), vbase);
    ctx->launches++;
    const double beta = norm(vbase, st.scal + 1);
    const double rel0 = beta / denom;
    if (res.history.empty()) res.history.push_back(rel0);
    if (rel0 <= cfg.rel_tol) {
      last_true = true_res();
      res.converged = last_true <= cfg.rel_tol;
      break;
    }
    init_cycle_kernel<<<1, 128, 0, s>>>(st, st.scal + 1, dc.nu);
    MSCG_CUDA(cudaMemsetAsync(dc.Hraw, 0, sizeof(double) * ldh * m, s));
    ctx->launches++;
    int mm = 0;
    bool breakdown = false, inner_conv = false;
    auto enqueue_iteration = [&](int j) {
      double* vj = vbase + ld * j;
      op_minv(vj, tmp.as<double>());
      op_a(tmp.as<double>(), w.as<double>());
      (dot16 ? dcgs2_dot_kernel<16, true> : dcgs2_dot_kernel<8, true>)<<<G, kThreads, 0, s>>>(
          n_dot, j, vbase, ld, w.as<double>(), ws.red, st, dc, 1);
      sum(dc.dots, 2 * j + 2);
      dcgs2_fix_kernel<<<1, kThreads, 0, s>>>(st, dc, j, 0);
      dcgs2_axpy_kernel<<<G, kThreads, 0, s>>>(nl, j, vbase, ld, w.as<double>(), st, dc, ws.red,
                                               denom, n_dot, 1);
      sum(dc.nu + j + 1, 1);
      dcgs2_prelim_kernel<<<1, kThreads, 0, s>>>(st, dc, j, denom);
      ctx->launches += 4;
      MSCG_CUDA(cudaMemcpyAsync(hs.p + 4 * (j & 1), st.status, 3 * sizeof(double),
                                cudaMemcpyDeviceToHost, s));
      MSCG_CUDA(cudaEventRecord(hs.ev[j & 1], s));
    };
    const int jmax = std::min(m, cfg.max_iters - res.iterations);
    if (jmax > 0) enqueue_iteration(0);
    for (int j = 0; j < jmax; ++j) {
      if (j + 1 < jmax) enqueue_iteration(j + 1);
      MSCG_CUDA(cudaEventSynchronize(hs.ev[j & 1]));
      const double* status = hs.p + 4 * (j & 1);
      breakdown = status[1] != 0.0;
      ++res.iterations;
      mm = j + 1;
      const double rel = status[0];
      res.history.push_back(rel);
      if (breakdown || rel <= cfg.rel_tol) {
        inner_conv = rel <= cfg.rel_tol;
        break;
      }
    }
    if (mm > 0 && mm >= jmax) {
      (dot16 ? dcgs2_dot_kernel<16, false> : dcgs2_dot_kernel<8, false>)<<<G, kThreads, 0, s>>>(
          n_dot, mm, vbase, ld, nullptr, ws.red, st, dc, 1);
      sum(dc.dots, 2 * mm + 2);
      dcgs2_fix_kernel<<<1, kThreads, 0, s>>>(st, dc, mm, 1);
      ctx->launches += 2;
    }
    backsolve_kernel<<<1, 32, 0, s>>>(st, mm);
    combine_kernel<<<G, kThreads, 0, s>>>(nl, mm, vbase, ld, st.y, w.as<double>());
    ctx->launches += 2;
    op_minv(w.as<double>(), tmp.as<double>());
    axpy1_kernel<<<G, kThreads, 0, s>>>(nl, tmp.as<double>(), xc.as<double>());
    ctx->launches++;
    last_true = true_res();
    if (last_true <= cfg.rel_tol) {
      res.converged = true;
      done = true;
    } else if (breakdown || res.iterations >= cfg.max_iters) {
      res.converged = false;
      done = true;
    } else if (inner_conv) {
      if (prev_cycle_true >= 0.0 && last_true >= 0.999 * prev_cycle_true) {
        res.converged = false;
        done = true;
      }
    }
    prev_cycle_true = last_true;
  }
  res.history.push_back(last_true);
  res.final_true = last_true;
  finish_x();
  MSCG_CUDA(cudaStreamSynchronize(s));
  res.seconds = std::chrono::duration<double>(clk::now() - t0).count();
  return res;
}

}  // namespace mscg
