// Block-diagonal triangular solve x_b = U_b^-1 L_b^-1 P_b r_b for every block
// of a FactorSet in one launch (reference `solve`, factorization.cpp:129-158,
// driven per block by block_solve, preconditioner.cpp:13-22).
//
// Design (B200, HBM-bound; SURVEY §7 "hard parts"):
//  * one CTA per block; the block's L-solve output z and U-solve output x
//    live in shared memory (2 x dim fp64, <= 54 KB at dim 3361);
//  * warp w owns rows w, w+NW, ... ("sync-free" scheduling): a warp streams
//    its row's (value, column) pairs from HBM with coalesced 256 B + 64 B
//    loads, independent of the dependency chain, and only the gather of
//    x[col] waits;
//  * readiness is encoded in the value itself: slots start as a signalling
//    NaN pattern (kPendingBits) that no arithmetic produces, so a consumer
//    spins on the 8-byte shared slot and never needs a flag or a fence;
//  * each row is reduced by the warp (lane-strided FMA partial sums +
//    butterfly shuffles); the rounding differs from the reference's
//    sequential sum by ~1e-16 relative, well inside the
//    1e-10 parity bar.
// Progress: row r's dependencies are rows < r (L) or > r (U); the smallest
// unfinished row always belongs to a warp whose earlier rows are done, so the
// spin never deadlocks while all NW warps of the CTA are resident.
#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kWarps = 16;
constexpr int kUnroll = 4;

struct TriArgs {
  const int* row0;
  const int* dim;
  const long long* loff;
  const long long* uoff;
  const int* lrp;
  const int* urp;
  const double* lval;
  const uint16_t* lcol;
  const double* uval;
  const uint16_t* ucol;
  const double* udiag;
  const int* perm;  // nullable
  int dim_max;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Dot product of one factor row with the (partially ready) solution vector.
__device__ __forceinline__ double row_dot(const double* __restrict__ vals,
                                          const uint16_t* __restrict__ cols, int s,
                                          int e, const double* sol, int lane) {
  double acc = 0.0;
  for (int k0 = s + lane; k0 < e; k0 += 32 * kUnroll) {
    double v[kUnroll];
    int c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int k = k0 + 32 * u;
      if (k < e) {
        v[u] = __ldg(vals + k);
        c[u] = __ldg(cols + k);
      } else {
        v[u] = 0.0;
        c[u] = -1;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (c[u] >= 0) acc = fma(v[u], wait_ready(sol + c[u]), acc);
  }
  return warp_sum(acc);
}

__global__ void __launch_bounds__(kWarps * 32) trisolve_kernel(TriArgs a,
                                                               const double* __restrict__ rhs,
                                                               double* __restrict__ out,
                                                               const double* __restrict__ sub) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const int n = a.dim[b], r0 = a.row0[b];
  double* z = sm;
  double* x = sm + a.dim_max;
  const double pend = pending_value();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    z[i] = pend;
    x[i] = pend;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* lr = a.lrp + r0 + b;
  const int* ur = a.urp + r0 + b;
  const double* lv = a.lval + a.loff[b];
  const uint16_t* lc = a.lcol + a.loff[b];
  const double* uv = a.uval + a.uoff[b];
  const uint16_t* uc = a.ucol + a.uoff[b];
  const int* pm = a.perm ? a.perm + r0 : nullptr;

  // Forward: z = L^-1 P r (unit lower).
  for (int i = warp; i < n; i += kWarps) {
    const double acc = row_dot(lv, lc, lr[i], lr[i + 1], z, lane);
    if (lane == 0) {
      const double bi = rhs[r0 + (pm ? pm[i] : i)];
      *reinterpret_cast<volatile double*>(z + i) = bi - acc;
    }
  }
  __syncthreads();
  // Backward: x = U^-1 z.
  for (int t = warp; t < n; t += kWarps) {
    const int i = n - 1 - t;
    const double acc = row_dot(uv, uc, ur[i], ur[i + 1], x, lane);
    if (lane == 0) {
      const double xi = (z[i] - acc) / a.udiag[r0 + i];
      *reinterpret_cast<volatile double*>(x + i) = xi;
      out[r0 + i] = sub ? sub[r0 + i] - xi : xi;
    }
  }
}

}  // namespace

void block_trisolve(const FactorSet& fs, const double* rhs, double* out, const double* sub,
                    cudaStream_t s) {
  if (fs.nblocks == 0) return;
  TriArgs a;
  a.row0 = fs.row0.as<int>();
  a.dim = fs.dim.as<int>();
  a.loff = fs.loff.as<long long>();
  a.uoff = fs.uoff.as<long long>();
  a.lrp = fs.lrp.as<int>();
  a.urp = fs.urp.as<int>();
  a.lval = fs.lval.as<double>();
  a.lcol = fs.lcol.as<uint16_t>();
  a.uval = fs.uval.as<double>();
  a.ucol = fs.ucol.as<uint16_t>();
  a.udiag = fs.udiag.as<double>();
  a.perm = fs.has_perm ? fs.perm.as<int>() : nullptr;
  a.dim_max = fs.max_dim;
  const size_t smem = 2 * sizeof(double) * static_cast<size_t>(fs.max_dim);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    MSCG_CUDA(cudaFuncSetAttribute(trisolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    configured = smem;
  }
  trisolve_kernel<<<fs.nblocks, kWarps * 32, smem, s>>>(a, rhs, out, sub);
  MSCG_CUDA(cudaGetLastError());
}

}  // namespace mscg
