// Block-diagonal triangular solve x_b = U_b^-1 L_b^-1 P_b r_b for every block
// of a FactorSet in one launch (reference `solve`, factorization.cpp:129-158,
// driven per block by block_solve, preconditioner.cpp:13-22).
//
// Why tiles (measured, SURVEY §8(a) A6 structure): an interior block of
// ~3000 rows is [velocities | pressures]; its L has a banded velocity part
// (~21 nnz/row, bandwidth <= 63), a wide velocity->pressure coupling
// (~450 nnz/row) and a ~45%-dense pressure triangle; U mirrors it.  The
// dependency chain is therefore ~one row deep per row in both triangles,
// while most bytes sit far from the diagonal.  The kernel splits every row
// at tile boundaries (kTile = 32 rows, near window = kNearTiles tiles):
//
//  * far entries (L: columns < 32(t-2), U: columns >= 32(t+3)) are streamed
//    from HBM by the worker warps, one warp per row (coalesced value/column
//    loads, 8-deep unrolled, next row's pointers prefetched), and reduced to
//    one partial sum per row into a small shared-memory ring -- they depend
//    only on tiles the chain finished two tiles earlier, so this traffic
//    runs ahead of the chain.  Banded velocity rows have no far entries and
//    never involve a worker;
//  * the near window (diagonal tile + the two neighbour tiles, dense
//    32 x 96 fp64, column-major) is brought into shared memory by TMA bulk
//    copies (cp.async.bulk + mbarrier ring issued by the solver warp) and
//    solved by one warp: lane j owns row j of the tile, neighbour tiles are
//    applied from registers via shuffles, and the 32-step diagonal chain
//    costs one shuffle + one FMA per row;
//  * z (L output) and x (U output) stay in shared memory; readiness is the
//    value itself (slots start as a signalling-NaN pattern no arithmetic
//    produces), so workers poll 8-byte slots without flags or fences, backing
//    off with __nanosleep to leave issue slots to the solver.
// Rounding differs from the reference's sequential row sums by ~1e-16
// relative, far inside the 1e-10 apply bar.
#include <cstdlib>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kWorkers = kWarps - 1;
constexpr int kUnroll = 8;
constexpr int kRing = 2;       // near-tile TMA ring depth
constexpr int kPartRing = 8;   // far-sum ring depth (tiles)
constexpr unsigned kTileBytes = kTileElems * sizeof(double);

struct TriArgs {
  const int* row0;
  const int* dim;
  const long long* loff;
  const long long* uoff;
  const long long* toff;
  const int* lrp;
  const int* urp;
  const double* lval;
  const uint16_t* lcol;
  const double* uval;
  const uint16_t* ucol;
  const double* ltile;
  const double* utile;
  const double* urdiag;
  const int* perm;  // nullable
  int dim_max;
  long long* trace;  // debug: clock64 stamps for block 0, or null
  unsigned sleep_ns; // worker back-off while polling (0 = spin)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Far-entry dot product of one row (all lanes), waiting per entry on sol.
__device__ __forceinline__ double far_dot(const double* __restrict__ vals,
                                          const uint16_t* __restrict__ cols, int s, int e,
                                          const double* sol, int lane, unsigned ns) {
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
      if (c[u] >= 0) acc = fma(v[u], (ns ? wait_ready_lazy(sol + c[u], ns) : wait_ready(sol + c[u])), acc);
  }
  return warp_sum(acc);
}

// sum_k T[(c0 + k) * 32 + j] * shfl(v, k) over one 32-column neighbour tile.
__device__ __forceinline__ double neighbour(const double* T, int c0, int j, double v) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int k = 0; k < kTile; k += 4) {
    a0 = fma(T[(c0 + k + 0) * kTile + j], __shfl_sync(0xffffffffu, v, k + 0), a0);
    a1 = fma(T[(c0 + k + 1) * kTile + j], __shfl_sync(0xffffffffu, v, k + 1), a1);
    a2 = fma(T[(c0 + k + 2) * kTile + j], __shfl_sync(0xffffffffu, v, k + 2), a2);
    a3 = fma(T[(c0 + k + 3) * kTile + j], __shfl_sync(0xffffffffu, v, k + 3), a3);
  }
  return (a0 + a1) + (a2 + a3);
}

__global__ void __launch_bounds__(kThreads) trisolve_kernel(TriArgs a,
                                                            const double* __restrict__ rhs,
                                                            double* __restrict__ out,
                                                            const double* __restrict__ sub) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                          // kRing near tiles
  double* part = ring + kRing * kTileElems;   // kPartRing x 32 far sums
  double* z = part + kPartRing * kTile;       // dim_max
  double* x = z + a.dim_max;                  // dim_max
  __shared__ __align__(8) uint64_t bars[kRing];
  __shared__ int done_l, done_u;

  const int b = blockIdx.x;
  const int n = a.dim[b], r0 = a.row0[b];
  const int nt = (n + kTile - 1) / kTile;
  const double* lt = a.ltile + a.toff[b] * kTileElems;
  const double* ut = a.utile + a.toff[b] * kTileElems;
  const int* lr = a.lrp + r0 + b;
  const int* ur = a.urp + r0 + b;
  const double pend = pending_value();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    z[i] = pend;
    x[i] = pend;
  }
  for (int i = threadIdx.x; i < kPartRing * kTile; i += blockDim.x) part[i] = pend;
  if (threadIdx.x == 0) {
    done_l = 0;
    done_u = 0;
    for (int r = 0; r < kRing; ++r) mbar_init(&bars[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Near-tile stream: items 0..nt-1 = L tiles 0..nt-1, items nt..2nt-1 = U
  // tiles nt-1..0.  Item q lives in ring slot q % kRing, phase (q / kRing) & 1.
  auto item_src = [&](int q) -> const double* {
    return q < nt ? lt + static_cast<long long>(q) * kTileElems
                  : ut + static_cast<long long>(2 * nt - 1 - q) * kTileElems;
  };
  auto refill = [&](int q_done) {  // solver warp: slot of q_done is free
    __syncwarp();
    const int q = q_done + kRing;
    if (lane == 0 && q < 2 * nt) {
      const int slot = q % kRing;
      mbar_expect_tx(&bars[slot], kTileBytes);
      bulk_load(ring + slot * kTileElems, item_src(q), kTileBytes, &bars[slot]);
    }
  };
  const int* pm = a.perm ? a.perm + r0 : nullptr;
  long long* tr = (a.trace && b == 0) ? a.trace : nullptr;
  const int j = lane;

  // ================================================================ L pass
  if (warp == 0) {
    if (lane == 0)
      for (int q = 0; q < kRing && q < 2 * nt; ++q) {
        mbar_expect_tx(&bars[q], kTileBytes);
        bulk_load(ring + q * kTileElems, item_src(q), kTileBytes, &bars[q]);
      }
    double zp1 = 0.0, zp2 = 0.0;  // z of tiles t-1, t-2 (lane k = row k)
    double bnext = 0.0;
    int fnext = 0;
    if (j < n) {
      bnext = rhs[r0 + (pm ? pm[j] : j)];
      fnext = lr[j + 1] - lr[j];
    }
    for (int t = 0; t < nt; ++t) {
      const int i = t * kTile + j;
      const bool valid = i < n;
      const double bi = bnext;
      const int nfar = fnext;
      const int in = i + kTile;  // prefetch next tile's scalars
      if (in < n) {
        bnext = rhs[r0 + (pm ? pm[in] : in)];
        fnext = lr[in + 1] - lr[in];
      }
      const int slot = t % kRing;
      mbar_wait(&bars[slot], (t / kRing) & 1);
      if (tr && lane == 0) tr[3 * t + 0] = clock64();
      const double* T = ring + slot * kTileElems;
      double nb = 0.0;
      if (t > 1) nb += neighbour(T, 0, j, zp2);
      if (t > 0) nb += neighbour(T, kTile, j, zp1);
      double td[kTile];
#pragma unroll
      for (int k = 0; k < kTile; ++k) td[k] = T[(2 * kTile + k) * kTile + j];
      double far = 0.0;
      if (valid && nfar > 0) {
        double* ps = part + (t % kPartRing) * kTile + j;
        far = wait_ready(ps);
        *ps = pend;
      }
      if (tr && lane == 0) tr[3 * t + 1] = clock64();
      // acc = b_i - (known sums); z_k = acc_k once step k is reached
      double acc = bi - (nb + far);
      double zj = 0.0;
#pragma unroll
      for (int k = 0; k < kTile; ++k) {
        const double zk = __shfl_sync(0xffffffffu, acc, k);
        if (j == k) zj = zk;
        if (j > k) acc = fma(-td[k], zk, acc);
      }
      if (!valid) zj = 0.0;
      if (valid) *reinterpret_cast<volatile double*>(z + i) = zj;
      zp2 = zp1;
      zp1 = zj;
      if (tr && lane == 0) tr[3 * t + 2] = clock64();
      refill(t);
      if (lane == 0) *reinterpret_cast<volatile int*>(&done_l) = t + 1;
    }
  } else {
    // workers: far sums of L rows, ascending
    const int w = warp - 1;
    const double* fv = a.lval + a.loff[b];
    const uint16_t* fc = a.lcol + a.loff[b];
    int sn = 0, en = 0;
    if (w < n) {
      sn = lr[w];
      en = lr[w + 1];
    }
    for (int i = w; i < n; i += kWorkers) {
      const int s = sn, e = en;
      if (i + kWorkers < n) {
        sn = lr[i + kWorkers];
        en = lr[i + kWorkers + 1];
      }
      if (e == s) continue;
      const int t = i / kTile;
      const double acc = far_dot(fv, fc, s, e, z, lane, a.sleep_ns);
      if (lane == 0) {
        // ring slot of tile t is free once tile t - kPartRing was consumed
        while (*reinterpret_cast<volatile int*>(&done_l) < t - (kPartRing - 1)) __nanosleep(128);
        *reinterpret_cast<volatile double*>(part + (t % kPartRing) * kTile + (i % kTile)) = acc;
      }
    }
  }
  __syncthreads();  // every L far sum consumed before U sums reuse the ring

  // ================================================================ U pass
  if (warp == 0) {
    double xn1 = 0.0, xn2 = 0.0;  // x of tiles t+1, t+2
    for (int tt = 0; tt < nt; ++tt) {
      const int t = nt - 1 - tt;
      const int q = nt + tt;
      const int i = t * kTile + j;
      const bool valid = i < n;
      double zi = 0.0, rd = 0.0, si = 0.0;
      int nfar = 0;
      if (valid) {
        zi = z[i];
        rd = a.urdiag[r0 + i];
        if (sub) si = sub[r0 + i];
        nfar = ur[i + 1] - ur[i];
      }
      const int slot = q % kRing;
      mbar_wait(&bars[slot], (q / kRing) & 1);
      if (tr && lane == 0) tr[3 * q + 0] = clock64();
      const double* T = ring + slot * kTileElems;
      double nb = 0.0;
      if (tt > 0) nb += neighbour(T, kTile, j, xn1);
      if (tt > 1) nb += neighbour(T, 2 * kTile, j, xn2);
      double td[kTile];
#pragma unroll
      for (int k = 0; k < kTile; ++k) td[k] = T[k * kTile + j];
      double far = 0.0;
      if (valid && nfar > 0) {
        double* ps = part + (t % kPartRing) * kTile + j;
        far = wait_ready(ps);
        *ps = pend;
      }
      if (tr && lane == 0) tr[3 * q + 1] = clock64();
      double acc = zi - (nb + far);
      double xj = 0.0;
#pragma unroll
      for (int k = kTile - 1; k >= 0; --k) {
        const double xk = __shfl_sync(0xffffffffu, acc * rd, k);
        if (j == k) xj = xk;
        if (j < k) acc = fma(-td[k], xk, acc);
      }
      if (!valid) xj = 0.0;
      if (valid) {
        *reinterpret_cast<volatile double*>(x + i) = xj;
        out[r0 + i] = sub ? si - xj : xj;
      }
      xn2 = xn1;
      xn1 = xj;
      if (tr && lane == 0) tr[3 * q + 2] = clock64();
      refill(q);
      if (lane == 0) *reinterpret_cast<volatile int*>(&done_u) = tt + 1;
    }
  } else {
    // workers: far sums of U rows, descending
    const int w = warp - 1;
    const double* fv = a.uval + a.uoff[b];
    const uint16_t* fc = a.ucol + a.uoff[b];
    int sn = 0, en = 0;
    if (w < n) {
      sn = ur[n - 1 - w];
      en = ur[n - w];
    }
    for (int r = w; r < n; r += kWorkers) {
      const int i = n - 1 - r;
      const int s = sn, e = en;
      if (r + kWorkers < n) {
        sn = ur[i - kWorkers];
        en = ur[i - kWorkers + 1];
      }
      if (e == s) continue;
      const int t = i / kTile;
      const int pos = nt - 1 - t;
      const double acc = far_dot(fv, fc, s, e, x, lane, a.sleep_ns);
      if (lane == 0) {
        while (*reinterpret_cast<volatile int*>(&done_u) < pos - (kPartRing - 1)) __nanosleep(128);
        *reinterpret_cast<volatile double*>(part + (t % kPartRing) * kTile + (i % kTile)) = acc;
      }
    }
  }
}

}  // namespace

size_t trisolve_smem_bytes(int dim_max) {
  return sizeof(double) * (static_cast<size_t>(kRing) * kTileElems + kPartRing * kTile +
                           2 * static_cast<size_t>(dim_max));
}

void block_trisolve(const FactorSet& fs, const double* rhs, double* out, const double* sub,
                    cudaStream_t s, long long* trace) {
  if (fs.nblocks == 0) return;
  TriArgs a;
  a.row0 = fs.row0.as<int>();
  a.dim = fs.dim.as<int>();
  a.loff = fs.loff.as<long long>();
  a.uoff = fs.uoff.as<long long>();
  a.toff = fs.toff.as<long long>();
  a.lrp = fs.lrp.as<int>();
  a.urp = fs.urp.as<int>();
  a.lval = fs.lval.as<double>();
  a.lcol = fs.lcol.as<uint16_t>();
  a.uval = fs.uval.as<double>();
  a.ucol = fs.ucol.as<uint16_t>();
  a.ltile = fs.ltile.as<double>();
  a.utile = fs.utile.as<double>();
  a.urdiag = fs.urdiag.as<double>();
  a.perm = fs.has_perm ? fs.perm.as<int>() : nullptr;
  a.dim_max = fs.max_dim;
  a.trace = trace;
  static const unsigned sleep_ns = [] {
    const char* e = getenv("MSCG_TRI_SLEEP_NS");
    return e ? static_cast<unsigned>(atoi(e)) : 64u;
  }();
  a.sleep_ns = sleep_ns;
  const size_t smem = trisolve_smem_bytes(fs.max_dim);
  if (smem > 227 * 1024)
    throw Error(1, "block_trisolve: block of " + std::to_string(fs.max_dim) +
                       " rows exceeds the shared-memory solution vectors");
  if (smem > 48 * 1024)
    MSCG_CUDA(cudaFuncSetAttribute(trisolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  trisolve_kernel<<<fs.nblocks, kThreads, smem, s>>>(a, rhs, out, sub);
  MSCG_CUDA(cudaGetLastError());
}

}  // namespace mscg
