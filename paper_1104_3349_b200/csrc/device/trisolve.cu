// Block-diagonal triangular solve x_b = U_b^-1 L_b^-1 P_b r_b for every block
// of a FactorSet in one launch (reference `solve`, factorization.cpp:129-158,
// driven per block by block_solve, preconditioner.cpp:13-22).
//
// Why tiles (measured, SURVEY §8(a) A6 structure): an interior block of
// ~3000 rows is [velocities | pressures]; its L has a banded velocity part
// (~21 nnz/row, bandwidth <= 63), a wide velocity->pressure coupling
// (~450 nnz/row) and a ~45%-dense pressure triangle; U mirrors it.  The
// dependency chain is therefore ~one row deep per row in both triangles,
// while most bytes sit far from the diagonal.  One CTA (16 warps) per block:
//
//  * solver (warp 0) walks the 32-row tiles in order.  The near window of a
//    tile (diagonal tile + the two neighbour tiles, dense 32 x 96 fp64,
//    column-major) arrives in shared memory by TMA bulk copy
//    (cp.async.bulk + mbarrier ring); lane j owns row j, neighbour tiles are
//    applied from registers through shuffles, and the 32-step diagonal chain
//    costs one shuffle + one FMA per row.  Per-row scalars of the next tile
//    are prefetched one tile ahead, and the solver issues no memory fence,
//    so no outstanding global load ever sits on the chain;
//  * workers (warps 1-15) stream the far entries (L: columns < 32(t-2), U:
//    columns >= 32(t+3)) from HBM.  Each row's far entries are cut into work
//    items of kSeg = 512 entries (one 16-deep unrolled round of coalesced
//    value/column loads per lane), listed per block at setup in the order
//    the chain consumes them; a worker publishes one partial sum per item
//    into a shared-memory ring that the solver sums in a fixed order
//    (deterministic results);
//  * z (L output) and x (U output) live in shared memory.  Readiness is the
//    value itself: slots start as a signalling-NaN pattern no arithmetic
//    produces and an aligned 8-byte shared store is single-copy atomic, so
//    consumers poll the slot (backing off with __nanosleep) and need neither
//    flags nor fences.
// Rounding differs from the reference's sequential row sums by ~1e-16
// relative, far inside the 1e-10 apply bar.
#include <cstdlib>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

// Kernel variants: (warps per CTA, load unroll per lane, read-only path).
constexpr int kRing = 2;               // near-tile TMA ring depth
constexpr int kPartRing = 8;           // far-sum ring depth (tiles)
constexpr int kPartTile = kTile * kMaxSeg;
constexpr unsigned kTileBytes = kTileElems * sizeof(double);

struct TriArgs {
  const int* row0;
  const int* dim;
  const long long* loff;
  const long long* uoff;
  const long long* toff;
  const long long* lioff;
  const long long* uioff;
  const int* lrp;
  const int* urp;
  const double* lval;
  const uint16_t* lcol;
  const double* uval;
  const uint16_t* ucol;
  const double* ltile;
  const double* utile;
  const double* urdiag;
  const int4* litems;  // {row, segment, begin, end}
  const int4* uitems;
  const int* perm;  // nullable
  int dim_max;
  long long* trace;  // debug: clock64 stamps for block 0, or null
  unsigned sleep_ns; // worker back-off while polling
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

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

// Fire-and-forget TMA prefetch of [p, p + bytes) into L2 (16-byte granules;
// allocations are 256-byte aligned, so the rounded range stays inside).
__device__ __forceinline__ void l2_prefetch(const void* p, long long bytes) {
  if (bytes <= 0) return;
  const unsigned long long lo = reinterpret_cast<unsigned long long>(p) & ~15ull;
  const unsigned long long hi = (reinterpret_cast<unsigned long long>(p) + bytes + 15) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo),
               "r"(static_cast<unsigned>(hi - lo))
               : "memory");
}

constexpr int kPrefetchTiles = 4;  // far data / near tiles prefetched ahead

// Partial dot product of entries [s, e) of a far row with the (partially
// computed) solution vector; all loads of the item are issued before the
// first wait.
template <int kUnroll, bool kNc>
__device__ __forceinline__ double seg_dot(const double* __restrict__ vals,
                                          const uint16_t* __restrict__ cols, int s, int e,
                                          const double* sol, int lane, unsigned ns) {
  double acc = 0.0, acc2 = 0.0;
  for (int k0 = s + lane; k0 < e; k0 += 32 * kUnroll) {
    double v[kUnroll];
    int c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int k = k0 + 32 * u;
      if (k < e) {
        v[u] = kNc ? __ldg(vals + k) : __ldcg(vals + k);
        c[u] = kNc ? __ldg(cols + k) : __ldcg(cols + k);
      } else {
        v[u] = 0.0;
        c[u] = -1;
      }
    }
    // Gather all operands first (independent shared loads, pipelined), and
    // only fall back to polling when one of them is still pending.
    const volatile double* vs = sol;
    double xv[kUnroll];
    bool pending = false;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      xv[u] = c[u] >= 0 ? vs[c[u]] : 0.0;
      pending |= is_pending(xv[u]);
    }
    if (pending) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (c[u] >= 0) xv[u] = wait_ready_lazy(sol + c[u], ns);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; u += 2) {
      acc = fma(v[u], xv[u], acc);
      acc2 = fma(v[u + 1], xv[u + 1], acc2);
    }
  }
  return warp_sum(acc + acc2);
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

// Solver: lane 0 waits until `expected` far items of the tile were published
// (one shared-memory poll per warp instead of one per lane and slot), then
// resets the counter for the ring tile's next use.  Slot values still carry
// their own readiness (take_far), so no fence orders slot vs counter.
__device__ __forceinline__ void wait_items(int* counter, int expected, int lane) {
  if (lane == 0 && expected > 0) {
    int spins = 0;
    while (vload(counter) < expected)
      if (++spins > 8) __nanosleep(20);
    *reinterpret_cast<volatile int*>(counter) = 0;
  }
  __syncwarp();
}

// Sum of the published far partial sums of one row, in item order, resetting
// the slots.
__device__ __forceinline__ double take_far(double* slots, int nseg, double pend) {
  double f = 0.0;
  for (int k = 0; k < nseg; ++k) {
    f += wait_ready(slots + k);
    slots[k] = pend;
  }
  return f;
}

template <int kWarps, int kUnroll, bool kNc, int kMinBlocks = 1>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks) trisolve_kernel(TriArgs a,
                                                            const double* __restrict__ rhs,
                                                            double* __restrict__ out,
                                                            const double* __restrict__ sub) {
  constexpr int kWorkers = kWarps - 1;
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                          // kRing near tiles
  double* part = ring + kRing * kTileElems;   // [kPartRing][32 rows][kMaxSeg]
  double* z = part + kPartRing * kPartTile;   // dim_max (L output)
  double* x = z + a.dim_max;                  // dim_max (U output)
  __shared__ __align__(8) uint64_t bars[kRing];
  __shared__ int done_l, done_u;
  __shared__ int cnt[kPartRing];  // far items published per ring tile

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
  for (int i = threadIdx.x; i < kPartRing * kPartTile; i += blockDim.x) part[i] = pend;
  if (threadIdx.x == 0) {
    done_l = 0;
    for (int r = 0; r < kPartRing; ++r) cnt[r] = 0;
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
    int pf_lo = 0, pf_hi = 0;  // far range of the next prefetch target tile (lane 0)
    if (lane == 0) {
      // far data of the first kPrefetchTiles tiles, and the item lists
      const int e0 = lr[min(kPrefetchTiles * kTile, n)];
      l2_prefetch(a.lval + a.loff[b], 8LL * e0);
      l2_prefetch(a.lcol + a.loff[b], 2LL * e0);
      l2_prefetch(a.litems + a.lioff[b], 16LL * (a.lioff[b + 1] - a.lioff[b]));
      l2_prefetch(a.uitems + a.uioff[b], 16LL * (a.uioff[b + 1] - a.uioff[b]));
      if (kPrefetchTiles < nt) {
        pf_lo = lr[kPrefetchTiles * kTile];
        pf_hi = lr[min((kPrefetchTiles + 1) * kTile, n)];
      }
    }
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
      // diagonal-tile column k of row j (registers when the budget allows)
      double td[kMinBlocks == 1 ? kTile : 1];
      if constexpr (kMinBlocks == 1) {
#pragma unroll
        for (int k = 0; k < kTile; ++k) td[k] = T[(2 * kTile + k) * kTile + j];
      }
      auto dcol = [&](int k) {
        if constexpr (kMinBlocks == 1) return td[k];
        else return T[(2 * kTile + k) * kTile + j];
      };
      double far = 0.0;
      {
        const int nseg = (valid && nfar > 0) ? far_segments(nfar) : 0;
        wait_items(&cnt[t % kPartRing], __reduce_add_sync(0xffffffffu, nseg), lane);
        if (nseg) far = take_far(part + (t % kPartRing) * kPartTile + j * kMaxSeg, nseg, pend);
      }
      if (tr && lane == 0) tr[3 * t + 1] = clock64();
      // acc = b_i - (known sums); z_k = acc_k once step k is reached
      double acc = bi - (nb + far);
      double zj = 0.0;
#pragma unroll
      for (int k = 0; k < kTile; ++k) {
        const double zk = __shfl_sync(0xffffffffu, acc, k);
        if (j == k) zj = zk;
        if (j > k) acc = fma(-dcol(k), zk, acc);
      }
      if (!valid) zj = 0.0;
      if (valid) *reinterpret_cast<volatile double*>(z + i) = zj;
      zp2 = zp1;
      zp1 = zj;
      if (lane == 0) {
        *reinterpret_cast<volatile int*>(&done_l) = t + 1;  // part-ring slot reuse only
        if (tr) tr[3 * t + 2] = clock64();
        // L2 prefetch ahead of the chain: far data of tile t + kPrefetchTiles
        // (row pointers loaded one tile earlier) and the near tile stream.
        const int u = t + kPrefetchTiles;
        if (u < nt) {
          l2_prefetch(a.lval + a.loff[b] + pf_lo, 8LL * (pf_hi - pf_lo));
          l2_prefetch(a.lcol + a.loff[b] + pf_lo, 2LL * (pf_hi - pf_lo));
          if (u + 1 < nt) {
            pf_lo = lr[(u + 1) * kTile];
            pf_hi = lr[min((u + 2) * kTile, n)];
          }
        }
        if (t + kRing + 1 < 2 * nt) l2_prefetch(item_src(t + kRing + 1), kTileBytes);
      }
      refill(t);
    }
  } else {
    // workers: far items of L rows, rows ascending
    const int w = warp - 1;
    const double* fv = a.lval + a.loff[b];
    const uint16_t* fc = a.lcol + a.loff[b];
    const int4* items = a.litems + a.lioff[b];
    const int nitems = static_cast<int>(a.lioff[b + 1] - a.lioff[b]);
    int4 nxt = w < nitems ? items[w] : make_int4(0, 0, 0, 0);
    for (int it = w; it < nitems; it += kWorkers) {
      const int4 d = nxt;
      if (it + kWorkers < nitems) nxt = items[it + kWorkers];
      const int i = d.x, k = d.y & 0xff, ss = d.z, ee = d.w;
      const int item = (i << 3) | k;
      const int t = i / kTile;
      long long* rt = (tr && lane == 0) ? tr + 6LL * nt + 4LL * it : nullptr;
      if (rt) rt[0] = clock64();
      // sleep until the tiles this item reads are published (one poll per
      // warp); per-value sentinels still guard the reads themselves
      if (lane == 0)
        while (vload(&done_l) < (d.y >> 8)) __nanosleep(a.sleep_ns);
      __syncwarp();
      const double acc = seg_dot<kUnroll, kNc>(fv, fc, ss, ee, z, lane, a.sleep_ns);
      if (rt) rt[1] = clock64();
      if (lane == 0) {
        // ring slot of tile t is free once tile t - kPartRing was consumed
        while (vload(&done_l) < t - (kPartRing - 1)) __nanosleep(a.sleep_ns);
        *reinterpret_cast<volatile double*>(part + (t % kPartRing) * kPartTile +
                                            (i % kTile) * kMaxSeg + k) = acc;
        atomicAdd(&cnt[t % kPartRing], 1);
        if (rt) {
          rt[2] = clock64();
          rt[3] = item;
        }
      }
    }
  }
  __syncthreads();  // every L far sum consumed before U sums reuse the ring

  // ================================================================ U pass
  if (warp == 0) {
    double xn1 = 0.0, xn2 = 0.0;  // x of tiles t+1, t+2
    int pf_lo = 0, pf_hi = 0;
    if (lane == 0) {
      const int t0 = nt - 1 - kPrefetchTiles;  // tiles above t0 prefetched now
      const int s0 = ur[max(t0 + 1, 0) * kTile];
      l2_prefetch(a.uval + a.uoff[b] + s0, 8LL * (ur[n] - s0));
      l2_prefetch(a.ucol + a.uoff[b] + s0, 2LL * (ur[n] - s0));
      if (t0 >= 0) {
        pf_lo = ur[t0 * kTile];
        pf_hi = ur[min((t0 + 1) * kTile, n)];
      }
    }
    double rdn = 0.0, sin_ = 0.0;
    int fn = 0;
    {
      const int i = (nt - 1) * kTile + j;
      if (i < n) {
        rdn = a.urdiag[r0 + i];
        if (sub) sin_ = sub[r0 + i];
        fn = ur[i + 1] - ur[i];
      }
    }
    for (int tt = 0; tt < nt; ++tt) {
      const int t = nt - 1 - tt;
      const int q = nt + tt;
      const int i = t * kTile + j;
      const bool valid = i < n;
      const double zi = valid ? z[i] : 0.0;
      const double rd = rdn, si = sin_;
      const int nfar = fn;
      const int ip = i - kTile;  // prefetch next (lower) tile's scalars
      if (ip >= 0) {
        rdn = a.urdiag[r0 + ip];
        if (sub) sin_ = sub[r0 + ip];
        fn = ur[ip + 1] - ur[ip];
      }
      const int slot = q % kRing;
      mbar_wait(&bars[slot], (q / kRing) & 1);
      if (tr && lane == 0) tr[3 * q + 0] = clock64();
      const double* T = ring + slot * kTileElems;
      double nb = 0.0;
      if (tt > 0) nb += neighbour(T, kTile, j, xn1);
      if (tt > 1) nb += neighbour(T, 2 * kTile, j, xn2);
      double td[kMinBlocks == 1 ? kTile : 1];
      if constexpr (kMinBlocks == 1) {
#pragma unroll
        for (int k = 0; k < kTile; ++k) td[k] = T[k * kTile + j];
      }
      auto dcol = [&](int k) {
        if constexpr (kMinBlocks == 1) return td[k];
        else return T[k * kTile + j];
      };
      double far = 0.0;
      {
        const int nseg = (valid && nfar > 0) ? far_segments(nfar) : 0;
        wait_items(&cnt[t % kPartRing], __reduce_add_sync(0xffffffffu, nseg), lane);
        if (nseg) far = take_far(part + (t % kPartRing) * kPartTile + j * kMaxSeg, nseg, pend);
      }
      if (tr && lane == 0) tr[3 * q + 1] = clock64();
      double acc = zi - (nb + far);
      double xj = 0.0;
#pragma unroll
      for (int k = kTile - 1; k >= 0; --k) {
        const double xk = __shfl_sync(0xffffffffu, acc * rd, k);
        if (j == k) xj = xk;
        if (j < k) acc = fma(-dcol(k), xk, acc);
      }
      if (!valid) xj = 0.0;
      if (valid) {
        *reinterpret_cast<volatile double*>(x + i) = xj;
        out[r0 + i] = sub ? si - xj : xj;
      }
      xn2 = xn1;
      xn1 = xj;
      if (lane == 0) {
        *reinterpret_cast<volatile int*>(&done_u) = tt + 1;
        if (tr) tr[3 * q + 2] = clock64();
        const int u = t - kPrefetchTiles;  // far data of the tile kPrefetchTiles below
        if (u >= 0) {
          l2_prefetch(a.uval + a.uoff[b] + pf_lo, 8LL * (pf_hi - pf_lo));
          l2_prefetch(a.ucol + a.uoff[b] + pf_lo, 2LL * (pf_hi - pf_lo));
          if (u - 1 >= 0) {
            pf_lo = ur[(u - 1) * kTile];
            pf_hi = ur[min(u * kTile, n)];
          }
        }
        if (q + kRing + 1 < 2 * nt) l2_prefetch(item_src(q + kRing + 1), kTileBytes);
      }
      refill(q);
    }
  } else {
    // workers: far items of U rows, rows descending
    const int w = warp - 1;
    const double* fv = a.uval + a.uoff[b];
    const uint16_t* fc = a.ucol + a.uoff[b];
    const int4* items = a.uitems + a.uioff[b];
    const int nitems = static_cast<int>(a.uioff[b + 1] - a.uioff[b]);
    const long long lit = a.lioff[b + 1] - a.lioff[b];
    int4 nxt = w < nitems ? items[w] : make_int4(0, 0, 0, 0);
    for (int it = w; it < nitems; it += kWorkers) {
      const int4 d = nxt;
      if (it + kWorkers < nitems) nxt = items[it + kWorkers];
      const int i = d.x, k = d.y & 0xff, ss = d.z, ee = d.w;
      const int item = (i << 3) | k;
      const int t = i / kTile;
      const int pos = nt - 1 - t;
      long long* rt = (tr && lane == 0) ? tr + 6LL * nt + 4LL * (lit + it) : nullptr;
      if (rt) rt[0] = clock64();
      if (lane == 0)
        while (vload(&done_u) < (d.y >> 8)) __nanosleep(a.sleep_ns);
      __syncwarp();
      const double acc = seg_dot<kUnroll, kNc>(fv, fc, ss, ee, x, lane, a.sleep_ns);
      if (rt) rt[1] = clock64();
      if (lane == 0) {
        while (vload(&done_u) < pos - (kPartRing - 1)) __nanosleep(a.sleep_ns);
        *reinterpret_cast<volatile double*>(part + (t % kPartRing) * kPartTile +
                                            (i % kTile) * kMaxSeg + k) = acc;
        atomicAdd(&cnt[t % kPartRing], 1);
        if (rt) {
          rt[2] = clock64();
          rt[3] = item;
        }
      }
    }
  }
}

}  // namespace

size_t trisolve_smem_bytes(int dim_max) {
  return sizeof(double) * (static_cast<size_t>(kRing) * kTileElems +
                           static_cast<size_t>(kPartRing) * kPartTile +
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
  a.lioff = fs.lioff.as<long long>();
  a.uioff = fs.uioff.as<long long>();
  a.lrp = fs.lrp.as<int>();
  a.urp = fs.urp.as<int>();
  a.lval = fs.lval.as<double>();
  a.lcol = fs.lcol.as<uint16_t>();
  a.uval = fs.uval.as<double>();
  a.ucol = fs.ucol.as<uint16_t>();
  a.ltile = fs.ltile.as<double>();
  a.utile = fs.utile.as<double>();
  a.urdiag = fs.urdiag.as<double>();
  a.litems = fs.litems.as<int4>();
  a.uitems = fs.uitems.as<int4>();
  a.perm = fs.has_perm ? fs.perm.as<int>() : nullptr;
  a.dim_max = fs.max_dim;
  a.trace = trace;
  static const unsigned sleep_ns = [] {
    const char* e = getenv("MSCG_TRI_SLEEP_NS");
    return e ? static_cast<unsigned>(atoi(e)) : 32u;
  }();
  a.sleep_ns = sleep_ns;
  const size_t smem = trisolve_smem_bytes(fs.max_dim);
  if (smem > 227 * 1024)
    throw Error(1, "block_trisolve: block of " + std::to_string(fs.max_dim) +
                       " rows exceeds the shared-memory solution vectors");
  static const int variant = [] {
    const char* e = getenv("MSCG_TRI_VARIANT");
    return e ? atoi(e) : 0;
  }();
  auto launch = [&](auto kern, int warps) {
    if (smem > 48 * 1024)
      MSCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    kern<<<fs.nblocks, warps * 32, smem, s>>>(a, rhs, out, sub);
  };
  switch (variant) {
    case 1: launch(trisolve_kernel<16, 8, true>, 16); break;
    case 2: launch(trisolve_kernel<16, 16, false>, 16); break;
    case 3: launch(trisolve_kernel<8, 16, true>, 8); break;
    case 4: launch(trisolve_kernel<8, 8, true>, 8); break;
    case 5: launch(trisolve_kernel<8, 16, false>, 8); break;
    case 6: launch(trisolve_kernel<16, 8, true, 2>, 16); break;
    case 7: launch(trisolve_kernel<16, 4, true, 2>, 16); break;
    case 8: launch(trisolve_kernel<12, 8, true, 2>, 12); break;
    case 9: launch(trisolve_kernel<16, 16, true>, 16); break;
    // default: 2 CTAs per SM (64 registers) — measured fastest at cfg4
    default: launch(trisolve_kernel<16, 4, true, 2>, 16); break;
  }
  MSCG_CUDA(cudaGetLastError());
}

}  // namespace mscg
