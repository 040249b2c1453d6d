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
//  * solver (warp 0) walks the 32-row tiles in order.  Everything a tile
//    needs — the near window (the two neighbour tiles dense, 32 x 64 fp64
//    column-major, and the strictly triangular part of the diagonal tile
//    packed by column), the per-row metadata (1/U_jj, number of far work
//    items) and, in the L pass, the tile's slice of the right-hand side —
//    arrives in shared memory by TMA bulk copies (cp.async.bulk + mbarrier,
//    double-buffered).  The solver issues no global loads: a load queued
//    behind the workers' streaming requests stalled the chain for ~30K
//    cycles per tile.  Lane j owns row j; the neighbour tiles are applied
//    with broadcast shared loads of their solution, then the 32-step
//    diagonal chain costs one shuffle + one FMA per row;
//  * workers (warps 1-15) stream the far entries (L: columns < 32(t-2), U:
//    columns >= 32(t+3)) from HBM.  Each row's far entries are cut into work
//    items of kSeg = 512 entries, listed per block at setup in the order the
//    chain consumes them together with the number of tiles that must be
//    published first; a worker issues an item's loads, sleeps until its
//    inputs are final, and publishes one partial sum per item into a
//    shared-memory ring that the solver sums in a fixed order (deterministic);
//  * the solution lives in shared memory, x overwriting z slot by slot (the
//    U pass reads z of a tile just before writing its x; workers read x only
//    of tiles already solved).  In the L pass readiness is the value itself:
//    slots start as a signalling-NaN pattern no arithmetic produces and an
//    aligned 8-byte shared store is single-copy atomic; the U pass counter
//    is published with release/acquire.  Every wait is warp-uniform (all
//    lanes poll the same word): a divergent spin sends the next shuffles to
//    their slow collective path.  The result leaves in one coalesced
//    epilogue.
// When the blocks are too few to fill the GPU (cfg2: 16, cfg3: 64), a
// thread-block cluster of 2-8 CTAs solves each block (kCluster): the home CTA
// is the kernel above; in the others warp 0 pulls every solved tile into the
// CTA's own copy of the solution over distributed shared memory and the
// remaining warps are workers that publish their partial sums straight into
// the home CTA's slots (see trisolve_kernel and block_trisolve).
// Rounding differs from the reference's sequential row sums by ~1e-16
// relative, far inside the 1e-10 apply bar.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kVecElems = 40;          // rhs slice: 32 + alignment slack
constexpr int kSlotElems = kTileElems + kVecElems;

struct TriArgs {
  const int* row0;
  const int* dim;
  const long long* loff;
  const long long* uoff;
  const long long* toff;
  const long long* lioff;
  const long long* uioff;
  const double* lval;
  const uint16_t* lcol;
  const double* uval;
  const uint16_t* ucol;
  const double* ltile;
  const double* utile;
  const int* lwidth;   // per tile: ELL width of the neighbour window or kDenseNbr
  const int* uwidth;
  const int4* litems;  // {row, segment | need << 8, begin, end}
  const int4* uitems;
  const int* lnum;     // items per block
  const int* unum;
  const int* lrp;      // far-entry row offsets, row0[b] + b + i
  const int* urp;
  const int* lslot;    // first far-sum slot of each row, row0[b] + i
  const int* uslot;
  int max_slots;       // far-sum slots per block (shared memory)
  const int* perm;  // nullable (Schur blocks)
  const int* order; // launch order of the blocks
  int pos0;          // first launch-order position of this launch
  int dim_max;
  long long* trace;  // debug: clock64 stamps for block 0, or null
  unsigned sleep_ns; // worker back-off while polling: first sleep
  unsigned sleep_max;  // and cap of the doubling
  int pf_items;      // far-data L2 prefetch distance in rounds of items, L pass (0 = off)
  int pf_u;          // same, U pass
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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
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
// Fire-and-forget TMA prefetch of [p, p + bytes) into L2.
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// L2 prefetch of far entries [s, e) (values + columns), widened to 16 B
// (32-bit arithmetic on entry offsets: this runs once per work item in loops
// that are issue-bound).
__device__ __forceinline__ void prefetch_far(const double* v, const uint16_t* c, int s, int e) {
  if (e <= s) return;
  const int mv = static_cast<int>(reinterpret_cast<unsigned long long>(v) >> 3) & 1;
  const int mc = static_cast<int>(reinterpret_cast<unsigned long long>(c) >> 1) & 7;
  const int sv = s - ((s + mv) & 1), ev = e + ((e + mv) & 1);
  const int sc = s - ((s + mc) & 7), ec = e + ((-(e + mc)) & 7);
  l2_prefetch(v + sv, 8u * static_cast<unsigned>(ev - sv));
  l2_prefetch(c + sc, 2u * static_cast<unsigned>(ec - sc));
}

// Entry c of the solution vector at shared-window address `base` (32-bit
// shared addressing: one address instruction per gather in the dot loops).
__device__ __forceinline__ double sol_at(uint32_t base, int c) {
  double x;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(x) : "r"(base + 8u * static_cast<uint32_t>(c)) : "memory");
  return x;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
// Pass counter read: acquire when the solution is overwritten in place (the
// U pass reuses z's slots, so a value's presence cannot mark readiness).
// Cluster solves read the home CTA's counter through a generic (distributed
// shared memory) address with cluster-scope acquire.
__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cluster(int* p, int v) {
  asm volatile("st.release.cluster.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <bool kAcquire, bool kRemote = false>
__device__ __forceinline__ int poll(const int* p) {
  return kAcquire ? (kRemote ? ld_acquire_cluster(p) : ld_acquire(p)) : vload(p);
}
// How a worker learns that `need` tiles of the pass are solved:
//   kWaitValue   relaxed counter as a hint, the solution slots' sentinels as
//                the guarantee (cluster solves: x kept apart from z, values
//                pulled over DSMEM);
//   kWaitAcquire the counter read with acquire (x overwrites z in place: a
//                value's presence cannot mark readiness);
//   kWaitTile    one mbarrier per tile and pass: the solver's arrive releases
//                the tile's stores, try_wait acquires them and suspends the
//                warp in hardware; no sentinel tests in the dot loops (the
//                streaming phases are issue-bound).
constexpr int kWaitValue = 0, kWaitAcquire = 1, kWaitTile = 2;
template <int kWait, bool kRemote>
__device__ __forceinline__ void wait_tiles(const int* done, int need, unsigned ns,
                                           unsigned ns_max, unsigned parity) {
  if constexpr (kWait == kWaitTile) {
    if (need > 0)
      mbar_wait(reinterpret_cast<uint64_t*>(const_cast<int*>(done)) + (need - 1), parity);
  } else {
    // every lane polls the same word: the loop exit is warp-uniform, so the
    // warp stays converged (divergent spins cost the shuffles afterwards
    // their fast path).  Exponential back-off: the solver finishes a tile
    // every few microseconds and short polls would steal its issue slots.
    for (unsigned sl = ns; poll<kWait == kWaitAcquire, kRemote>(done) < need;
         sl = min(2 * sl, ns_max))
      __nanosleep(sl);
  }
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// generic address of `p` (a shared-memory location of this CTA) in CTA
// `rank` of the cluster
template <class T>
__device__ __forceinline__ T* map_rank(T* p, unsigned rank) {
  T* out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
  return out;
}

// A vector slice [p, p + 32) copied by TMA needs 16-byte aligned ends:
// copy the enclosing aligned range and remember the offset (0 or 1).
struct Slice {
  const double* src;
  unsigned bytes;
  int off;
};
__device__ __forceinline__ Slice aligned_slice(const double* p, int len) {
  const unsigned long long a = reinterpret_cast<unsigned long long>(p);
  const unsigned long long lo = a & ~15ull;
  const unsigned long long hi = (a + 8ull * len + 15) & ~15ull;
  return {reinterpret_cast<const double*>(lo), static_cast<unsigned>(hi - lo),
          static_cast<int>((a - lo) >> 3)};
}

// Partial dot product of far entries [s, e) with the (partially computed)
// solution vector.  The trip count is warp-uniform (per-lane predicates
// instead of per-lane loop bounds) so the final reduction runs converged.
// The first round's loads are issued before the readiness wait (one poll
// per warp on the tile counter).
template <int kUnroll, int kWait, bool kRemote = false>
__device__ __forceinline__ double seg_dot(const double* __restrict__ vals,
                                          const uint16_t* __restrict__ cols, int s, int e,
                                          const double* sol, int lane, unsigned ns,
                                          const int* done, int need, unsigned ns_max,
                                          unsigned parity) {
  constexpr bool kInPlace = kWait != kWaitValue;  // no sentinel tests
  double acc = 0.0, acc2 = 0.0;
  const uint32_t vs = smem_addr(sol);
  bool waited = false;
  auto wait = [&]() {
    wait_tiles<kWait, kRemote>(done, need, ns, ns_max, parity);
    waited = true;
  };
  // Gather operands (independent shared loads); poll only if one is still
  // pending (the counter is a hint, the sentinel is the guarantee).
  auto settle = [&](double (&xv)[kUnroll], const int (&c)[kUnroll]) {
    if (kInPlace) return;
    bool pending = false;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) pending |= is_pending(xv[u]);
    while (__any_sync(0xffffffffu, pending)) {
      __nanosleep(ns);
      pending = false;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (c[u] >= 0 && is_pending(xv[u])) xv[u] = sol_at(vs, c[u]);
        pending |= is_pending(xv[u]);
      }
    }
  };
  int base = s;
  // Full rounds: no bounds predicates.  The streaming phases of the solve are
  // issue-bound (16 warps per scheduler pair), and a predicated load costs
  // its own descriptor moves on top of the compare.
  const double* pv = vals + s + lane;
  const uint16_t* pc = cols + s + lane;
  for (; base + 32 * kUnroll <= e; base += 32 * kUnroll) {
    double v[kUnroll];
    int c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      v[u] = __ldg(pv + 32 * u);
      c[u] = __ldg(pc + 32 * u);
    }
    pv += 32 * kUnroll;
    pc += 32 * kUnroll;
    if (!waited) wait();
    double xv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) xv[u] = sol_at(vs, c[u]);
    settle(xv, c);
#pragma unroll
    for (int u = 0; u < kUnroll; u += 2) {
      acc = fma(v[u], xv[u], acc);
      acc2 = fma(v[u + 1], xv[u + 1], acc2);
    }
  }
  if (base < e) {  // the last, partial round
    double v[kUnroll];
    int c[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int k = base + lane + 32 * u;
      if (k < e) {
        v[u] = __ldg(vals + k);
        c[u] = __ldg(cols + k);
      } else {
        v[u] = 0.0;
        c[u] = -1;
      }
    }
    if (!waited) wait();
    double xv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) xv[u] = c[u] >= 0 ? sol_at(vs, c[u]) : 0.0;
    settle(xv, c);
#pragma unroll
    for (int u = 0; u < kUnroll; u += 2) {
      acc = fma(v[u], xv[u], acc);
      acc2 = fma(v[u + 1], xv[u + 1], acc2);
    }
  }
  return warp_sum(acc + acc2);
}

// A multi-row item: rows [row0, row0 + span) of one tile, entries [s, e)
// (at most 32 * kUnroll).  One round of loads for all rows; each product goes
// to the warp's shared scratch.  Row r is summed by the P = 32 / span (rounded
// down to a power of two) lanes r * P .. r * P + P - 1: lane `sub` of the row
// adds every P-th product of the row's run and the P partial sums meet in a
// fixed butterfly (deterministic).  The first lane of each row returns the row
// sum, with the row's far-sum slot in `my` (has = the row has entries).
template <int kUnroll, int kWait, bool kRemote = false>
__device__ __forceinline__ double group_dot(const double* __restrict__ vals,
                                             const uint16_t* __restrict__ cols, int s, int e,
                                             const int* rp, const int* slots, int row0, int span,
                                             const double* sol, double* scratch, int lane,
                                             unsigned ns, const int* done, int need,
                                             unsigned ns_max, unsigned parity, int& my,
                                             bool& has) {
  constexpr bool kInPlace = kWait != kWaitValue;
  double v[kUnroll];
  int c[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int k = s + lane + 32 * u;
    v[u] = k < e ? __ldg(vals + k) : 0.0;
    c[u] = k < e ? __ldg(cols + k) : -1;
  }
  const int lg = 31 - __clz(32 / span);  // log2 of the lanes per row
  const int r = lane >> lg, sub = lane & ((1 << lg) - 1);
  const bool mine = r < span;
  const int rb = mine ? __ldg(rp + row0 + r) : 0;
  const int re = mine ? __ldg(rp + row0 + r + 1) : 0;
  my = mine && sub == 0 ? __ldg(slots + row0 + r) : 0;
  wait_tiles<kWait, kRemote>(done, need, ns, ns_max, parity);
  const uint32_t vs = smem_addr(sol);
  double xv[kUnroll];
  bool pending = false;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    xv[u] = c[u] >= 0 ? sol_at(vs, c[u]) : 0.0;
    pending |= is_pending(xv[u]);
  }
  while (!kInPlace && __any_sync(0xffffffffu, pending)) {
    __nanosleep(ns);
    pending = false;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (c[u] >= 0 && is_pending(xv[u])) xv[u] = sol_at(vs, c[u]);
      pending |= is_pending(xv[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) scratch[lane + 32 * u] = v[u] * xv[u];
  __syncwarp();
  double acc = 0.0;
  for (int k = rb + sub; k < re; k += 1 << lg) acc += scratch[k - s];
  __syncwarp();  // converged again; scratch is reused by the warp's next item
  for (int off = (1 << lg) >> 1; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  has = re > rb && sub == 0;
  return acc;
}

// sum_k T[(c0 + k) * 32 + j] * v[k] over one 32-column neighbour tile; v is
// the neighbour tile's solution in shared memory, read as broadcast 16-byte
// loads (measured: a shuffle costs 3x the issue slots of a broadcast load, and
// the chain is issue-bound).
__device__ __forceinline__ double neighbour(const double* T, int c0, int j, const double* v) {
  const double2* v2 = reinterpret_cast<const double2*>(v);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int k = 0; k < kTile; k += 4) {
    const double2 p = v2[k / 2], q = v2[k / 2 + 1];
    a0 = fma(T[(c0 + k + 0) * kTile + j], p.x, a0);
    a1 = fma(T[(c0 + k + 1) * kTile + j], p.y, a1);
    a2 = fma(T[(c0 + k + 2) * kTile + j], q.x, a2);
    a3 = fma(T[(c0 + k + 3) * kTile + j], q.y, a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// Same over the ELL neighbour window (see internal.hpp): W entries per row,
// window columns as bytes (4 per word), values as double2 pairs; win = the
// solution of the two neighbour tiles (64 slots).
__device__ __forceinline__ double ell_neighbours(const double* T, int w, int j,
                                                 const double* win) {
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(T + kNbrOff);
  const double2* vv = reinterpret_cast<const double2*>(T + kNbrOff + 4 * w);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  // unrolled so that several rounds of shared loads are in flight
#pragma unroll 4
  for (int e4 = 0; e4 < (w >> 2); ++e4) {
    const uint32_t c = cw[e4 * kTile + j];
    const double2 p = vv[(2 * e4) * kTile + j], q = vv[(2 * e4 + 1) * kTile + j];
    a0 = fma(p.x, win[c & 0xff], a0);
    a1 = fma(p.y, win[(c >> 8) & 0xff], a1);
    a2 = fma(q.x, win[(c >> 16) & 0xff], a2);
    a3 = fma(q.y, win[c >> 24], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// Row j of the diagonal tile's inverse times the tile's residuals r (shared,
// read as broadcast 16-byte loads): L: z_j = r_j + sum_{k<j} Linv_jk r_k;
// U: x_j = r_j / U_jj + sum_{k>j} Uinv_jk r_k.  Four partial sums in a fixed
// order (deterministic).
template <bool kLower>
__device__ __forceinline__ double tile_inverse_dot(const double* T, const double* r, int j) {
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double a0 = kLower ? r[j] : r[j] * T[kMetaDiag + j], a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int k = 0; k < kTile; k += 4) {
    const double2 p = r2[k / 2], q = r2[k / 2 + 1];
    const bool i0 = kLower ? k < j : k > j, i1 = kLower ? k + 1 < j : k + 1 > j;
    const bool i2 = kLower ? k + 2 < j : k + 2 > j, i3 = kLower ? k + 3 < j : k + 3 > j;
    const double c0 = i0 ? T[kTriOff + (kLower ? tri_l(j, k) : tri_u(j, k))] : 0.0;
    const double c1 = i1 ? T[kTriOff + (kLower ? tri_l(j, k + 1) : tri_u(j, k + 1))] : 0.0;
    const double c2 = i2 ? T[kTriOff + (kLower ? tri_l(j, k + 2) : tri_u(j, k + 2))] : 0.0;
    const double c3 = i3 ? T[kTriOff + (kLower ? tri_l(j, k + 3) : tri_u(j, k + 3))] : 0.0;
    a0 = fma(c0, p.x, a0);
    a1 = fma(c1, p.y, a1);
    a2 = fma(c2, q.x, a2);
    a3 = fma(c3, q.y, a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// Sum of the published far partial sums of one row, in item order, resetting
// the slots.  Warp-uniform trip count (max over the lanes' item counts).
__device__ __forceinline__ double take_far(double* slots, int nseg, double pend) {
  const int kmax = __reduce_max_sync(0xffffffffu, nseg);
  double f = 0.0;
  for (int k = 0; k < kmax; ++k) {
    const bool mine = k < nseg;
    const volatile double* vp = slots + k;
    double v = mine ? *vp : 0.0;
    while (__any_sync(0xffffffffu, mine && is_pending(v)))
      if (mine) v = *vp;
    if (mine) {
      f += v;
      slots[k] = pend;
    }
  }
  return f;
}

__device__ __forceinline__ int meta_int(const double* T, int idx) {
  return static_cast<int>(__double_as_longlong(T[idx]));
}

// kInPlace: x overwrites z slot by slot (one solution vector in shared memory
// instead of two).  kProducer:
// warp 1 issues the near-tile copies (the solver's issue of a bulk copy costs
// ~400 cycles of its chain per tile) and warps 2.. are the workers.
// kCluster > 1: a cluster of kCluster CTAs solves one block.  CTA 0 (home)
// is the single-CTA kernel (solver + workers, solution and far-sum slots in
// its shared memory).  In CTAs 1.. warp 0 pulls each solved tile from the
// home CTA into the CTA's own copy of the solution (generic addresses from
// mapa; a value is its own readiness when x is kept apart from z, which the
// cluster launches do) and warps 1.. are workers that gather locally and
// store their partial sums into the home CTA's slots.  Used when the blocks
// are too few to fill the GPU (cfg2 / cfg3): a block's far entries then
// stream through kCluster SMs instead of one.
// kTileBars (in-place single-CTA solves): readiness of both passes through
// one mbarrier per tile (kWaitTile; phase 0 = the L pass, phase 1 = the U
// pass) instead of the release/acquire counters: cfg5 D-solve 6.86 -> 6.78 ms.
// Costs 8 bytes of shared memory per tile, so the launcher falls back to the
// counters when that would cost the second CTA per SM.
// kTrace: clock stamps of block 0 (tools/trace_dsolve.py); a separate
// instantiation, so the production kernels carry no trace tests.
// kSolvers = 2: warps 0 and 1 solve alternate tiles (item q belongs to warp
// q & 1, which also owns ring slot q & 1 and refills it).  A tile's
// prologue — waiting for its copy, metadata, collecting the far sums — and
// its epilogue — the refill — need nothing from the previous tile, so they
// run while the other warp is on the chain; only the neighbour window, the
// tile-inverse dot and the publication stay on it.  The hand-off is the
// tile's own publication (mbarrier phase or release/acquire counter).
template <int kWarps, int kUnroll, int kMinBlocks, bool kInPlace, bool kProducer,
          int kCluster = 1, bool kTileBars = false, bool kTrace = false, int kSolvers = 1>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
    trisolve_kernel(TriArgs a, const double* __restrict__ rhs, double* __restrict__ out,
                    const double* __restrict__ sub) {
  static_assert(kSolvers == 1 || (kSolvers == 2 && kRing == 2 && !kProducer),
                "two solvers: items alternate between them");
  // Ring slots.  One solver: kRing (the next-but-one tile is in flight while
  // a tile is solved).  Two solvers (one CTA per SM, shared memory to spare):
  // two slots per warp — with one, a warp's refill, issued when its tile
  // ends, had a full DRAM round trip before the warp's next tile and was the
  // bound of the chain.  Copy sizes then come from the width tables (the
  // tile headers only carry the size of the item kRing ahead).
  constexpr int kDepth = kSolvers == 2 ? 4 : kRing;
  constexpr int kFirstWorker = kProducer ? 2 : kSolvers;
  constexpr int kWorkers = kWarps - kFirstWorker;
  constexpr bool kCl = kCluster > 1;
  static_assert(!kTileBars || (kInPlace && !kCl), "tile barriers: in-place single-CTA solve");
  // in-place single-CTA solves publish the L pass like the U pass
  // (release/acquire counter): no sentinel tests in the workers' dot loops,
  // which are issue-bound (cfg5 D-solve 7.05 -> 6.86 ms)
  constexpr bool kAcqL = kInPlace && !kCl && !kTileBars;
  constexpr int kWaitL = kTileBars ? kWaitTile : (kAcqL ? kWaitAcquire : kWaitValue);
  constexpr int kWaitU = !kInPlace ? kWaitValue : (kTileBars ? kWaitTile : kWaitAcquire);
  // workers of the whole cluster: the home CTA's, then warps 1.. of the
  // others (warp 0 of a remote CTA pulls the solution, see below)
  constexpr int kAllWorkers = kWorkers + (kCluster - 1) * (kWarps - 1);
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                        // kDepth slots: tile | meta | rhs slice
  double* part = ring + kDepth * kSlotElems; // far sums, one slot per work item
  double* z = part + ((a.max_slots + 1) & ~1);  // L output
  const int dpad = (a.dim_max + kTile - 1) & ~(kTile - 1);
  double* x = kInPlace ? z : z + dpad;      // U output
  double* scratch = x + dpad;               // [workers][kGroupEntries]
  // (a remote CTA of a cluster has kWarps - 1 workers)
  constexpr int kScratchSlots = kCl ? kWarps - 1 : kWorkers;
  // solver: the tile's residuals (one buffer per solver warp)
  double* rbuf = scratch + kScratchSlots * kGroupEntries +
                 (threadIdx.x >> 5 < kSolvers ? (threadIdx.x >> 5) * kTile : 0);
  // kTileBars: tbar[t] completes phase 0 with L tile t, phase 1 with the
  // t-th tile of the U pass
  uint64_t* tbar = reinterpret_cast<uint64_t*>(scratch + kScratchSlots * kGroupEntries + kSolvers * kTile);
  __shared__ __align__(8) uint64_t bars[kDepth];  // near item landed (TMA)
  __shared__ __align__(8) uint64_t empty[kRing];  // near item consumed (producer variant)
  __shared__ int done_l, done_u;

  const unsigned crank = kCl ? cluster_rank() : 0u;
  const bool home = crank == 0;
  const int b = a.order[a.pos0 + blockIdx.x / kCluster];  // heaviest blocks first (LPT)
  const int n = a.dim[b], r0 = a.row0[b];
  const int nt = (n + kTile - 1) / kTile;
  const double* lt = a.ltile + a.toff[b] * kTileStride;
  const double* ut = a.utile + a.toff[b] * kTileStride;
  const double pend = pending_value();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Cluster: every CTA keeps its own copy of the solution and pass counters
  // (warp 0 of a remote CTA pulls each solved tile from the home CTA over
  // DSMEM, so workers gather locally and the solver's chain does no extra
  // work); far sums go to the home CTA's slots.
  double* const zh = z;
  double* const xh = x;
  double* parth = kCl && !home ? map_rank(part, 0) : part;
  int* const done_lh = &done_l;
  int* const done_uh = &done_u;
  for (int i = threadIdx.x; i < nt * kTile; i += blockDim.x) {
    // rows past the block's end read as zero by the neighbour products
    z[i] = i < n ? pend : 0.0;
    if (!kInPlace) x[i] = i < n ? pend : 0.0;
  }
  for (int i = threadIdx.x; i < a.max_slots; i += blockDim.x) part[i] = pend;
  if constexpr (kTileBars)
    for (int t = threadIdx.x; t < nt; t += blockDim.x) mbar_init(&tbar[t], 1);
  if (threadIdx.x == 0) {
    done_l = 0;
    done_u = 0;
    for (int r = 0; r < kDepth; ++r) mbar_init(&bars[r], 1);
    for (int r = 0; r < kRing; ++r) mbar_init(&empty[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if constexpr (kCl) cluster_sync_all();  // the home's sentinels are in place

  // Near item q: q < nt -> L tile q (+ rhs slice), else U tile 2nt-1-q.
  // Item q lives in slot q % kDepth, phase (q / kDepth) & 1.
  const int* pm = a.perm ? a.perm + r0 : nullptr;
  // `bytes`: the item's used prefix (its predecessor kRing items earlier
  // carries it in its header; the first kRing come from the width tables).
  auto issue = [&](int q, unsigned bytes) {  // solver lane 0
    const int slot = q % kDepth;
    double* dst = ring + slot * kSlotElems;
    const bool lpass = q < nt;
    const int t = lpass ? q : 2 * nt - 1 - q;
    const double* tile = (lpass ? lt : ut) + static_cast<long long>(t) * kTileStride;
    Slice sr{nullptr, 0, 0};
    if (lpass && !pm) sr = aligned_slice(rhs + r0 + t * kTile, min(kTile, n - t * kTile));
    mbar_expect_tx(&bars[slot], bytes + sr.bytes);
    bulk_load(dst, tile, bytes, &bars[slot]);
    if (sr.bytes) bulk_load(dst + kTileElems, sr.src, sr.bytes, &bars[slot]);
  };
  auto first_bytes = [&](int q) {
    const long long tb = a.toff[b];
    const int w = q < nt ? a.lwidth[tb + q] : a.uwidth[tb + 2 * nt - 1 - q];
    return static_cast<unsigned>(8 * tile_elems(w));
  };
  // copy size of item q + kRing, from item q's header (slot still intact)
  auto next_bytes = [&](int q) {
    return static_cast<unsigned>(meta_int(ring + (q % kRing) * kSlotElems, kHdr + 1));
  };
  // Producer: issue near items [q0, q1) as their slots free up — item q
  // reuses the slot of item q - kRing, whose consumption the solver signals
  // on the slot's empty barrier (use (q - kRing) / kRing of that slot).
  auto produce = [&](int q0, int q1) {
    for (int q = q0; q < q1; ++q) {
      const int prev = q - kRing;
      mbar_wait(&empty[q % kRing], (prev / kRing) & 1);
      if (lane == 0) issue(q, next_bytes(prev));
      __syncwarp();
    }
  };
  long long* tr = (kTrace && a.trace && b == 0 && home) ? a.trace : nullptr;
  const int j = lane;

  // ================================================================ L pass
  if (home && warp < kSolvers) {
    if (warp == 0 && lane == 0) {
      for (int q = 0; q < kDepth && q < 2 * nt; ++q) issue(q, first_bytes(q));
      // the block's work-item lists go to L2 once
      l2_prefetch(reinterpret_cast<const void*>(reinterpret_cast<unsigned long long>(
                      a.litems + a.lioff[b]) & ~15ull),
                  16u * static_cast<unsigned>(a.lioff[b + 1] - a.lioff[b]) + 16);
    }
    __syncwarp();
    for (int t = warp; t < nt; t += kSolvers) {
      const int i = t * kTile + j;
      const bool valid = i < n;
      const int slot = t % kDepth;
      // Schur blocks (row_perm): gather the right-hand side directly.
      double bperm = 0.0;
      if (pm && valid) bperm = rhs[r0 + pm[i]];
      // deep ring: the refill's size, loaded now, used when the tile ends
      unsigned nbytes = 0;
      if (kDepth != kRing && t + kDepth < 2 * nt) nbytes = first_bytes(t + kDepth);
      mbar_wait(&bars[slot], (t / kDepth) & 1);
      if (tr && lane == 0) tr[4 * t + 0] = clock64();
      const double* T = ring + slot * kSlotElems;
      const int off = static_cast<int>((reinterpret_cast<unsigned long long>(rhs + r0 + t * kTile) & 15) >> 3);
      const double bi = valid ? (pm ? bperm : T[kTileElems + off + j]) : 0.0;
      const int fm = valid ? meta_int(T, kMetaSeg + j) : 0;  // items | first slot << 8
      const int wn = meta_int(T, kHdr);
      double far = 0.0;
      if constexpr (kSolvers > 1) {
        // off the chain: the far sums, then wait for the other warp's tile
        far = take_far(part + (fm >> 8), fm & 0xff, pend);
        __syncwarp();
        if (t > 0) {
          if constexpr (kTileBars) {
            mbar_wait(&tbar[t - 1], 0);
          } else if constexpr (kWaitL == kWaitValue) {
            // the previous tile's values are their own readiness (lane j
            // watches row j; the warp leaves the spin together)
            const volatile double* pz = z + (t - 1) * kTile + lane;
            while (__any_sync(0xffffffffu, is_pending(*pz))) {
            }
          } else {
            while (ld_acquire(&done_l) < t) {
            }
          }
        }
      }
      double nb = 0.0;
      if (wn == kDenseNbr) {
        if (t > 1) nb += neighbour(T + kNbrOff, 0, j, z + (t - 2) * kTile);
        if (t > 0) nb += neighbour(T + kNbrOff, kTile, j, z + (t - 1) * kTile);
      } else {
        nb = ell_neighbours(T, wn, j, z + (t - 2) * kTile);
      }
      if constexpr (kSolvers == 1) far = take_far(part + (fm >> 8), fm & 0xff, pend);
      __syncwarp();
      if (tr && lane == 0) tr[4 * t + 1] = clock64();
      // z_t = L_tt^-1 r with r = b - (known sums): one dot product per row
      // over the tile's residuals instead of a 32-step substitution chain
      rbuf[j] = bi - (nb + far);
      __syncwarp();
      double zj = valid ? tile_inverse_dot<true>(T, rbuf, j) : 0.0;
      __syncwarp();  // rbuf is rewritten by the next tile
      if (valid) *reinterpret_cast<volatile double*>(z + i) = zj;
      __syncwarp();  // every lane is done with the slot
      if (lane == 0) {
        if (kProducer) mbar_arrive(&empty[slot]);
        if constexpr (kTileBars)
          mbar_arrive(&tbar[t]);  // release: the tile's z is visible to whoever acquires it
        else if constexpr (kAcqL)
          st_release(&done_l, t + 1);
        else
          *reinterpret_cast<volatile int*>(&done_l) = t + 1;
        if (tr) tr[4 * t + 2] = clock64();
        if (!kProducer && t + kDepth < 2 * nt)
          issue(t + kDepth, kDepth != kRing ? nbytes : next_bytes(t));
      }
      __syncwarp();
      if (tr && lane == 0) tr[4 * t + 3] = clock64();
    }
  } else if (kProducer && home && warp == 1) {
    produce(kRing, min(nt + kRing, 2 * nt));
  } else if (kCl && !home && warp == 0) {
    // puller: copy each tile the home solver publishes into this CTA's copy
    // (readiness is the value itself: spin on the sentinel), then publish the
    // tile count locally
    const volatile int* hd = map_rank(&done_l, 0);
    const double* hz = map_rank(z, 0);
    int pl = 0;
    for (unsigned sl = a.sleep_ns; pl < nt;) {
      const int hv = *hd;
      if (hv <= pl) {
        __nanosleep(sl);
        sl = min(2 * sl, a.sleep_max);
        continue;
      }
      sl = a.sleep_ns;
      for (int t = pl; t < hv; ++t) {
        const int i = t * kTile + lane;
        if (i < n) {
          const volatile double* src = hz + i;
          double v = *src;
          while (is_pending(v)) v = *src;
          *reinterpret_cast<volatile double*>(z + i) = v;
        }
      }
      __syncwarp();
      if (lane == 0) *reinterpret_cast<volatile int*>(&done_l) = hv;
      pl = hv;
    }
  } else {
    // workers: far items of L rows, rows ascending
    const int lw = home ? warp - kFirstWorker : warp - 1;  // scratch slot in this CTA
    const int w = home ? lw : kWorkers + static_cast<int>(crank - 1) * (kWarps - 1) + lw;
    const double* fv = a.lval + a.loff[b];
    const uint16_t* fc = a.lcol + a.loff[b];
    const int4* items = a.litems + a.lioff[b];
    const int nitems = a.lnum[b];
    const int* rp = a.lrp + r0 + b;
    double* scr = scratch + lw * kGroupEntries;
    const int* wait_l = kTileBars ? reinterpret_cast<const int*>(tbar) : done_lh;
    int4 nxt = w < nitems ? items[w] : make_int4(0, 0, 0, 0);
    if (lane < a.pf_items && w + kAllWorkers * lane < nitems) {  // warm the first items
      const int4 d = items[w + kAllWorkers * lane];
      prefetch_far(fv, fc, d.z, d.w);
    }
    for (int it = w; it < nitems; it += kAllWorkers) {
      const int4 d = nxt;
      if (it + kAllWorkers < nitems) nxt = items[it + kAllWorkers];
      if (lane == 0 && a.pf_items && it + kAllWorkers * a.pf_items < nitems) {
        if (a.pf_items == 1) {  // the descriptor just loaded
          prefetch_far(fv, fc, nxt.z, nxt.w);
        } else {
          const int4 f = items[it + kAllWorkers * a.pf_items];
          prefetch_far(fv, fc, f.z, f.w);
        }
      }

      const int i = d.x & 0xffff, k = d.y & 0xff;
      const int slot = static_cast<int>(static_cast<unsigned>(d.x) >> 16);
      long long* rt = (tr && lane == 0) ? tr + 8LL * nt + 4LL * it : nullptr;
      if (rt) rt[0] = clock64();
      if (k & kMultiFlag) {
        const int span = (k & 0x7f) + 1;
        int my;
        bool has;
        const double acc = group_dot<kGroupEntries / 32, kWaitL>(
            fv, fc, d.z, d.w, rp, a.lslot + r0, i, span, zh, scr, lane, a.sleep_ns, wait_l,
            d.y >> 8, a.sleep_max, 0u, my, has);
        if (rt) rt[1] = clock64();
        if (has) *reinterpret_cast<volatile double*>(parth + my) = acc;
      } else {
        const double acc = seg_dot<kUnroll, kWaitL>(fv, fc, d.z, d.w, zh, lane, a.sleep_ns,
                                                    wait_l, d.y >> 8, a.sleep_max, 0u);
        if (rt) rt[1] = clock64();
        if (lane == 0) *reinterpret_cast<volatile double*>(parth + slot) = acc;
      }
      if (rt) {
        rt[2] = clock64();
        rt[3] = (static_cast<long long>(d.y >> 8) << 32) | (i << 3) | (k & 7);
      }
    }
  }
  __syncthreads();  // every L far sum consumed (slots pending again) before the U pass
  if constexpr (kCl) cluster_sync_all();

  // ================================================================ U pass
  if (home && warp < kSolvers) {
    // item q = nt + tt belongs to warp q & 1 (its ring slot)
    for (int tt = kSolvers > 1 ? ((warp - nt) & 1) : 0; tt < nt; tt += kSolvers) {
      const int t = nt - 1 - tt;
      const int q = nt + tt;
      const int i = t * kTile + j;
      const bool valid = i < n;
      const int slot = q % kDepth;
      const double zi = valid ? z[i] : 0.0;
      unsigned nbytes = 0;
      if (kDepth != kRing && q + kDepth < 2 * nt) nbytes = first_bytes(q + kDepth);
      mbar_wait(&bars[slot], (q / kDepth) & 1);
      if (tr && lane == 0) tr[4 * q + 0] = clock64();
      const double* T = ring + slot * kSlotElems;
      const int fm = valid ? meta_int(T, kMetaSeg + j) : 0;
      const int wn = meta_int(T, kHdr);
      double far = 0.0;
      if constexpr (kSolvers > 1) {
        far = take_far(part + (fm >> 8), fm & 0xff, pend);
        __syncwarp();
        if (tt > 0) {
          if constexpr (kTileBars) {
            mbar_wait(&tbar[tt - 1], 1);
          } else if constexpr (kWaitU == kWaitValue) {
            const volatile double* px = x + (t + 1) * kTile + lane;
            while (__any_sync(0xffffffffu, is_pending(*px))) {
            }
          } else {
            while (ld_acquire(&done_u) < tt) {
            }
          }
        }
      }
      double nb = 0.0;
      if (wn == kDenseNbr) {
        if (tt > 0) nb += neighbour(T + kNbrOff, 0, j, x + (t + 1) * kTile);
        if (tt > 1) nb += neighbour(T + kNbrOff, kTile, j, x + (t + 2) * kTile);
      } else {
        nb = ell_neighbours(T, wn, j, x + (t + 1) * kTile);
      }
      if constexpr (kSolvers == 1) far = take_far(part + (fm >> 8), fm & 0xff, pend);
      __syncwarp();
      if (tr && lane == 0) tr[4 * q + 1] = clock64();
      // x_t = U_tt^-1 r with r = z - (known sums)
      rbuf[j] = zi - (nb + far);
      __syncwarp();
      double xj = valid ? tile_inverse_dot<false>(T, rbuf, j) : 0.0;
      __syncwarp();
      if (valid) *reinterpret_cast<volatile double*>(x + i) = xj;
      __syncwarp();
      if (lane == 0) {
        if (kProducer) mbar_arrive(&empty[slot]);
        if constexpr (kTileBars) {
          mbar_arrive(&tbar[tt]);
        } else if (kInPlace) {
          if constexpr (kCl) {
            // cluster scope: the remote pullers acquire it before copying x
            st_release_cluster(&done_u, tt + 1);
          } else {
            st_release(&done_u, tt + 1);
          }
        } else {
          *reinterpret_cast<volatile int*>(&done_u) = tt + 1;
        }
        if (tr) tr[4 * q + 2] = clock64();
        if (!kProducer && q + kDepth < 2 * nt)
          issue(q + kDepth, kDepth != kRing ? nbytes : next_bytes(q));
      }
      __syncwarp();
      if (tr && lane == 0) tr[4 * q + 3] = clock64();
    }
  } else if (kProducer && home && warp == 1) {
    produce(nt + kRing, 2 * nt);
  } else if (kCl && !home && warp == 0) {
    // puller, U pass.  Separate x (the cluster kernels): readiness is the
    // value itself, as in the L pass, so the solver publishes its counter
    // without a cluster-scope fence.  In place: the home's counter with
    // cluster-scope acquire, republished locally with a release.
    const int* hd = map_rank(&done_u, 0);
    const double* hx = map_rank(x, 0);
    int pu = 0;
    for (unsigned sl = a.sleep_ns; pu < nt;) {
      const int hv = kInPlace ? ld_acquire_cluster(hd) : *reinterpret_cast<const volatile int*>(hd);
      if (hv <= pu) {
        __nanosleep(sl);
        sl = min(2 * sl, a.sleep_max);
        continue;
      }
      sl = a.sleep_ns;
      for (int tt = pu; tt < hv; ++tt) {
        const int i = (nt - 1 - tt) * kTile + lane;
        if (i < n) {
          const volatile double* src = hx + i;
          double v = *src;
          while (!kInPlace && is_pending(v)) v = *src;
          *reinterpret_cast<volatile double*>(x + i) = v;
        }
      }
      __syncwarp();
      if (lane == 0) {
        if (kInPlace)
          st_release(&done_u, hv);
        else
          *reinterpret_cast<volatile int*>(&done_u) = hv;
      }
      pu = hv;
    }
  } else {
    // workers: far items of U rows, rows descending
    const int lw = home ? warp - kFirstWorker : warp - 1;
    const int w = home ? lw : kWorkers + static_cast<int>(crank - 1) * (kWarps - 1) + lw;
    const double* fv = a.uval + a.uoff[b];
    const uint16_t* fc = a.ucol + a.uoff[b];
    const int4* items = a.uitems + a.uioff[b];
    const int nitems = a.unum[b];
    const long long lit = a.lnum[b];
    const int* rp = a.urp + r0 + b;
    double* scr = scratch + lw * kGroupEntries;
    const int* wait_u = kTileBars ? reinterpret_cast<const int*>(tbar) : done_uh;
    int4 nxt = w < nitems ? items[w] : make_int4(0, 0, 0, 0);
    if (lane < a.pf_u && w + kAllWorkers * lane < nitems) {  // warm the first items
      const int4 d = items[w + kAllWorkers * lane];
      prefetch_far(fv, fc, d.z, d.w);
    }
    for (int it = w; it < nitems; it += kAllWorkers) {
      const int4 d = nxt;
      if (it + kAllWorkers < nitems) nxt = items[it + kAllWorkers];
      if (lane == 0 && a.pf_u && it + kAllWorkers * a.pf_u < nitems) {
        if (a.pf_u == 1) {  // the descriptor just loaded
          prefetch_far(fv, fc, nxt.z, nxt.w);
        } else {
          const int4 f = items[it + kAllWorkers * a.pf_u];
          prefetch_far(fv, fc, f.z, f.w);
        }
      }

      const int i = d.x & 0xffff, k = d.y & 0xff;
      const int slot = static_cast<int>(static_cast<unsigned>(d.x) >> 16);
      long long* rt = (tr && lane == 0) ? tr + 8LL * nt + 4LL * (lit + it) : nullptr;
      if (rt) rt[0] = clock64();
      if (k & kMultiFlag) {
        const int span = (k & 0x7f) + 1;
        int my;
        bool has;
        const double acc = group_dot<kGroupEntries / 32, kWaitU>(
            fv, fc, d.z, d.w, rp, a.uslot + r0, i, span, xh, scr, lane, a.sleep_ns, wait_u,
            d.y >> 8, a.sleep_max, 1u, my, has);
        if (rt) rt[1] = clock64();
        if (has) *reinterpret_cast<volatile double*>(parth + my) = acc;
      } else {
        const double acc = seg_dot<kUnroll, kWaitU>(fv, fc, d.z, d.w, xh, lane, a.sleep_ns,
                                                    wait_u, d.y >> 8, a.sleep_max, 1u);
        if (rt) rt[1] = clock64();
        if (lane == 0) *reinterpret_cast<volatile double*>(parth + slot) = acc;
      }
      if (rt) {
        rt[2] = clock64();
        rt[3] = (static_cast<long long>(d.y >> 8) << 32) | (i << 3) | (k & 7);
      }
    }
  }
  __syncthreads();
  // the home CTA's shared memory stays alive until every remote worker is done
  if constexpr (kCl) cluster_sync_all();
  if (!home) return;
  // epilogue: the block's solution leaves in one coalesced sweep
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    out[r0 + i] = sub ? sub[r0 + i] - x[i] : x[i];
}

template <bool kInPlace>
size_t smem_bytes(int dim_max, int workers, int slots, bool tile_bars = false, int depth = kRing) {
  const size_t dpad = (static_cast<size_t>(dim_max) + kTile - 1) & ~static_cast<size_t>(kTile - 1);
  return sizeof(double) * (static_cast<size_t>(depth) * kSlotElems +
                           ((static_cast<size_t>(slots) + 1) & ~static_cast<size_t>(1)) +
                           (kInPlace ? 1 : 2) * dpad +
                           static_cast<size_t>(workers) * kGroupEntries + 2 * kTile +
                           (tile_bars ? dpad / kTile : 0));  // one mbarrier per tile
}

}  // namespace

void ensure_smem(const void* kern, size_t smem) {
  // the attribute is per device: cache it per (device, kernel)
  static std::mutex mu;
  struct Entry {
    int dev;
    const void* kern;
    size_t smem;
  };
  static std::vector<Entry> set;
  int dev = 0;
  MSCG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : set)
    if (e.dev == dev && e.kern == kern) {
      if (smem > e.smem) {
        MSCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
        e.smem = smem;
      }
      return;
    }
  if (smem > 48 * 1024)
    MSCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  set.push_back({dev, kern, std::max<size_t>(smem, 48 * 1024)});
}

void block_trisolve(const FactorSet& fs, const double* rhs, double* out, const double* sub,
                    cudaStream_t s, long long* trace, int chunk, const int* order, int norder) {
  if (fs.nblocks == 0) return;
  if (order) chunk = -1;
  const int pos0 = chunk < 0 ? 0 : fs.h_chunk[chunk];
  const int npos = order ? norder : (chunk < 0 ? fs.nblocks : fs.h_chunk[chunk + 1] - pos0);
  if (npos <= 0) return;
  TriArgs a;
  a.row0 = fs.row0.as<int>();
  a.dim = fs.dim.as<int>();
  a.loff = fs.loff.as<long long>();
  a.uoff = fs.uoff.as<long long>();
  a.toff = fs.toff.as<long long>();
  a.lioff = fs.lioff.as<long long>();
  a.uioff = fs.uioff.as<long long>();
  a.lval = fs.lval.as<double>();
  a.lcol = fs.lcol.as<uint16_t>();
  a.uval = fs.uval.as<double>();
  a.ucol = fs.ucol.as<uint16_t>();
  a.ltile = fs.ltile.as<double>();
  a.utile = fs.utile.as<double>();
  a.lwidth = fs.lwidth.as<int>();
  a.uwidth = fs.uwidth.as<int>();
  a.litems = fs.litems.as<int4>();
  a.uitems = fs.uitems.as<int4>();
  a.lnum = fs.lnum.as<int>();
  a.unum = fs.unum.as<int>();
  a.lrp = fs.lrp.as<int>();
  a.urp = fs.urp.as<int>();
  a.lslot = fs.lslot.as<int>();
  a.uslot = fs.uslot.as<int>();
  a.max_slots = fs.max_slots;
  a.perm = fs.has_perm ? fs.perm.as<int>() : nullptr;
  a.order = order ? order : (chunk < 0 ? fs.order.as<int>() : fs.order_chunked.as<int>());
  a.pos0 = pos0;
  a.dim_max = fs.max_dim;
  a.trace = trace;
  static const unsigned sleep_ns = [] {
    const char* e = getenv("MSCG_TRI_SLEEP_NS");
    return e ? static_cast<unsigned>(atoi(e)) : 32u;
  }();
  a.sleep_ns = sleep_ns;
  static const unsigned sleep_max = [] {
    const char* e = getenv("MSCG_TRI_SLEEP_MAX");
    return e ? static_cast<unsigned>(atoi(e)) : 256u;
  }();
  a.sleep_max = sleep_max < sleep_ns ? sleep_ns : sleep_max;
  static const int pf_items = [] {
    const char* e = getenv("MSCG_TRI_PF");
    return e ? atoi(e) : 1;
  }();
  a.pf_items = pf_items;
  static const int pf_u = [] {
    const char* e = getenv("MSCG_TRI_PFU");
    return e ? atoi(e) : 1;
  }();
  a.pf_u = pf_u;
  static const int variant = [] {
    const char* e = getenv("MSCG_TRI_VARIANT");
    return e ? atoi(e) : 0;
  }();
  // Readiness through per-tile mbarriers (MSCG_TRI_TILEBARS=0: the
  // release/acquire counters).  With two CTAs per SM the barriers must not
  // cost the second CTA: 228 KB per SM, 1 KB reserved per CTA.
  static const bool tb_env = [] {
    const char* e = getenv("MSCG_TRI_TILEBARS");
    return e ? atoi(e) != 0 : true;
  }();
  constexpr size_t kTwoPerSm = (228 * 1024 - 2 * 1024) / 2 - 128;  // less the static part
  // Solver warps per block (MSCG_TRI_SOLVERS=1|2; see trisolve_kernel): two
  // where the chain is the bound (few blocks: clusters and 32-warp CTAs)
  static const int solvers_env = [] {
    const char* e = getenv("MSCG_TRI_SOLVERS");
    return e ? atoi(e) : 0;
  }();
  const bool two_wide = solvers_env ? solvers_env == 2 : true;    // 32-warp kernels
  const bool two_k16 = solvers_env ? solvers_env == 2 : false;    // 16-warp kernels
  auto check_smem = [&](size_t smem) {
    if (smem > 227 * 1024)
      throw Error(1, "block_trisolve: block of " + std::to_string(fs.max_dim) +
                         " rows exceeds the shared-memory solution vector");
  };
  auto launch = [&](auto kern, int warps, size_t smem) {
    check_smem(smem);
    // the attribute is raised once per kernel and size (a driver call on
    // every launch costs the stream its back-to-back launches)
    ensure_smem(reinterpret_cast<const void*>(kern), smem);
    static const bool verbose = getenv("MSCG_VERBOSE") != nullptr;
    if (verbose)
      fprintf(stderr, "block_trisolve: %d blocks, dim_max %d, far-sum slots %d, smem %zu B\n",
              npos, fs.max_dim, fs.max_slots, smem);
    kern<<<npos, warps * 32, smem, s>>>(a, rhs, out, sub);
  };
  const int d = fs.max_dim, ns = fs.max_slots;
  // Fewer blocks than SMs (cfg2/cfg3): each block has an SM to itself, so
  // large blocks get 31 workers (1024 threads) instead of 15 (cfg2 D-solve
  // 0.645 -> 0.417 ms); small ones (cfg1, ~400 rows) are faster without.
  int sms = 148;
  {
    int dev = 0;
    MSCG_CUDA(cudaGetDevice(&dev));
    MSCG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // Fewer blocks than fill the GPU: a thread-block cluster of C CTAs (C SMs)
  // per block — the home CTA solves, the others stream far entries into its
  // shared memory over DSMEM (MSCG_TRI_CLUSTER=0 off, =C forces the size).
  static const int cl_env = [] {
    const char* e = getenv("MSCG_TRI_CLUSTER");
    return e ? atoi(e) : -1;
  }();
  // (a traced solve always takes the default kernel: only it is instantiated
  // with kTrace)
  if (variant == 0 && d > 1024 && cl_env != 0 && npos * 2 <= sms && !trace) {
    // separate z and x (not in place): the U pass needs no cluster fence
    // (31 workers in the remote CTAs; two solvers need the four-slot ring)
    const bool two_cl = two_wide && smem_bytes<false>(d, 31, ns, false, 4) <= 227 * 1024;
    const size_t smc = smem_bytes<false>(d, 31, ns, false, two_cl ? 4 : kRing);
    check_smem(smc);
    auto config = [&](int c) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(npos * c);
      cfg.blockDim = dim3(32 * 32);
      cfg.dynamicSmemBytes = smc;
      cfg.stream = s;
      return cfg;
    };
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    // the largest cluster whose clusters all fit at once (a cluster must sit
    // in one GPC: 16 clusters of 8 full SMs need not fit even when 128 SMs
    // are free; cfg2 16 blocks: 6 CTAs 0.288 ms, 4: 0.297, 1: 0.420)
    auto try_size = [&](int c, auto kern) {
      if (cl_env > 0 ? c != cl_env : npos * c > sms) return false;
      ensure_smem(reinterpret_cast<const void*>(kern), smc);
      cudaLaunchConfig_t cfg = config(c);
      at[0].val.clusterDim.x = c;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int active = 0;
      if (cl_env <= 0 &&
          (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) != cudaSuccess || active < npos)) {
        cudaGetLastError();
        return false;
      }
      MSCG_CUDA(cudaLaunchKernelEx(&cfg, kern, a, rhs, out, sub));
      MSCG_CUDA(cudaGetLastError());
      return true;
    };
    if (two_cl
            ? (try_size(8, trisolve_kernel<32, 4, 1, false, false, 8, false, false, 2>) ||
               try_size(6, trisolve_kernel<32, 4, 1, false, false, 6, false, false, 2>) ||
               try_size(4, trisolve_kernel<32, 4, 1, false, false, 4, false, false, 2>) ||
               try_size(3, trisolve_kernel<32, 4, 1, false, false, 3, false, false, 2>) ||
               try_size(2, trisolve_kernel<32, 4, 1, false, false, 2, false, false, 2>))
            : (try_size(8, trisolve_kernel<32, 4, 1, false, false, 8>) ||
               try_size(6, trisolve_kernel<32, 4, 1, false, false, 6>) ||
               try_size(4, trisolve_kernel<32, 4, 1, false, false, 4>) ||
               try_size(3, trisolve_kernel<32, 4, 1, false, false, 3>) ||
               try_size(2, trisolve_kernel<32, 4, 1, false, false, 2>)))
      return;
  }
  if (variant == 0 && npos <= sms && d > 1024 && !trace) {
    if (tb_env && smem_bytes<true>(d, 31, ns, true) <= 227 * 1024) {
      if (two_wide && smem_bytes<true>(d, 30, ns, true, 4) <= 227 * 1024)
        launch(trisolve_kernel<32, 4, 1, true, false, 1, true, false, 2>, 32,
               smem_bytes<true>(d, 30, ns, true, 4));
      else
        launch(trisolve_kernel<32, 4, 1, true, false, 1, true>, 32,
               smem_bytes<true>(d, 31, ns, true));
    } else {
      launch(trisolve_kernel<32, 4, 1, true, false>, 32, smem_bytes<true>(d, 31, ns));
    }
    MSCG_CUDA(cudaGetLastError());
    return;
  }
  // Last partial wave (T < SMs blocks after the full waves of 2 CTAs per
  // SM, cfg4: 1024 = 3 x 296 + 136): its blocks, the smallest in LPT order,
  // run as 32-warp CTAs on a side stream so each gets a whole SM's workers
  // as SMs drain, instead of half-empty SMs at the end of one launch.
  const int tail = npos % (2 * sms);
  static const bool split_tail = getenv("MSCG_TRI_NO_TAIL") == nullptr;
  if (split_tail && !trace && variant == 0 && chunk < 0 && d > 1024 && npos > 2 * sms && tail > 0 &&
      tail <= sms) {
    std::lock_guard<std::mutex> lk(fs.tail_mu);
    if (!fs.tail_stream) {
      MSCG_CUDA(cudaStreamCreateWithFlags(&fs.tail_stream, cudaStreamNonBlocking));
      MSCG_CUDA(cudaEventCreateWithFlags(&fs.tail_ev[0], cudaEventDisableTiming));
      MSCG_CUDA(cudaEventCreateWithFlags(&fs.tail_ev[1], cudaEventDisableTiming));
    }
    MSCG_CUDA(cudaEventRecord(fs.tail_ev[0], s));
    MSCG_CUDA(cudaStreamWaitEvent(fs.tail_stream, fs.tail_ev[0], 0));
    const int head = npos - tail;
    check_smem(smem_bytes<true>(d, 31, ns));
    {
      const bool tb = tb_env && smem_bytes<true>(d, 15, ns, true) <= kTwoPerSm;
      const bool two16 = tb && two_k16 && smem_bytes<true>(d, 14, ns, true, 4) <= 227 * 1024;
      auto k16 = tb ? (two16 ? trisolve_kernel<16, 4, 2, true, false, 1, true, false, 2>
                             : trisolve_kernel<16, 4, 2, true, false, 1, true>)
                    : trisolve_kernel<16, 4, 2, true, false>;
      const size_t sm16 = two16 ? smem_bytes<true>(d, 14, ns, true, 4) : smem_bytes<true>(d, 15, ns, tb);
      ensure_smem(reinterpret_cast<const void*>(k16), sm16);
      k16<<<head, 16 * 32, sm16, s>>>(a, rhs, out, sub);
      MSCG_CUDA(cudaGetLastError());
    }
    {
      TriArgs at = a;
      at.pos0 = pos0 + head;
      const bool tb = tb_env && smem_bytes<true>(d, 31, ns, true) <= 227 * 1024;
      const bool two = tb && two_wide && smem_bytes<true>(d, 30, ns, true, 4) <= 227 * 1024;
      auto k32 = tb ? (two ? trisolve_kernel<32, 4, 1, true, false, 1, true, false, 2>
                           : trisolve_kernel<32, 4, 1, true, false, 1, true>)
                    : trisolve_kernel<32, 4, 1, true, false>;
      const size_t sm32 = two ? smem_bytes<true>(d, 30, ns, true, 4) : smem_bytes<true>(d, 31, ns, tb);
      ensure_smem(reinterpret_cast<const void*>(k32), sm32);
      k32<<<tail, 32 * 32, sm32, fs.tail_stream>>>(at, rhs, out, sub);
      MSCG_CUDA(cudaGetLastError());
    }
    MSCG_CUDA(cudaEventRecord(fs.tail_ev[1], fs.tail_stream));
    MSCG_CUDA(cudaStreamWaitEvent(s, fs.tail_ev[1], 0));
    return;
  }
  switch (variant) {
    case 2:  // producer warp issues the near tiles, 14 workers
      launch(trisolve_kernel<16, 4, 2, true, true>, 16, smem_bytes<true>(d, 14, ns));
      break;
    case 3:  // separate z and x vectors
      launch(trisolve_kernel<16, 4, 2, false, false>, 16, smem_bytes<false>(d, 15, ns));
      break;
    default:  // 2 CTAs/SM (64 registers), x overwrites z in place
      if (trace && smem_bytes<true>(d, 15, ns, true) <= kTwoPerSm)
        launch(trisolve_kernel<16, 4, 2, true, false, 1, true, true>, 16,
               smem_bytes<true>(d, 15, ns, true));
      else if (tb_env && two_k16 && smem_bytes<true>(d, 14, ns, true, 4) <= 227 * 1024)
        launch(trisolve_kernel<16, 4, 2, true, false, 1, true, false, 2>, 16,
               smem_bytes<true>(d, 14, ns, true, 4));
      else if (tb_env && smem_bytes<true>(d, 15, ns, true) <= kTwoPerSm)
        launch(trisolve_kernel<16, 4, 2, true, false, 1, true>, 16,
               smem_bytes<true>(d, 15, ns, true));
      else
        launch(trisolve_kernel<16, 4, 2, true, false>, 16, smem_bytes<true>(d, 15, ns));
      break;
  }
  MSCG_CUDA(cudaGetLastError());
}

}  // namespace mscg
