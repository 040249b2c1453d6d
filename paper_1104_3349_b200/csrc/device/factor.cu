// Batched numeric factorisation of independent blocks (setup-side hot path).
//
//  * ilut_kernel — one warp owns one block (persistent CTAs pull blocks from
//    an atomic counter) and replays the reference's row-wise IKJ ILUT
//    (factor_ilut, proj/src/factorization.cpp:34-127) exactly:
//      - tau = tol * sqrt(sum of squares of the original block row), summed
//        in column order (:55-58);
//      - pending pivots k < i processed in ascending order (the std::set of
//        :64-94): fills only add indices > k, so "next set bit of the
//        presence bitmap after k" is the same sequence;
//      - multiplier m = w_k / u_kk dropped if |m| < tau or m == 0 (:77-80);
//      - work[j] -= m * u_kj with separately rounded multiply and subtract
//        (no FMA), one lane per j: the same operations in the same order per
//        entry as the reference, so factors are bit-identical;
//      - L keeps nonzero multipliers, U keeps |v| >= tau && v != 0, the
//        diagonal always; a zero diagonal is SingularMatrixError(i) (:97-116).
//    The working row lives in shared memory (dense fp64 + presence bitmap);
//    kept U rows stream to a global pool and are replayed from L2.
//  * dense_lu_kernel — one CTA per block: the reference's partial-pivoting
//    LU (dense_lu, proj/src/dense_matrix.cpp:85-123: first maximum wins,
//    exactly-zero pivot column throws, whole-row swaps) on an L2-resident
//    dense copy, then re-sparsified like factor_exact (factorization.cpp:11-32).
//    Used for the interface (Schur) blocks and for interior blocks with
//    dim <= sA.
//  * pack_kernel — moves each block's rows from the pools into the solve
//    layout (block-contiguous, uint16 local columns; see FactorSet).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>
#include <string>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

struct PoolView {
  uint16_t* lcol;
  double* lval;
  uint16_t* ucol;
  double* uval;
  unsigned long long* lused;  // entries handed out
  unsigned long long* uused;
  unsigned long long cap;     // entries per pool
  // per factor-set row (row0[b] + i)
  uint32_t* lstart;
  int* llen;
  uint32_t* ustart;
  int* ulen;
  double* udiag;
  // per block
  long long* blk_nnz_l;
  long long* blk_nnz_u;
  unsigned long long* err;     // min over (block << 32 | pivot) of failures
  int* overflow;
};

constexpr unsigned kChunk = 1u << 18;  // ILUT pool chunk (entries)

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

// ---- ILUT ------------------------------------------------------------------

// Finished-row record read by later pivots: {U_kk bits, ustart | ulen << 32}.
__device__ __forceinline__ longlong2 load_rec(const longlong2* recs, int g) {
  return recs[g];
}

constexpr int kIlutBatch = 4;  // U-row entries per lane in flight per round
constexpr int kNone = 0x7fffffff;
constexpr int kPfCands = 32;   // cached candidates whose U rows are L2-prefetched at refill
constexpr bool kIlutPrefetch = true;

// Fire-and-forget L2 prefetch of a finished U row (values + columns): the
// pivots' U rows are re-read from HBM (a block's U outgrows its share of
// L2), so the rows of the upcoming pivots are requested well ahead.
__device__ __forceinline__ void prefetch_urow(const PoolView& pool, long long ry) {
  const uint32_t s0 = static_cast<uint32_t>(ry);
  const int len = static_cast<int>(static_cast<unsigned long long>(ry) >> 32);
  if (len <= 0) return;
  const unsigned long long v0 = reinterpret_cast<unsigned long long>(pool.uval + s0) & ~15ull;
  const unsigned long long v1 = (reinterpret_cast<unsigned long long>(pool.uval + s0 + len) + 15) & ~15ull;
  const unsigned long long c0 = reinterpret_cast<unsigned long long>(pool.ucol + s0) & ~15ull;
  const unsigned long long c1 = (reinterpret_cast<unsigned long long>(pool.ucol + s0 + len) + 15) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v0), "r"(static_cast<unsigned>(v1 - v0)) : "memory");
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c0), "r"(static_cast<unsigned>(c1 - c0)) : "memory");
}

// Candidate cache: lane L holds one pending column (cand, kNone if empty) and
// its row record (rec, loaded asynchronously).  Invariant: the cache holds
// every pending column in (kk, hi) — refill() scans the bitmap from `from`,
// caches the first (up to) 32 set bits below `end` and returns hi.
__device__ __forceinline__ int refill(const uint32_t* bits, int from, int end, unsigned lane,
                                      int* slot, const longlong2* brec, int& cand,
                                      longlong2& rec, bool& pf) {
  cand = kNone;
  pf = false;
  for (int wb = from >> 5; (wb << 5) < end; wb += 32) {
    const int w = wb + static_cast<int>(lane);
    unsigned word = 0;
    if ((w << 5) < end) {
      word = bits[w];
      if (w == (from >> 5)) word &= ~0u << (from & 31);
      if (((w + 1) << 5) > end) word &= (1u << (end & 31)) - 1u;
    }
    const int c = __popc(word);
    int pre = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, pre, o);
      if (static_cast<int>(lane) >= o) pre += v;
    }
    const int total = __shfl_sync(0xffffffffu, pre, 31);
    if (total == 0) continue;
    for (int r = pre - c; word && r < 32; ++r) {
      slot[r] = (w << 5) + __ffs(word) - 1;
      word &= word - 1;
    }
    __syncwarp();
    if (static_cast<int>(lane) < min(total, 32)) {
      cand = slot[lane];
      rec = load_rec(brec, cand);
      pf = static_cast<int>(lane) < kPfCands;
    }
    const int hi = total > 32 ? slot[31] + 1 : min(end, (wb + 32) << 5);
    __syncwarp();  // slot is rewritten by the next refill
    return hi;
  }
  return end;
}

// Insert a new pending column f (kk < f < hi) into the cache.
__device__ __forceinline__ void cache_insert(int f, unsigned lane, const longlong2* brec,
                                             int& cand, longlong2& rec, int& hi, bool& pf) {
  if (f >= hi) return;
  const unsigned freem = __ballot_sync(0xffffffffu, cand == kNone);
  if (freem) {
    if (static_cast<int>(lane) == __ffs(freem) - 1) {
      cand = f;
      rec = load_rec(brec, f);
      pf = true;
    }
    return;
  }
  const int mx = __reduce_max_sync(0xffffffffu, cand);
  if (mx > f) {  // full: the largest candidate leaves, hi drops to it
    hi = mx;
    if (cand == mx) {
      cand = f;
      rec = load_rec(brec, f);
      pf = true;
    }
  } else {
    hi = f;
  }
}

// Slots of a round of R entries per lane that hold entries (warp-uniform).
template <int R>
__device__ __forceinline__ int round_slots(int len, int base) {
  return min(R, (len - base + 31) >> 5);
}
template <int R>
__device__ __forceinline__ void load_round(const PoolView& pool, uint32_t s0, int len, int base,
                                           unsigned lane, int (&jj)[R], double (&uu)[R]) {
  const int nr = round_slots<R>(len, base);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int q = base + static_cast<int>(lane) + 32 * r;
    jj[r] = -1;
    if (r < nr && q < len) {
      jj[r] = pool.ucol[s0 + q];
      uu[r] = pool.uval[s0 + q];
    }
  }
}

// Absent entries of the working row hold a NaN pattern no arithmetic
// produces, so the update's own load tells whether an entry is new (the
// reference's `present` flag, factorization.cpp:84-88) without an atomic
// round trip; the bitmap (ascending scans) is kept exact by setting a bit
// only when an entry appears.
constexpr long long kAbsent = 0x7ff4a85a5e5a0001LL;
__device__ __forceinline__ double absent_value() { return __longlong_as_double(kAbsent); }
__device__ __forceinline__ bool is_absent(double v) { return __double_as_longlong(v) == kAbsent; }

// work[j] -= m * u_kj for one round of a U row (reference factorization.cpp:
// 84-94: a new entry starts at 0.0), new entries' bits set, and new pending
// columns below hi inserted into the candidate cache.
template <int R>
__device__ __forceinline__ void update_round(const int (&jj)[R], const double (&uu)[R], int nr,
                                             double m, int kk, double* work, uint32_t* bits,
                                             unsigned lane, const longlong2* brec, int& cand,
                                             longlong2& rec, int& hi, bool& pf) {
  double wv[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r < nr && jj[r] >= 0) wv[r] = work[jj[r]];
  unsigned fills = 0;  // slots whose entry is new and a pending pivot below hi
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r < nr && jj[r] >= 0) {
      const int j = jj[r];
      const bool fresh = is_absent(wv[r]);
      work[j] = __dsub_rn(fresh ? 0.0 : wv[r], __dmul_rn(m, uu[r]));
      if (fresh) {
        atomicOr(&bits[j >> 5], 1u << (j & 31));
        if (j > kk && j < hi) fills |= 1u << r;
      }
    }
  }
  if (__any_sync(0xffffffffu, fills != 0)) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      unsigned fm = __ballot_sync(0xffffffffu, (fills >> r) & 1u);
      while (fm) {
        const int src = __ffs(fm) - 1;
        fm &= fm - 1;
        cache_insert(__shfl_sync(0xffffffffu, jj[r], src), lane, brec, cand, rec, hi, pf);
      }
    }
  }
}

__global__ void __launch_bounds__(32) ilut_kernel(
    int nblocks, const int* __restrict__ blk_row0, const int* __restrict__ blk_dim,
    const int* __restrict__ blk_col0, const int* __restrict__ set_row0,
    const int* __restrict__ blk_ids, const int* __restrict__ a_rp,
    const int* __restrict__ a_ci, const double* __restrict__ a_v, double tol,
    PoolView pool, longlong2* recs, int* block_counter, int dim_max) {
  // The warp's shared memory is only the working row (dense fp64), its
  // presence bitmap and a 32-entry scratch, so that 8 warps fit per SM;
  // finished rows are read back through their 16-byte records and the pools
  // (L1/L2), the records of upcoming pivots cached one per lane.
  extern __shared__ __align__(16) unsigned char smem[];
  double* work = reinterpret_cast<double*>(smem);
  uint32_t* bits = reinterpret_cast<uint32_t*>(work + dim_max);
  int* slot = reinterpret_cast<int*>(bits + ((dim_max + 31) / 32 + 1));
  const unsigned lane = lane_id();
  const unsigned ltmask = (1u << lane) - 1u;

  for (int i = lane; i < dim_max; i += 32) work[i] = absent_value();
  for (int i = lane; i < (dim_max + 31) / 32 + 1; i += 32) bits[i] = 0u;
  unsigned long long lcur = 0, lend = 0, ucur = 0, uend = 0;
  __syncwarp();

  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(block_counter, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nblocks) break;
    const int b = blk_ids[t];
    const int row0 = blk_row0[b], dim = blk_dim[b], col0 = blk_col0[b];
    const int srow0 = set_row0[b];
    const longlong2* brec = recs + srow0;
    long long tot_l = 0, tot_u = 0;
    bool failed = false;

    for (int i = 0; i < dim && !failed; ++i) {
      const int rb = a_rp[row0 + i], re = a_rp[row0 + i + 1];
      // Row norm over in-block entries, in column order (lane 0, rows are short).
      double norm = 0.0;
      if (lane == 0) {
        for (int k = rb; k < re; ++k) {
          const int c = a_ci[k] - col0;
          if (c >= 0 && c < dim) {
            const double v = a_v[k];
            norm = __dadd_rn(norm, __dmul_rn(v, v));
          }
        }
      }
      norm = __shfl_sync(0xffffffffu, norm, 0);
      const double tau = __dmul_rn(tol, __dsqrt_rn(norm));
      for (int k = rb + lane; k < re; k += 32) {
        const int c = a_ci[k] - col0;
        if (c >= 0 && c < dim) {
          work[c] = a_v[k];
          atomicOr(&bits[c >> 5], 1u << (c & 31));
        }
      }
      __syncwarp();

      // Pivot loop over the pending columns k < i in ascending order: the
      // next pivot is the smallest cached candidate (fills of each update
      // are inserted), and the U row of the one after it is in flight while
      // the current pivot's update runs.
      int cand = kNone;
      longlong2 rec = make_longlong2(0, 0);
      bool pf = false;  // this lane's candidate row still to be prefetched
      int hi = refill(bits, 0, i, lane, slot, brec, cand, rec, pf);
      int kk = __reduce_min_sync(0xffffffffu, cand);
      int jj[kIlutBatch], pj[kIlutBatch];
      double uu[kIlutBatch], pu[kIlutBatch];
      bool have = false;
      while (kk != kNone) {
        const int own = __ffs(__ballot_sync(0xffffffffu, cand == kk)) - 1;
        const long long rx = __shfl_sync(0xffffffffu, rec.x, own);
        const long long ry = __shfl_sync(0xffffffffu, rec.y, own);
        if (static_cast<int>(lane) == own) {
          cand = kNone;
          pf = false;
        }
        const double ukk = __longlong_as_double(rx);
        const uint32_t s0 = static_cast<uint32_t>(ry);
        const int len = static_cast<int>(static_cast<unsigned long long>(ry) >> 32);
        if (!have) load_round<kIlutBatch>(pool, s0, len, 0, lane, jj, uu);
        // the next candidate's U row goes in flight now
        const int k2 = __reduce_min_sync(0xffffffffu, cand);
        if (k2 != kNone) {
          const int own2 = __ffs(__ballot_sync(0xffffffffu, cand == k2)) - 1;
          const long long ry2 = __shfl_sync(0xffffffffu, rec.y, own2);
          load_round<kIlutBatch>(pool, static_cast<uint32_t>(ry2),
                                 static_cast<int>(static_cast<unsigned long long>(ry2) >> 32), 0,
                                 lane, pj, pu);
        }
        if (kIlutPrefetch && pf) {
          prefetch_urow(pool, rec.y);
          pf = false;
        }
        const double m = __ddiv_rn(work[kk], ukk);
        if (fabs(m) < tau || m == 0.0) {
          if (lane == 0) work[kk] = 0.0;
        } else {
          if (lane == 0) work[kk] = m;
          // the first round (prefetched, kIlutBatch entries per lane), then
          // wider rounds for long rows, each round's loads in flight while
          // the previous round updates
          constexpr int kWide = 2 * kIlutBatch;
          int nj[kWide];
          double nu[kWide];
          int base = 32 * kIlutBatch;
          if (base < len) load_round<kWide>(pool, s0, len, base, lane, nj, nu);
          update_round<kIlutBatch>(jj, uu, round_slots<kIlutBatch>(len, 0), m, kk, work, bits,
                                   lane, brec, cand, rec, hi, pf);
          while (base < len) {
            int cj[kWide];
            double cu[kWide];
#pragma unroll
            for (int r = 0; r < kWide; ++r) {
              cj[r] = nj[r];
              cu[r] = nu[r];
            }
            const int cbase = base;
            base += 32 * kWide;
            if (base < len) load_round<kWide>(pool, s0, len, base, lane, nj, nu);
            update_round<kWide>(cj, cu, round_slots<kWide>(len, cbase), m, kk, work, bits, lane,
                                brec, cand, rec, hi, pf);
          }
        }
        __syncwarp();
        int nxt = __reduce_min_sync(0xffffffffu, cand);
        if (nxt == kNone && hi < i) {
          hi = refill(bits, hi, i, lane, slot, brec, cand, rec, pf);
          nxt = __reduce_min_sync(0xffffffffu, cand);
        }
        have = nxt == k2 && k2 != kNone;
        if (have) {
#pragma unroll
          for (int r = 0; r < kIlutBatch; ++r) {
            jj[r] = pj[r];
            uu[r] = pu[r];
          }
        }
        kk = nxt;
      }

      // Reserve pool space for the worst case of this row.
      if (lane == 0) {
        if (lend - lcur < static_cast<unsigned long long>(i)) {
          lcur = atomicAdd(pool.lused, static_cast<unsigned long long>(kChunk));
          lend = lcur + kChunk;
          if (lend > pool.cap) atomicExch(pool.overflow, 1);
        }
        if (uend - ucur < static_cast<unsigned long long>(dim - 1 - i)) {
          ucur = atomicAdd(pool.uused, static_cast<unsigned long long>(kChunk));
          uend = ucur + kChunk;
          if (uend > pool.cap) atomicExch(pool.overflow, 1);
        }
      }
      if (__shfl_sync(0xffffffffu, lend, 0) > pool.cap ||
          __shfl_sync(0xffffffffu, uend, 0) > pool.cap) {
        failed = true;  // overflow: host retries with larger pools
        break;
      }
      unsigned long long lpos = __shfl_sync(0xffffffffu, lcur, 0);
      unsigned long long upos = __shfl_sync(0xffffffffu, ucur, 0);
      const unsigned long long l0 = lpos, u0 = upos;

      // Collect the working row in ascending column order.
      double diag = 0.0;
      const int nwords = (dim + 31) >> 5;
      for (int wb = 0; wb < nwords; wb += 32) {
        const int w = wb + lane;
        const unsigned word = (w < nwords) ? bits[w] : 0u;
        unsigned nz = __ballot_sync(0xffffffffu, word != 0u);
        while (nz) {
          const int f = __ffs(nz) - 1;
          nz &= nz - 1;
          const unsigned wf = __shfl_sync(0xffffffffu, word, f);
          const int j = ((wb + f) << 5) + lane;
          const bool present = (wf >> lane) & 1u;
          const double v = present ? work[j] : 0.0;
          const bool isL = present && j < i && v != 0.0;
          const bool isU = present && j > i && fabs(v) >= tau && v != 0.0;
          const unsigned bl = __ballot_sync(0xffffffffu, isL);
          const unsigned bu = __ballot_sync(0xffffffffu, isU);
          const unsigned bd = __ballot_sync(0xffffffffu, present && j == i);
          if (isL) {
            const unsigned long long pos = lpos + __popc(bl & ltmask);
            pool.lcol[pos] = static_cast<uint16_t>(j);
            pool.lval[pos] = v;
          }
          if (isU) {
            const unsigned long long pos = upos + __popc(bu & ltmask);
            pool.ucol[pos] = static_cast<uint16_t>(j);
            pool.uval[pos] = v;
          }
          if (bd) diag = __shfl_sync(0xffffffffu, v, __ffs(bd) - 1);
          lpos += __popc(bl);
          upos += __popc(bu);
          if (present) work[j] = absent_value();
        }
        if (w < nwords) bits[w] = 0u;
      }
      const int nl = static_cast<int>(lpos - l0), nu = static_cast<int>(upos - u0);
      if (lane == 0) {
        lcur = lpos;
        ucur = upos;
        const int g = srow0 + i;
        pool.lstart[g] = static_cast<uint32_t>(l0);
        pool.llen[g] = nl;
        pool.ustart[g] = static_cast<uint32_t>(u0);
        pool.ulen[g] = nu;
        pool.udiag[g] = diag;
        recs[g] = make_longlong2(__double_as_longlong(diag),
                                 static_cast<long long>((static_cast<unsigned long long>(nu) << 32) |
                                                        static_cast<uint32_t>(u0)));
      }
      tot_l += nl;
      tot_u += nu;
      if (diag == 0.0) {
        if (lane == 0)
          atomicMin(pool.err, (static_cast<unsigned long long>(b) << 32) |
                                  static_cast<unsigned>(i));
        failed = true;
      }
      __syncwarp();
    }
    if (failed) {
      // leave the shared work row clean for the next block
      for (int i = lane; i < dim_max; i += 32) work[i] = absent_value();
      for (int i = lane; i < (dim_max + 31) / 32 + 1; i += 32) bits[i] = 0u;
      __syncwarp();
    }
    if (lane == 0) {
      pool.blk_nnz_l[b] = tot_l;
      pool.blk_nnz_u[b] = tot_u;
    }
  }
}

// ---- dense partial-pivoting LU ---------------------------------------------

constexpr int kLuThreads = 256;

__global__ void __launch_bounds__(kLuThreads) dense_lu_kernel(
    const int* __restrict__ blk_ids, const int* __restrict__ blk_row0,
    const int* __restrict__ blk_dim, const int* __restrict__ blk_col0,
    const int* __restrict__ set_row0, const long long* __restrict__ dense_off,
    double* __restrict__ dense, int* __restrict__ perm_out,
    const int* __restrict__ a_rp, const int* __restrict__ a_ci,
    const double* __restrict__ a_v, PoolView pool) {
  const int b = blk_ids[blockIdx.x];
  const int row0 = blk_row0[b], n = blk_dim[b], col0 = blk_col0[b], srow0 = set_row0[b];
  double* a = dense + dense_off[blockIdx.x];
  int* perm = perm_out + srow0;
  const int tid = threadIdx.x;
  __shared__ double red_v[kLuThreads / 32];
  __shared__ int red_i[kLuThreads / 32];
  __shared__ int s_piv;
  __shared__ double s_best;
  __shared__ unsigned long long s_lbase, s_ubase;
  __shared__ long long s_nl, s_nu;

  for (long long t = tid; t < static_cast<long long>(n) * n; t += blockDim.x) a[t] = 0.0;
  for (int i = tid; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x)
    for (int k = a_rp[row0 + i]; k < a_rp[row0 + i + 1]; ++k) {
      const int c = a_ci[k] - col0;
      if (c >= 0 && c < n) a[static_cast<long long>(i) * n + c] = a_v[k];
    }
  __syncthreads();

  for (int k = 0; k < n; ++k) {
    // argmax |a(i,k)|, i >= k, smallest index among equal maxima.
    double bv = -1.0;
    int bi = n;
    for (int i = k + tid; i < n; i += blockDim.x) {
      const double v = fabs(a[static_cast<long long>(i) * n + k]);
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
      for (int w = 1; w < kLuThreads / 32; ++w)
        if (red_v[w] > v || (red_v[w] == v && red_i[w] < idx)) {
          v = red_v[w];
          idx = red_i[w];
        }
      s_best = v;
      s_piv = idx;
    }
    __syncthreads();
    // All-NaN column: the reference keeps piv = k and continues.
    if (s_piv < n && s_best == 0.0) {  // exactly zero pivot column
      if (tid == 0)
        atomicMin(pool.err, (static_cast<unsigned long long>(b) << 32) |
                                static_cast<unsigned>(k));
      return;
    }
    const int piv = s_piv < n ? s_piv : k;
    if (piv != k) {
      for (int j = tid; j < n; j += blockDim.x) {
        const double t1 = a[static_cast<long long>(k) * n + j];
        a[static_cast<long long>(k) * n + j] = a[static_cast<long long>(piv) * n + j];
        a[static_cast<long long>(piv) * n + j] = t1;
      }
      if (tid == 0) {
        const int t2 = perm[k];
        perm[k] = perm[piv];
        perm[piv] = t2;
      }
    }
    __syncthreads();
    const double pivot = a[static_cast<long long>(k) * n + k];
    for (int i = k + 1 + tid; i < n; i += blockDim.x) {
      double* ai = a + static_cast<long long>(i) * n;
      ai[k] = __ddiv_rn(ai[k], pivot);
    }
    __syncthreads();
    const int m = n - k - 1;
    const long long work = static_cast<long long>(m) * m;
    for (long long t = tid; t < work; t += blockDim.x) {
      const int i = k + 1 + static_cast<int>(t / m);
      const int j = k + 1 + static_cast<int>(t % m);
      const double lik = a[static_cast<long long>(i) * n + k];
      if (lik != 0.0) {
        double* aij = a + static_cast<long long>(i) * n + j;
        *aij = __dsub_rn(*aij, __dmul_rn(lik, a[static_cast<long long>(k) * n + j]));
      }
    }
    __syncthreads();
  }

  // Re-sparsify: count, reserve one contiguous range per block, write rows.
  long long nl = 0, nu = 0;
  for (int i = tid; i < n; i += blockDim.x) {
    const double* ai = a + static_cast<long long>(i) * n;
    for (int j = 0; j < i; ++j) nl += ai[j] != 0.0;
    for (int j = i + 1; j < n; ++j) nu += ai[j] != 0.0;
  }
  if (tid == 0) {
    s_nl = 0;
    s_nu = 0;
  }
  __syncthreads();
  atomicAdd(reinterpret_cast<unsigned long long*>(&s_nl), static_cast<unsigned long long>(nl));
  atomicAdd(reinterpret_cast<unsigned long long*>(&s_nu), static_cast<unsigned long long>(nu));
  __syncthreads();
  if (tid == 0) {
    s_lbase = atomicAdd(pool.lused, static_cast<unsigned long long>(s_nl));
    s_ubase = atomicAdd(pool.uused, static_cast<unsigned long long>(s_nu));
    if (s_lbase + s_nl > pool.cap || s_ubase + s_nu > pool.cap) atomicExch(pool.overflow, 1);
    pool.blk_nnz_l[b] = s_nl;
    pool.blk_nnz_u[b] = s_nu;
  }
  __syncthreads();
  if (s_lbase + s_nl > pool.cap || s_ubase + s_nu > pool.cap) return;
  // Row offsets within the block: sequential prefix by one warp per row is
  // simplest at these sizes; thread 0 computes them.
  __shared__ int s_dummy;
  (void)s_dummy;
  if (tid == 0) {
    unsigned long long lp = s_lbase, up = s_ubase;
    for (int i = 0; i < n; ++i) {
      const double* ai = a + static_cast<long long>(i) * n;
      int cl = 0, cu = 0;
      for (int j = 0; j < i; ++j) cl += ai[j] != 0.0;
      for (int j = i + 1; j < n; ++j) cu += ai[j] != 0.0;
      pool.lstart[srow0 + i] = static_cast<uint32_t>(lp);
      pool.llen[srow0 + i] = cl;
      pool.ustart[srow0 + i] = static_cast<uint32_t>(up);
      pool.ulen[srow0 + i] = cu;
      pool.udiag[srow0 + i] = ai[i];
      lp += cl;
      up += cu;
    }
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned ltmask = (1u << lane) - 1u;
  for (int i = warp; i < n; i += kLuThreads / 32) {
    const double* ai = a + static_cast<long long>(i) * n;
    unsigned long long lp = pool.lstart[srow0 + i], up = pool.ustart[srow0 + i];
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const double v = j < n ? ai[j] : 0.0;
      const bool isL = j < i && v != 0.0;
      const bool isU = j > i && j < n && v != 0.0;
      const unsigned bl = __ballot_sync(0xffffffffu, isL);
      const unsigned bu = __ballot_sync(0xffffffffu, isU);
      if (isL) {
        pool.lcol[lp + __popc(bl & ltmask)] = static_cast<uint16_t>(j);
        pool.lval[lp + __popc(bl & ltmask)] = v;
      }
      if (isU) {
        pool.ucol[up + __popc(bu & ltmask)] = static_cast<uint16_t>(j);
        pool.uval[up + __popc(bu & ltmask)] = v;
      }
      lp += __popc(bl);
      up += __popc(bu);
    }
  }
}

// ---- pools -> tiled solve layout -------------------------------------------

// Far entries: L columns < 32(t-2), U columns >= 32(t+3) (t = row's tile).
__device__ __forceinline__ bool l_far(int c, int i) {
  return c < ((i >> 5) - (kNearTiles - 1)) * kTile;
}
__device__ __forceinline__ bool u_far(int c, int i) {
  return c >= ((i >> 5) + kNearTiles) * kTile;
}
// Neighbour-window entries (the two tiles next to the diagonal tile).
__device__ __forceinline__ bool l_nbr(int c, int i) { return !l_far(c, i) && c < (i >> 5) * kTile; }
__device__ __forceinline__ bool u_nbr(int c, int i) { return !u_far(c, i) && c >= ((i >> 5) + 1) * kTile; }

// Per row far counts (into lrp/urp scratch slots) and per block totals.
__global__ void __launch_bounds__(256) count_far_kernel(
    const int* __restrict__ set_row0, const int* __restrict__ blk_dim, PoolView pool,
    int* __restrict__ lcnt, int* __restrict__ ucnt, int* __restrict__ lnb,
    int* __restrict__ unb, long long* __restrict__ far_l, long long* __restrict__ far_u,
    long long* __restrict__ items_l, long long* __restrict__ items_u, int pieces_l,
    int pieces_u) {
  const int b = blockIdx.x;
  const int r0 = set_row0[b], n = blk_dim[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ unsigned long long sl, su, il, iu;
  if (threadIdx.x == 0) {
    sl = 0;
    su = 0;
    il = 0;
    iu = 0;
  }
  __syncthreads();
  unsigned long long tl = 0, tu = 0, jl = 0, ju = 0;
  for (int i = warp; i < n; i += blockDim.x / 32) {
    const uint32_t ls = pool.lstart[r0 + i], us = pool.ustart[r0 + i];
    const int ll = pool.llen[r0 + i], ul = pool.ulen[r0 + i];
    int cl = 0, cu = 0, nl = 0, nu = 0;
    for (int q = lane; q < ll; q += 32) {
      const int c = pool.lcol[ls + q];
      cl += l_far(c, i);
      nl += l_nbr(c, i);
    }
    for (int q = lane; q < ul; q += 32) {
      const int c = pool.ucol[us + q];
      cu += u_far(c, i);
      nu += u_nbr(c, i);
    }
    cl = __reduce_add_sync(0xffffffffu, cl);
    cu = __reduce_add_sync(0xffffffffu, cu);
    nl = __reduce_add_sync(0xffffffffu, nl);
    nu = __reduce_add_sync(0xffffffffu, nu);
    if (lane == 0) {
      lcnt[r0 + i] = cl;
      ucnt[r0 + i] = cu;
      lnb[r0 + i] = nl;
      unb[r0 + i] = nu;
      tl += cl;
      tu += cu;
      jl += far_pieces(cl, pieces_l);  // upper bounds (the pack may choose fewer)
      ju += far_pieces(cu, pieces_u);
    }
  }
  if (lane == 0) {
    atomicAdd(&sl, tl);
    atomicAdd(&su, tu);
    atomicAdd(&il, jl);
    atomicAdd(&iu, ju);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    far_l[b] = static_cast<long long>(sl);
    far_u[b] = static_cast<long long>(su);
    items_l[b] = static_cast<long long>(il);
    items_u[b] = static_cast<long long>(iu);
  }
}

// Scatter pool rows into near tiles (dense) and far CSR.
__global__ void __launch_bounds__(256) pack_tiled_kernel(
    const int* __restrict__ set_row0, const int* __restrict__ blk_dim, PoolView pool,
    const int* __restrict__ lcnt, const int* __restrict__ ucnt,
    const long long* __restrict__ loff, const long long* __restrict__ uoff,
    const long long* __restrict__ toff, int* __restrict__ lrp, int* __restrict__ urp,
    double* __restrict__ lval, uint16_t* __restrict__ lcol, double* __restrict__ uval,
    uint16_t* __restrict__ ucol, double* __restrict__ ltile, double* __restrict__ utile,
    double* __restrict__ urdiag, const long long* __restrict__ lioff,
    const long long* __restrict__ uioff, int4* __restrict__ litems, int4* __restrict__ uitems,
    int* __restrict__ lnum, int* __restrict__ unum, const int* __restrict__ lnb,
    const int* __restrict__ unb, int* __restrict__ lwidth, int* __restrict__ uwidth,
    int* __restrict__ lslot, int* __restrict__ uslot, int* __restrict__ nslots,
    int4* __restrict__ ltmp, int4* __restrict__ utmp, int pieces_l, int pieces_u, int slack_l,
    int slack_u) {
  const int b = blockIdx.x;
  const int r0 = set_row0[b], n = blk_dim[b];
  const int ntb = (n + kTile - 1) / kTile;
  int* lr = lrp + r0 + b;
  int* ur = urp + r0 + b;
  // pieces per long row chosen for this block (<= pieces_l / pieces_u)
  __shared__ int s_pl, s_pu;
  if (threadIdx.x == 0) {
    // Long rows are cut into pieces by readiness (see `cuts` below); more
    // pieces let a row's early columns stream while the chain is still far
    // from the row.  Every piece owns a far-sum slot in shared memory, so a
    // pass takes more pieces only while its slots stay within what the block
    // needs anyway (the larger of the two passes with the default cut).
    auto slots = [&](const int* cnt, int pieces) {
      int q = 0;
      for (int i = 0; i < n; ++i) q += far_pieces(cnt[r0 + i], pieces);
      return q;
    };
    const int budget = max(slots(lcnt, 1), slots(ucnt, 1));
    int pl = pieces_l, pu = pieces_u;
    while (pl > 1 && slots(lcnt, pl) > budget) --pl;
    while (pu > 1 && slots(ucnt, pu) > budget) --pu;
    s_pl = pl;
    s_pu = pu;
    int sl = 0, su = 0, ql = 0, qu = 0;
    for (int i = 0; i < n; ++i) {
      lr[i] = sl;
      ur[i] = su;
      sl += lcnt[r0 + i];
      su += ucnt[r0 + i];
      // far-sum slots of the row's work items (one per piece)
      lslot[r0 + i] = ql;
      uslot[r0 + i] = qu;
      ql += far_pieces(lcnt[r0 + i], pl);
      qu += far_pieces(ucnt[r0 + i], pu);
    }
    lr[n] = sl;
    ur[n] = su;
    nslots[b] = max(ql, qu);
    // Piece boundaries of a long row, as offsets e[0..ns] into the row's far
    // entries taken in the order they become computable (L: columns
    // ascending; U: descending).  One piece per kSeg entries by count when
    // the block keeps the default; otherwise by readiness: piece q ends where
    // the readiness coordinate passes (q/ns)^2 of the row's range, so the
    // early pieces are small and available early, and no piece is empty.
    auto cuts = [&](int i, int cnt, int pieces, bool lower, int* e) {
      const int ns = far_pieces(cnt, pieces);
      e[0] = 0;
      e[ns] = cnt;
      if (pieces <= 1) {
        for (int q = 1; q < ns; ++q) e[q] = q * kSeg;
        return ns;
      }
      const uint16_t* col = lower ? pool.lcol + pool.lstart[r0 + i]
                                  : pool.ucol + pool.ustart[r0 + i] + pool.ulen[r0 + i] - cnt;
      auto rho = [&](int k) {  // readiness coordinate of the k-th entry in readiness order
        return lower ? static_cast<int>(col[k]) : ntb * kTile - 1 - static_cast<int>(col[cnt - 1 - k]);
      };
      const long long span = rho(cnt - 1) + 1;
      for (int q = 1; q < ns; ++q) {
        const int thr = static_cast<int>(span * q * q / (ns * ns));
        int lo = 0, hi = cnt;  // first k with rho(k) >= thr
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (rho(mid) >= thr) hi = mid; else lo = mid + 1;
        }
        e[q] = min(max(lo, e[q - 1] + 1), cnt - (ns - q));
      }
      return ns;
    };
    // Work items in solve order (entry offsets within the block).  Long rows:
    // {row, segment, begin, end}, kSeg entries per segment.  Runs of short
    // rows of one tile: one multi-row item (see kShortRow).
    // x = row | first far-sum slot << 16.
    auto build = [&](int4* out, const int* rp, const int* cnt, const int* slot, bool asc,
                     int pieces) {
      int4* o = out;
      int g0 = -1, g1 = -1, gent = 0;  // open group: rows [g0, g1], entries
      auto close = [&]() {
        if (g0 < 0) return;
        const int x = g0 | (slot[r0 + g0] << 16);
        if (g0 == g1)
          *o++ = make_int4(x, 0, rp[g0], rp[g0 + 1]);
        else
          *o++ = make_int4(x, kMultiFlag | (g1 - g0), rp[g0], rp[g1 + 1]);
        g0 = g1 = -1;
        gent = 0;
      };
      for (int k = 0; k < n; ++k) {
        const int i = asc ? k : n - 1 - k;
        const int c = cnt[r0 + i];
        if (c == 0) continue;
        if (c <= kShortRow) {
          const int lo = g0 < 0 ? i : min(g0, i), hi = g0 < 0 ? i : max(g1, i);
          if (g0 >= 0 && ((i >> 5) != (g0 >> 5) || gent + c > kGroupEntries || hi - lo >= 32))
            close();
          if (g0 < 0) {
            g0 = g1 = i;
          } else {
            g0 = min(g0, i);
            g1 = max(g1, i);
          }
          gent += c;
          continue;
        }
        close();
        int e[kMaxSeg + 1];
        const int ns = cuts(i, c, pieces, asc, e);
        for (int q = 0; q < ns; ++q) {
          // U: readiness order runs from the row's last entry backwards
          const int b0 = asc ? rp[i] + e[q] : rp[i] + c - e[q + 1];
          const int b1 = asc ? rp[i] + e[q + 1] : rp[i] + c - e[q];
          *o++ = make_int4(i | ((slot[r0 + i] + q) << 16), q, b0, b1);
        }
      }
      close();
      return static_cast<int>(o - out);
    };
    lnum[b] = build(litems + lioff[b], lr, lcnt, lslot, true, pl);
    unum[b] = build(uitems + uioff[b], ur, ucnt, uslot, false, pu);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned ltmask = (1u << lane) - 1u;
  const long long lb = loff[b], ub = uoff[b];
  const int nt = (n + kTile - 1) / kTile;
  const long long tb = toff[b];
  double* lt = ltile + tb * kTileStride;
  double* ut = utile + tb * kTileStride;
  // Neighbour-window format per tile: ELL width (widest row) or dense.
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    int ml = 0, mu = 0;
    for (int i = t * kTile; i < min(n, (t + 1) * kTile); ++i) {
      ml = max(ml, lnb[r0 + i]);
      mu = max(mu, unb[r0 + i]);
    }
    lwidth[tb + t] = ell_width(ml);
    uwidth[tb + t] = ell_width(mu);
  }
  __syncthreads();
  // Headers: the solver issues near items q = 0 .. 2nt-1 (L tiles ascending,
  // then U tiles descending); item q carries the copy size of item q + kRing.
  auto item_w = [&](int q) { return q < nt ? lwidth[tb + q] : uwidth[tb + 2 * nt - 1 - q]; };
  for (int q = threadIdx.x; q < 2 * nt; q += blockDim.x) {
    double* T = q < nt ? lt + static_cast<long long>(q) * kTileStride
                       : ut + static_cast<long long>(2 * nt - 1 - q) * kTileStride;
    T[kHdr] = __longlong_as_double(item_w(q));
    T[kHdr + 1] = __longlong_as_double(
        q + kRing < 2 * nt ? 8LL * tile_elems(item_w(q + kRing)) : 0LL);
  }
  for (int i = warp; i < nt * kTile; i += blockDim.x / 32) {
    const int t = i >> 5, j = i & 31;
    const bool row = i < n;
    double* ltt = lt + static_cast<long long>(t) * kTileStride;
    double* utt = ut + static_cast<long long>(t) * kTileStride;
    const int wl = lwidth[tb + t], wu = uwidth[tb + t];
    if (lane == 0 && row) {
      const double rd = 1.0 / pool.udiag[r0 + i];
      urdiag[r0 + i] = rd;
      // tile metadata for the solver (see kMetaDiag / kMetaSeg)
      utt[kMetaDiag + j] = rd;
      ltt[kMetaSeg + j] = __longlong_as_double(far_pieces(lcnt[r0 + i], s_pl) |
                                               (static_cast<long long>(lslot[r0 + i]) << 8));
      utt[kMetaSeg + j] = __longlong_as_double(far_pieces(ucnt[r0 + i], s_pu) |
                                               (static_cast<long long>(uslot[r0 + i]) << 8));
    }
    // window padding: every ELL slot past the row's entries reads a solved slot
    if (wl != kDenseNbr)
      for (int e = (row ? lnb[r0 + i] : 0) + lane; e < wl; e += 32)
        reinterpret_cast<unsigned char*>(ltt)[ell_colbyte(j, e)] = kPadColL;
    if (wu != kDenseNbr)
      for (int e = (row ? unb[r0 + i] : 0) + lane; e < wu; e += 32)
        reinterpret_cast<unsigned char*>(utt)[ell_colbyte(j, e)] = kPadColU;
    if (!row) continue;
    {
      const uint32_t ls = pool.lstart[r0 + i];
      const int ll = pool.llen[r0 + i];
      long long w = lb + lr[i];
      int e0 = 0;  // neighbour entries of the row so far
      for (int q0 = 0; q0 < ll; q0 += 32) {
        const int q = q0 + lane;
        const bool in = q < ll;
        const int c = in ? pool.lcol[ls + q] : 0;
        const double v = in ? pool.lval[ls + q] : 0.0;
        const bool far = in && l_far(c, i);
        const bool nbr = in && l_nbr(c, i);
        const unsigned bf = __ballot_sync(0xffffffffu, far);
        const unsigned bn = __ballot_sync(0xffffffffu, nbr);
        const int k = c - (t - (kNearTiles - 1)) * kTile;  // window column 0..95
        if (far) {
          lval[w + __popc(bf & ltmask)] = v;
          lcol[w + __popc(bf & ltmask)] = static_cast<uint16_t>(c);
        } else if (nbr) {
          const int e = e0 + __popc(bn & ltmask);
          if (wl == kDenseNbr) {
            ltt[kNbrOff + k * kTile + j] = v;
          } else {
            ltt[ell_val(wl, j, e)] = v;
            reinterpret_cast<unsigned char*>(ltt)[ell_colbyte(j, e)] = static_cast<unsigned char>(k);
          }
        } else if (in) {
          ltt[kOrigOff + tri_l(j, k - 2 * kTile)] = v;
        }
        w += __popc(bf);
        e0 += __popc(bn);
      }
    }
    {
      const uint32_t us = pool.ustart[r0 + i];
      const int ul = pool.ulen[r0 + i];
      long long w = ub + ur[i];
      int e0 = 0;
      for (int q0 = 0; q0 < ul; q0 += 32) {
        const int q = q0 + lane;
        const bool in = q < ul;
        const int c = in ? pool.ucol[us + q] : 0;
        const double v = in ? pool.uval[us + q] : 0.0;
        const bool far = in && u_far(c, i);
        const bool nbr = in && u_nbr(c, i);
        const unsigned bf = __ballot_sync(0xffffffffu, far);
        const unsigned bn = __ballot_sync(0xffffffffu, nbr);
        const int k = c - t * kTile;  // 0..95
        if (far) {
          uval[w + __popc(bf & ltmask)] = v;
          ucol[w + __popc(bf & ltmask)] = static_cast<uint16_t>(c);
        } else if (nbr) {
          const int e = e0 + __popc(bn & ltmask);
          if (wu == kDenseNbr) {
            utt[kNbrOff + (k - kTile) * kTile + j] = v;
          } else {
            utt[ell_val(wu, j, e)] = v;
            reinterpret_cast<unsigned char*>(utt)[ell_colbyte(j, e)] =
                static_cast<unsigned char>(k - kTile);
          }
        } else if (in) {
          utt[kOrigOff + tri_u(j, k)] = v;
        }
        w += __popc(bf);
        e0 += __popc(bn);
      }
    }
  }
  // Inverses of the diagonal tiles (lane k builds column k by substitution
  // on the tile's own triangle; rows past the block end have U_jj^-1 = 0).
  __syncthreads();
  for (int t = warp; t < nt; t += blockDim.x / 32) {
    // (written by other threads of this CTA above: read through L2)
    const double* lo = lt + static_cast<long long>(t) * kTileStride + kOrigOff;
    const double* uo = ut + static_cast<long long>(t) * kTileStride + kOrigOff;
    double* li = lt + static_cast<long long>(t) * kTileStride + kTriOff;
    double* ui = ut + static_cast<long long>(t) * kTileStride + kTriOff;
    const double* rdg = ut + static_cast<long long>(t) * kTileStride + kMetaDiag;
    const int k = lane;
    {  // column k of L_tt^-1: x_k = 1, x_j = -sum_{k<=m<j} L_jm x_m
      double x[kTile];
#pragma unroll
      for (int q = 0; q < kTile; ++q) x[q] = 0.0;
#pragma unroll
      for (int jr = 0; jr < kTile; ++jr) {
        if (jr < k) continue;
        if (jr == k) {
          x[jr] = 1.0;
          continue;
        }
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < kTile; ++m)
          if (m >= k && m < jr) acc = fma(-__ldcg(lo + tri_l(jr, m)), x[m], acc);
        x[jr] = acc;
        li[tri_l(jr, k)] = acc;
      }
    }
    {  // column k of U_tt^-1: x_k = 1/U_kk, x_j = -(sum_{j<m<=k} U_jm x_m) / U_jj
      double x[kTile];
#pragma unroll
      for (int q = 0; q < kTile; ++q) x[q] = 0.0;
#pragma unroll
      for (int jr = kTile - 1; jr >= 0; --jr) {
        if (jr > k) continue;
        if (jr == k) {
          x[jr] = __ldcg(rdg + k);
          continue;
        }
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < kTile; ++m)
          if (m > jr && m <= k) acc = fma(-__ldcg(uo + tri_u(jr, m)), x[m], acc);
        x[jr] = acc * __ldcg(rdg + jr);
        ui[tri_u(jr, k)] = x[jr];
      }
    }
  }
  // Readiness tile count of every work item (item.y |= need << 8): the solve
  // must have published `need` tiles of its pass before the item's columns
  // are all final.  L: highest column's tile + 1; U: tiles above the lowest.
  __syncthreads();
  for (long long q = lioff[b] + threadIdx.x; q < lioff[b] + lnum[b]; q += blockDim.x) {
    int4 d = litems[q];
    const int r = d.x & 0xffff;
    int c = lcol[lb + d.w - 1];
    if (d.y & kMultiFlag)  // highest column over the group's rows
      for (int i = r; i <= r + (d.y & 0x7f); ++i)
        if (lr[i + 1] > lr[i]) c = max(c, static_cast<int>(lcol[lb + lr[i + 1] - 1]));
    d.y = (d.y & 0xff) | (((c >> 5) + 1) << 8);
    litems[q] = d;
  }
  for (long long q = uioff[b] + threadIdx.x; q < uioff[b] + unum[b]; q += blockDim.x) {
    int4 d = uitems[q];
    const int r = d.x & 0xffff;
    int c = ucol[ub + d.z];
    if (d.y & kMultiFlag)  // lowest column over the group's rows
      for (int i = r; i <= r + (d.y & 0x7f); ++i)
        if (ur[i + 1] > ur[i]) c = min(c, static_cast<int>(ucol[ub + ur[i]]));
    d.y = (d.y & 0xff) | ((nt - (c >> 5)) << 8);
    uitems[q] = d;
  }
  // Workers take items in order of readiness (stable counting sort by need):
  // an item whose inputs are final never waits behind one whose are not, so
  // the far entries of late rows stream while the chain is still early.
  // Each item writes its own far-sum slot, so the sums stay deterministic.
  __syncthreads();
  // With a slack (tiles) the key is max(need, deadline - slack), deadline =
  // the tiles solved before the item's own: an item computable early but due
  // late (U: velocity rows against pressure columns) no longer queues ahead
  // of the items the chain is about to wait for.  need <= key <= deadline - 2,
  // so an item is still computable when the workers reach it in key order
  // whenever the chain has passed its key.
  __shared__ int hist[2][kMaxNeed + 2];
  auto sort_items = [&](int4* items, int4* tmp, int cnt, int* h, bool lower, int slack) {
    auto key = [&](const int4& d) {
      const int need = d.y >> 8;
      if (slack <= 0) return need;
      const int t = (d.x & 0xffff) >> 5;
      return max(need, (lower ? t : nt - 1 - t) - slack);
    };
    for (int k = threadIdx.x; k < kMaxNeed + 2; k += blockDim.x) h[k] = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      tmp[q] = items[q];
      atomicAdd(&h[key(items[q]) + 1], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 1; k < kMaxNeed + 2; ++k) h[k] += h[k - 1];
    __syncthreads();
    if (threadIdx.x == 0)  // stable scatter
      for (int q = 0; q < cnt; ++q) items[h[key(tmp[q])]++] = tmp[q];
    __syncthreads();
  };
  sort_items(litems + lioff[b], ltmp + lioff[b], lnum[b], hist[0], true, slack_l);
  sort_items(uitems + uioff[b], utmp + uioff[b], unum[b], hist[1], false, slack_u);
}

template <class T>
DevBuf upload_vec(const std::vector<T>& h, cudaStream_t s) {
  DevBuf d(sizeof(T) * std::max<size_t>(1, h.size()));
  if (!h.empty()) MSCG_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
  return d;
}

}  // namespace

std::unique_ptr<FactorSet> factor_blocks(Ctx* ctx, const int* a_rp, const int* a_ci,
                                         const double* a_v,
                                         const std::vector<BlockSpec>& blocks,
                                         const std::vector<char>& exact, double tol,
                                         const char* what, FactorTimes* times) {
  using clk = std::chrono::steady_clock;
  cudaStream_t s = ctx->stream;
  auto fs = std::make_unique<FactorSet>();
  const int nb = static_cast<int>(blocks.size());
  fs->nblocks = nb;
  fs->h_row0.resize(nb);
  fs->h_dim.resize(nb);
  fs->h_exact = exact;
  std::vector<int> brow0(nb), bcol0(nb);
  int total = 0, dmax = 0;
  long long in_nnz_est = 0;
  for (int b = 0; b < nb; ++b) {
    if (blocks[b].dim < 1) throw Error(1, std::string("factor: empty ") + what);
    if (blocks[b].dim > 65535)
      throw Error(1, std::string("factor: ") + what + " " + std::to_string(b) +
                         " exceeds 65535 rows (uint16 local columns)");
    fs->h_row0[b] = total;
    fs->h_dim[b] = blocks[b].dim;
    brow0[b] = blocks[b].row0;
    bcol0[b] = blocks[b].col0;
    total += blocks[b].dim;
    dmax = std::max(dmax, blocks[b].dim);
    in_nnz_est += exact[b] ? static_cast<long long>(blocks[b].dim) * blocks[b].dim
                           : 8LL * blocks[b].dim;
  }
  fs->total_rows = total;
  fs->max_dim = dmax;
  fs->has_perm = std::any_of(exact.begin(), exact.end(), [](char e) { return e != 0; });

  DevBuf d_row0 = upload_vec(brow0, s), d_col0 = upload_vec(bcol0, s);
  fs->row0 = upload_vec(fs->h_row0, s);
  fs->dim = upload_vec(fs->h_dim, s);
  std::vector<int> ilut_ids, lu_ids;
  for (int b = 0; b < nb; ++b) (exact[b] ? lu_ids : ilut_ids).push_back(b);
  // largest blocks first, so the last wave holds the smallest (LPT)
  std::stable_sort(ilut_ids.begin(), ilut_ids.end(),
                   [&](int x, int y) { return blocks[x].dim > blocks[y].dim; });
  DevBuf d_ilut_ids = upload_vec(ilut_ids, s), d_lu_ids = upload_vec(lu_ids, s);

  // Per-row pool metadata and per-block totals.
  DevBuf lstart(sizeof(uint32_t) * total), llen(sizeof(int) * total);
  DevBuf ustart(sizeof(uint32_t) * total), ulen(sizeof(int) * total);
  fs->udiag = DevBuf(sizeof(double) * total);
  DevBuf recs(sizeof(longlong2) * total);
  DevBuf nnzl(sizeof(long long) * nb), nnzu(sizeof(long long) * nb);
  DevBuf counters(64);
  if (fs->has_perm) {
    // identity for ILUT blocks; the dense LU overwrites its own rows
    std::vector<int> ident(total);
    for (int b = 0; b < nb; ++b)
      std::iota(ident.begin() + fs->h_row0[b], ident.begin() + fs->h_row0[b] + fs->h_dim[b], 0);
    fs->perm = upload_vec(ident, s);
  }

  // Dense scratch for the exact blocks.
  std::vector<long long> doff(lu_ids.size() + 1, 0);
  for (size_t t = 0; t < lu_ids.size(); ++t)
    doff[t + 1] = doff[t] + static_cast<long long>(blocks[lu_ids[t]].dim) * blocks[lu_ids[t]].dim;
  DevBuf d_doff = upload_vec(doff, s);

  // Pool capacity: generous first guess, doubled on overflow.
  size_t free_b = 0, tot_b = 0;
  MSCG_CUDA(cudaMemGetInfo(&free_b, &tot_b));
  const unsigned long long hard_cap = (1ull << 32) - 1;
  unsigned long long cap = std::max<unsigned long long>(
      4ull * kChunk, static_cast<unsigned long long>(in_nnz_est) * 40ull +
                         static_cast<unsigned long long>(ilut_ids.size() + 2) * kChunk * 2ull);
  cap = std::min(cap, hard_cap);
  const size_t dense_bytes = sizeof(double) * std::max<long long>(1, doff.back());

  int ilut_smem = 0;
  {
    const int words = (dmax + 31) / 32 + 1;
    ilut_smem = dmax * 8 + words * 4 + 32 * 4 + 16;
    ilut_smem = (ilut_smem + 15) & ~15;
  }
  int ilut_grid = 0;
  if (!ilut_ids.empty()) {
    MSCG_CUDA(cudaFuncSetAttribute(ilut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   ilut_smem));
    int per_sm = 0;
    MSCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ilut_kernel, 32, ilut_smem));
    if (per_sm < 1)
      throw Error(1, std::string("factor_ilut: block of ") + std::to_string(dmax) +
                         " rows exceeds the shared-memory working row");
    ilut_grid = std::min<int>(static_cast<int>(ilut_ids.size()), per_sm * ctx->sm_count);
  }

  DevBuf lpool_c, lpool_v, upool_c, upool_v;
  for (int attempt = 0;; ++attempt) {
    MSCG_CUDA(cudaMemGetInfo(&free_b, &tot_b));
    const size_t need = 2 * cap * (sizeof(double) + sizeof(uint16_t)) + dense_bytes;
    if (need + (256ull << 20) > free_b) {
      const unsigned long long fit =
          (free_b > dense_bytes + (512ull << 20))
              ? (free_b - dense_bytes - (512ull << 20)) / (2 * (sizeof(double) + sizeof(uint16_t)))
              : 0;
      if (fit < 4ull * kChunk) throw Error(4, "factor: out of device memory for factor pools");
      cap = std::min(cap, fit);
    }
    lpool_c = DevBuf(cap * sizeof(uint16_t));
    lpool_v = DevBuf(cap * sizeof(double));
    upool_c = DevBuf(cap * sizeof(uint16_t));
    upool_v = DevBuf(cap * sizeof(double));
    DevBuf dense(lu_ids.empty() ? 8 : dense_bytes);
    MSCG_CUDA(cudaMemsetAsync(counters.p, 0, 64, s));
    unsigned long long errinit = ~0ull;
    MSCG_CUDA(cudaMemcpyAsync(counters.as<char>() + 16, &errinit, 8, cudaMemcpyHostToDevice, s));
    PoolView pv;
    pv.lcol = lpool_c.as<uint16_t>();
    pv.lval = lpool_v.as<double>();
    pv.ucol = upool_c.as<uint16_t>();
    pv.uval = upool_v.as<double>();
    pv.lused = reinterpret_cast<unsigned long long*>(counters.as<char>() + 0);
    pv.uused = reinterpret_cast<unsigned long long*>(counters.as<char>() + 8);
    pv.err = reinterpret_cast<unsigned long long*>(counters.as<char>() + 16);
    pv.overflow = reinterpret_cast<int*>(counters.as<char>() + 24);
    int* block_counter = reinterpret_cast<int*>(counters.as<char>() + 28);
    pv.cap = cap;
    pv.lstart = lstart.as<uint32_t>();
    pv.llen = llen.as<int>();
    pv.ustart = ustart.as<uint32_t>();
    pv.ulen = ulen.as<int>();
    pv.udiag = fs->udiag.as<double>();
    pv.blk_nnz_l = nnzl.as<long long>();
    pv.blk_nnz_u = nnzu.as<long long>();

    auto t0 = clk::now();
    if (!ilut_ids.empty()) {
      ilut_kernel<<<ilut_grid, 32, ilut_smem, s>>>(
          static_cast<int>(ilut_ids.size()), d_row0.as<int>(), fs->dim.as<int>(),
          d_col0.as<int>(), fs->row0.as<int>(), d_ilut_ids.as<int>(), a_rp, a_ci, a_v, tol,
          pv, recs.as<longlong2>(), block_counter, dmax);
      MSCG_CUDA(cudaGetLastError());
      ctx->launches++;
    }
    MSCG_CUDA(cudaStreamSynchronize(s));
    auto t1 = clk::now();
    if (!lu_ids.empty()) {
      dense_lu_kernel<<<static_cast<int>(lu_ids.size()), kLuThreads, 0, s>>>(
          d_lu_ids.as<int>(), d_row0.as<int>(), fs->dim.as<int>(), d_col0.as<int>(),
          fs->row0.as<int>(), d_doff.as<long long>(), dense.as<double>(), fs->perm.as<int>(), a_rp,
          a_ci, a_v, pv);
      MSCG_CUDA(cudaGetLastError());
      ctx->launches++;
    }
    unsigned long long hc[4];
    MSCG_CUDA(cudaMemcpyAsync(hc, counters.p, 32, cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaStreamSynchronize(s));
    auto t2 = clk::now();
    if (times) {
      times->ilut_s += std::chrono::duration<double>(t1 - t0).count();
      times->lu_s += std::chrono::duration<double>(t2 - t1).count();
    }
    const int overflow = static_cast<int>(hc[3] & 0xffffffffu);
    if (hc[2] != ~0ull) {
      const int blk = static_cast<int>(hc[2] >> 32), piv = static_cast<int>(hc[2] & 0xffffffffu);
      const bool ex = exact[blk] != 0;
      // what == "" : a standalone factor_ilut / factor_exact call, whose
      // message carries no block prefix (factorization.cpp:113,
      // dense_matrix.cpp:103)
      std::string msg = (what[0] ? std::string(what) + " " + std::to_string(blk) + ": "
                                 : std::string()) +
                        (ex ? "dense_lu" : "factor_ilut") + ": zero pivot at index " +
                        std::to_string(piv);
      throw Error(2, msg, blk, piv);
    }
    if (overflow) {
      if (cap >= hard_cap || attempt >= 4) throw Error(4, "factor: factor pools overflowed");
      cap = std::min(hard_cap, cap * 4);
      continue;
    }
    break;
  }

  // Tiled solve layout (FactorSet, internal.hpp).
  auto t3 = clk::now();
  fs->h_nnz_l.resize(nb);
  fs->h_nnz_u.resize(nb);
  MSCG_CUDA(cudaMemcpyAsync(fs->h_nnz_l.data(), nnzl.p, sizeof(long long) * nb, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaMemcpyAsync(fs->h_nnz_u.data(), nnzu.p, sizeof(long long) * nb, cudaMemcpyDeviceToHost, s));
  PoolView pv{};
  pv.lcol = lpool_c.as<uint16_t>();
  pv.lval = lpool_v.as<double>();
  pv.ucol = upool_c.as<uint16_t>();
  pv.uval = upool_v.as<double>();
  pv.lstart = lstart.as<uint32_t>();
  pv.llen = llen.as<int>();
  pv.ustart = ustart.as<uint32_t>();
  pv.ulen = ulen.as<int>();
  pv.udiag = fs->udiag.as<double>();
  DevBuf lcnt(sizeof(int) * total), ucnt(sizeof(int) * total);
  DevBuf lnb(sizeof(int) * total), unb(sizeof(int) * total);
  DevBuf farl(sizeof(long long) * nb), faru(sizeof(long long) * nb);
  DevBuf itl(sizeof(long long) * nb), itu(sizeof(long long) * nb);
  // Work-item policy of the pack (see pack_tiled_kernel): pieces per long row
  // and the ordering slack, per pass.
  auto env_int = [](const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
  };
  const int pieces_l = std::min(kMaxSeg, std::max(1, env_int("MSCG_PACK_PIECES_L", 1)));
  const int pieces_u = std::min(kMaxSeg, std::max(1, env_int("MSCG_PACK_PIECES_U", 1)));
  const int slack_l = env_int("MSCG_PACK_SLACK_L", 0);
  const int slack_u = env_int("MSCG_PACK_SLACK_U", 8);
  count_far_kernel<<<nb, 256, 0, s>>>(fs->row0.as<int>(), fs->dim.as<int>(), pv, lcnt.as<int>(),
                                      ucnt.as<int>(), lnb.as<int>(), unb.as<int>(),
                                      farl.as<long long>(), faru.as<long long>(),
                                      itl.as<long long>(), itu.as<long long>(), pieces_l,
                                      pieces_u);
  MSCG_CUDA(cudaGetLastError());
  ctx->launches++;
  std::vector<long long> hl(nb), hu(nb), hil(nb), hiu(nb);
  MSCG_CUDA(cudaMemcpyAsync(hl.data(), farl.p, sizeof(long long) * nb, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaMemcpyAsync(hu.data(), faru.p, sizeof(long long) * nb, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaMemcpyAsync(hil.data(), itl.p, sizeof(long long) * nb, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaMemcpyAsync(hiu.data(), itu.p, sizeof(long long) * nb, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  fs->h_loff.assign(nb + 1, 0);
  fs->h_uoff.assign(nb + 1, 0);
  fs->h_toff.assign(nb + 1, 0);
  fs->h_lioff.assign(nb + 1, 0);
  fs->h_uioff.assign(nb + 1, 0);
  for (int b = 0; b < nb; ++b) {
    fs->h_loff[b + 1] = fs->h_loff[b] + hl[b];
    fs->h_uoff[b + 1] = fs->h_uoff[b] + hu[b];
    fs->h_toff[b + 1] = fs->h_toff[b] + (fs->h_dim[b] + kTile - 1) / kTile;
    fs->h_lioff[b + 1] = fs->h_lioff[b] + hil[b];
    fs->h_uioff[b + 1] = fs->h_uioff[b] + hiu[b];
  }
  fs->loff = upload_vec(fs->h_loff, s);
  fs->uoff = upload_vec(fs->h_uoff, s);
  fs->toff = upload_vec(fs->h_toff, s);
  fs->lioff = upload_vec(fs->h_lioff, s);
  fs->uioff = upload_vec(fs->h_uioff, s);
  fs->litems = DevBuf(sizeof(int4) * std::max<long long>(1, fs->h_lioff[nb]));
  fs->uitems = DevBuf(sizeof(int4) * std::max<long long>(1, fs->h_uioff[nb]));
  fs->lnum = DevBuf(sizeof(int) * std::max(1, nb));
  fs->unum = DevBuf(sizeof(int) * std::max(1, nb));
  fs->lrp = DevBuf(sizeof(int) * (total + nb));
  fs->urp = DevBuf(sizeof(int) * (total + nb));
  fs->lval = DevBuf(sizeof(double) * std::max<long long>(1, fs->far_l()));
  fs->lcol = DevBuf(sizeof(uint16_t) * std::max<long long>(1, fs->far_l()));
  fs->uval = DevBuf(sizeof(double) * std::max<long long>(1, fs->far_u()));
  fs->ucol = DevBuf(sizeof(uint16_t) * std::max<long long>(1, fs->far_u()));
  const size_t tile_bytes = sizeof(double) * kTileStride * std::max<long long>(1, fs->tiles());
  fs->ltile = DevBuf(tile_bytes);
  fs->utile = DevBuf(tile_bytes);
  fs->urdiag = DevBuf(sizeof(double) * total);
  fs->lwidth = DevBuf(sizeof(int) * std::max<long long>(1, fs->tiles()));
  fs->uwidth = DevBuf(sizeof(int) * std::max<long long>(1, fs->tiles()));
  fs->lslot = DevBuf(sizeof(int) * std::max(1, total));
  fs->uslot = DevBuf(sizeof(int) * std::max(1, total));
  DevBuf nslots(sizeof(int) * std::max(1, nb));
  DevBuf ltmp(sizeof(int4) * std::max<long long>(1, fs->h_lioff[nb]));
  DevBuf utmp(sizeof(int4) * std::max<long long>(1, fs->h_uioff[nb]));
  MSCG_CUDA(cudaMemsetAsync(fs->ltile.p, 0, tile_bytes, s));
  MSCG_CUDA(cudaMemsetAsync(fs->utile.p, 0, tile_bytes, s));
  pack_tiled_kernel<<<nb, 256, 0, s>>>(
      fs->row0.as<int>(), fs->dim.as<int>(), pv, lcnt.as<int>(), ucnt.as<int>(),
      fs->loff.as<long long>(), fs->uoff.as<long long>(), fs->toff.as<long long>(),
      fs->lrp.as<int>(), fs->urp.as<int>(), fs->lval.as<double>(), fs->lcol.as<uint16_t>(),
      fs->uval.as<double>(), fs->ucol.as<uint16_t>(), fs->ltile.as<double>(),
      fs->utile.as<double>(), fs->urdiag.as<double>(), fs->lioff.as<long long>(),
      fs->uioff.as<long long>(), fs->litems.as<int4>(), fs->uitems.as<int4>(),
      fs->lnum.as<int>(), fs->unum.as<int>(), lnb.as<int>(), unb.as<int>(),
      fs->lwidth.as<int>(), fs->uwidth.as<int>(), fs->lslot.as<int>(), fs->uslot.as<int>(),
      nslots.as<int>(), ltmp.as<int4>(), utmp.as<int4>(), pieces_l, pieces_u, slack_l, slack_u);
  MSCG_CUDA(cudaGetLastError());
  ctx->launches++;
  {
    std::vector<int> hs(std::max(1, nb));
    MSCG_CUDA(cudaMemcpyAsync(hs.data(), nslots.p, sizeof(int) * hs.size(), cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaStreamSynchronize(s));
    fs->max_slots = nb ? *std::max_element(hs.begin(), hs.end()) : 0;
  }
  fs->h_lwidth.resize(fs->tiles());
  fs->h_uwidth.resize(fs->tiles());
  if (fs->tiles()) {
    MSCG_CUDA(cudaMemcpyAsync(fs->h_lwidth.data(), fs->lwidth.p, sizeof(int) * fs->tiles(), cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaMemcpyAsync(fs->h_uwidth.data(), fs->uwidth.p, sizeof(int) * fs->tiles(), cudaMemcpyDeviceToHost, s));
  }
  MSCG_CUDA(cudaStreamSynchronize(s));
  {
    // Launch order for the solve: longest blocks first, so the last wave of
    // CTAs holds the shortest blocks (LPT).  Cost ~ bytes: far entries plus
    // the copied near tiles.
    std::vector<int> ord(nb);
    std::iota(ord.begin(), ord.end(), 0);
    std::vector<long long> tile_cost(nb, 0);
    for (int b = 0; b < nb; ++b)
      for (long long t = fs->h_toff[b]; t < fs->h_toff[b + 1]; ++t)
        tile_cost[b] += tile_elems(fs->h_lwidth[t]) + tile_elems(fs->h_uwidth[t]);
    auto cost = [&](int b) { return 10 * (hl[b] + hu[b]) + 8 * tile_cost[b]; };
    fs->h_chunk.assign(kSolveChunks + 1, 0);
    for (int c = 0; c <= kSolveChunks; ++c)
      fs->h_chunk[c] = static_cast<int>(static_cast<long long>(nb) * c / kSolveChunks);
    auto by_cost = [&](int x, int y) { return cost(x) > cost(y); };
    std::vector<int> whole = ord;
    std::stable_sort(whole.begin(), whole.end(), by_cost);
    fs->order = upload_vec(whole, s);  // one launch over all blocks
    for (int c = 0; c < kSolveChunks; ++c)
      std::stable_sort(ord.begin() + fs->h_chunk[c], ord.begin() + fs->h_chunk[c + 1], by_cost);
    fs->order_chunked = upload_vec(ord, s);  // chunk launches (host-buffer paths)
  }

  if (times) times->pack_s += std::chrono::duration<double>(clk::now() - t3).count();
  return fs;
}

FactorSet::~FactorSet() {
  if (tail_stream) cudaStreamDestroy(tail_stream);
  for (auto e : tail_ev)
    if (e) cudaEventDestroy(e);
}

int64_t FactorSet::nnz_l() const {
  int64_t s = 0;
  for (auto v : h_nnz_l) s += v;
  return s;
}
int64_t FactorSet::nnz_u() const {
  int64_t s = 0;
  for (auto v : h_nnz_u) s += v;
  return s;
}

// Reference layout from the tiled layout: L row = far entries (columns <
// 32(t-2)) then the nonzeros of the near window; U row = diagonal, near
// nonzeros, then far entries (columns >= 32(t+3)).
void download_factor(const FactorSet& fs, int idx, std::vector<int>& lrp,
                     std::vector<int>& lci, std::vector<double>& lv,
                     std::vector<int>& urp, std::vector<int>& uci,
                     std::vector<double>& uv, std::vector<int>& perm) {
  const int n = fs.h_dim[idx], r0 = fs.h_row0[idx];
  const long long lb = fs.h_loff[idx], le = fs.h_loff[idx + 1];
  const long long ub = fs.h_uoff[idx], ue = fs.h_uoff[idx + 1];
  const long long t0 = fs.h_toff[idx], nt = fs.h_toff[idx + 1] - t0;
  const size_t tsz = kTileStride;
  std::vector<int> hlr(n + 1), hur(n + 1);
  std::vector<uint16_t> hlc(le - lb), huc(ue - ub);
  std::vector<double> hlv(le - lb), huv(ue - ub), hd(n), hlt(tsz * nt), hut(tsz * nt);
  MSCG_CUDA(cudaMemcpy(hlr.data(), fs.lrp.as<int>() + r0 + idx, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost));
  MSCG_CUDA(cudaMemcpy(hur.data(), fs.urp.as<int>() + r0 + idx, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost));
  if (le > lb) {
    MSCG_CUDA(cudaMemcpy(hlc.data(), fs.lcol.as<uint16_t>() + lb, sizeof(uint16_t) * (le - lb), cudaMemcpyDeviceToHost));
    MSCG_CUDA(cudaMemcpy(hlv.data(), fs.lval.as<double>() + lb, sizeof(double) * (le - lb), cudaMemcpyDeviceToHost));
  }
  if (ue > ub) {
    MSCG_CUDA(cudaMemcpy(huc.data(), fs.ucol.as<uint16_t>() + ub, sizeof(uint16_t) * (ue - ub), cudaMemcpyDeviceToHost));
    MSCG_CUDA(cudaMemcpy(huv.data(), fs.uval.as<double>() + ub, sizeof(double) * (ue - ub), cudaMemcpyDeviceToHost));
  }
  MSCG_CUDA(cudaMemcpy(hlt.data(), fs.ltile.as<double>() + t0 * tsz, sizeof(double) * tsz * nt, cudaMemcpyDeviceToHost));
  MSCG_CUDA(cudaMemcpy(hut.data(), fs.utile.as<double>() + t0 * tsz, sizeof(double) * tsz * nt, cudaMemcpyDeviceToHost));
  MSCG_CUDA(cudaMemcpy(hd.data(), fs.udiag.as<double>() + r0, sizeof(double) * n, cudaMemcpyDeviceToHost));
  perm.resize(n);
  if (fs.has_perm && fs.h_exact[idx]) {
    MSCG_CUDA(cudaMemcpy(perm.data(), fs.perm.as<int>() + r0, sizeof(int) * n, cudaMemcpyDeviceToHost));
  } else {
    std::iota(perm.begin(), perm.end(), 0);
  }
  lrp.assign(n + 1, 0);
  urp.assign(n + 1, 0);
  lci.clear();
  lv.clear();
  uci.clear();
  uv.clear();
  for (int i = 0; i < n; ++i) {
    const int t = i / kTile, j = i % kTile;
    for (int k = hlr[i]; k < hlr[i + 1]; ++k) {
      lci.push_back(hlc[k]);
      lv.push_back(hlv[k]);
    }
    // near window in ascending column order: neighbour tiles, then the
    // diagonal tile (absent entries are zeros; stored values never are)
    auto nbr_entries = [&](const double* T, int w, int j, auto&& emit) {
      if (w == kDenseNbr) {
        for (int k = 0; k < 2 * kTile; ++k) emit(k, T[kNbrOff + k * kTile + j]);
      } else {
        const unsigned char* cb = reinterpret_cast<const unsigned char*>(T);
        for (int e = 0; e < w; ++e) emit(cb[ell_colbyte(j, e)], T[ell_val(w, j, e)]);
      }
    };
    const double* LT = &hlt[t * tsz];
    const double* UT = &hut[t * tsz];
    nbr_entries(LT, fs.h_lwidth[t0 + t], j, [&](int k, double v) {
      const int c = (t - (kNearTiles - 1)) * kTile + k;
      if (c >= 0 && v != 0.0) {
        lci.push_back(c);
        lv.push_back(v);
      }
    });
    for (int k = 0; k < j; ++k) {
      const double v = LT[kOrigOff + tri_l(j, k)];
      if (v != 0.0) {
        lci.push_back(t * kTile + k);
        lv.push_back(v);
      }
    }
    lrp[i + 1] = static_cast<int>(lci.size());
    uci.push_back(i);
    uv.push_back(hd[i]);
    for (int k = j + 1; k < kTile; ++k) {
      const double v = UT[kOrigOff + tri_u(j, k)];
      if (t * kTile + k < n && v != 0.0) {
        uci.push_back(t * kTile + k);
        uv.push_back(v);
      }
    }
    nbr_entries(UT, fs.h_uwidth[t0 + t], j, [&](int k, double v) {
      const int c = (t + 1) * kTile + k;
      if (c < n && v != 0.0) {
        uci.push_back(c);
        uv.push_back(v);
      }
    });
    for (int k = hur[i]; k < hur[i + 1]; ++k) {
      uci.push_back(huc[k]);
      uv.push_back(huv[k]);
    }
    urp[i + 1] = static_cast<int>(uci.size());
  }
}

}  // namespace mscg
