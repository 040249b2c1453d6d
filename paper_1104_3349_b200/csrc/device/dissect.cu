// Nested dissection on the device (reference nested_dissection / dissect /
// bisect / pseudo_peripheral / bfs_levels, proj/src/graph.cpp:70-230; SURVEY
// 8(f) row 2).  The result — blocks in depth-first leaf order, each sorted,
// and the sorted separator — is the reference's, node for node.
//
// The dissection tree is expanded level by level; every piece of a level is
// bisected at once.  A bisection is three breadth-first searches restricted
// to the piece: from its first minimum-degree node (first component only),
// from the last node that search visits, and — from the smaller of the two
// pseudo-peripheral ends — a full search that restarts at the smallest
// unvisited node whenever a component is exhausted.  The reference's cut
// (half the nodes, extended to the end of the level) only needs, per piece,
// the round in which the search passes node size/2, so the third search keeps
// no order, just each node's round.
//
// The FIFO order of a search is reproduced level-synchronously: a frontier
// entry's virtual index e (pieces' frontiers concatenated in piece order,
// each in visit order) is the discovery key; a node is discovered by the
// smallest e that reaches it (atomicMin), and the next frontier is written in
// (e, adjacency position) order — exactly the order a FIFO queue appends
// nodes.  Each piece's frontier lives in its own region of the frontier
// buffers ([pstart[k], pstart[k] + size)), so pieces restart components and
// finish independently.  One round = 6 kernels with fixed grids (no host
// synchronisation); the host polls the frontier total every kPoll rounds.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

constexpr int kT = 256;
constexpr int kPoll = 8;

struct Level {
  int n;
  int K;                  // pieces at this level
  const long long* off;   // graph CSR
  const int* adj;
  const int* piece;       // node -> piece (-1: separator)
  const int* plist;       // nodes sorted by (piece, id)
  const int* pstart;      // [K+1] piece ranges in plist (and frontier regions)
  const int* active;      // [K] piece is bisected at this level
  int* dist;              // node -> round visited (-1: not yet)
  int* disc;              // node -> discovering virtual entry
  int* fcnt;              // [K] current frontier size
  int* vpre;              // [K+1] exclusive prefix of fcnt (vpre[K] = total)
  int* offs;              // per virtual entry: exclusive offset within its CTA chunk
  int* btot;              // [G+1] CTA chunk totals, then their exclusive prefix
  int* fend;              // [K] last node of the search (modes 0/1)
  int* cursor;            // [K] plist cursor for component restarts (mode 2)
  int* cum;               // [K] nodes visited before this round (mode 2)
  int* cutround;          // [K] round holding node size/2 (mode 2)
  int* include;           // [K] that round belongs to the left half
  int* restart;           // [K] the piece's component is exhausted (mode 2)
};

// Virtual entry e -> piece, by binary search in the staged prefix.
__device__ __forceinline__ int find_piece(const int* vp, int K, int e) {
  int lo = 0, hi = K;  // vp[lo] <= e < vp[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (vp[mid] <= e)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Stage vpre in shared memory when it fits (pieces <= 8191).
constexpr int kStageMax = 8192;

__device__ __forceinline__ const int* stage_vpre(const Level& L, int* sm) {
  if (L.K + 1 > kStageMax) return L.vpre;
  for (int i = threadIdx.x; i <= L.K; i += blockDim.x) sm[i] = L.vpre[i];
  __syncthreads();
  return sm;
}

__global__ void vprefix_kernel(Level L) {
  // one CTA: exclusive scan of fcnt over the pieces
  __shared__ int carry;
  __shared__ int wsum[kT / 32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < L.K; base += kT) {
    const int k = base + threadIdx.x;
    const int v = k < L.K ? L.fcnt[k] : 0;
    int x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int wpre = 0;
    for (int i = 0; i < w; ++i) wpre += wsum[i];
    int tot = 0;
    for (int i = 0; i < kT / 32; ++i) tot += wsum[i];
    if (k < L.K) L.vpre[k] = carry + wpre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) L.vpre[L.K] = carry;
}

// (b) discovery: the smallest virtual entry reaching each unvisited node
__global__ void __launch_bounds__(kT) expand_kernel(Level L, const int* cur) {
  __shared__ int svp[kStageMax];
  const int* vp = stage_vpre(L, svp);
  const int total = vp[L.K];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int k = find_piece(vp, L.K, e);
    const int u = cur[L.pstart[k] + (e - vp[k])];
    for (long long a = L.off[u]; a < L.off[u + 1]; ++a) {
      const int v = L.adj[a];
      if (L.piece[v] == k && L.dist[v] < 0) atomicMin(&L.disc[v], e);
    }
  }
}

__device__ __forceinline__ int chunk_of(int total) {
  return (total + gridDim.x - 1) / gridDim.x;
}

// (c) per entry: how many nodes it discovered; exclusive offsets inside the
// CTA's contiguous chunk of entries
__global__ void __launch_bounds__(kT) count_kernel(Level L, const int* cur) {
  __shared__ int svp[kStageMax];
  __shared__ int wsum[kT / 32];
  __shared__ int carry;
  const int* vp = stage_vpre(L, svp);
  const int total = vp[L.K];
  const int chunk = chunk_of(total);
  const int e0 = min(total, blockIdx.x * chunk), e1 = min(total, e0 + chunk);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = e0; base < e1; base += kT) {
    const int e = base + threadIdx.x;
    int c = 0;
    if (e < e1) {
      const int k = find_piece(vp, L.K, e);
      const int u = cur[L.pstart[k] + (e - vp[k])];
      for (long long a = L.off[u]; a < L.off[u + 1]; ++a) {
        const int v = L.adj[a];
        c += (L.piece[v] == k && L.dist[v] < 0 && L.disc[v] == e);
      }
    }
    int x = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int i = 0; i < kT / 32; ++i) {
      if (i < w) wpre += wsum[i];
      tot += wsum[i];
    }
    if (e < e1) L.offs[e] = carry + wpre + x - c;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) L.btot[blockIdx.x] = carry;
}

// (d) exclusive prefix of the CTA chunk totals (one CTA; G + 1 entries)
__global__ void chunk_prefix_kernel(int* btot, int G) {
  if (threadIdx.x == 0) {
    int s = 0;
    for (int b = 0; b < G; ++b) {
      const int t = btot[b];
      btot[b] = s;
      s += t;
    }
    btot[G] = s;
  }
}

__device__ __forceinline__ int goff(const Level& L, int e, int total, int chunk) {
  return e >= total ? L.btot[gridDim.x] : L.btot[e / chunk] + L.offs[e];
}

// (e) the next frontier, in (entry, adjacency) order, into each piece's region
__global__ void __launch_bounds__(kT) write_kernel(Level L, const int* cur, int* nxt, int round) {
  __shared__ int svp[kStageMax];
  const int* vp = stage_vpre(L, svp);
  const int total = vp[L.K];
  const int chunk = chunk_of(total);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int k = find_piece(vp, L.K, e);
    const int u = cur[L.pstart[k] + (e - vp[k])];
    int pos = L.pstart[k] + goff(L, e, total, chunk) - goff(L, vp[k], total, chunk);
    for (long long a = L.off[u]; a < L.off[u + 1]; ++a) {
      const int v = L.adj[a];
      if (L.piece[v] == k && L.dist[v] < 0 && L.disc[v] == e) {
        nxt[pos++] = v;
        L.dist[v] = round + 1;
      }
    }
  }
}

// (f) per piece: the cut round (mode 2), the new frontier size, the end of
// a first-component search (modes 0/1) or a component restart (mode 2)
__global__ void bookkeep_kernel(Level L, const int* cur, int round, int mode, int G) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L.K) return;
  const int fc = L.fcnt[k];
  if (fc == 0) return;
  const int total = L.vpre[L.K];
  const int chunk = (total + G - 1) / G;  // the count / write kernels' chunking
  auto g = [&](int e) { return e >= total ? L.btot[G] : L.btot[e / chunk] + L.offs[e]; };
  const int nc = g(L.vpre[k + 1]) - g(L.vpre[k]);
  if (mode == 2) {
    const int half = (L.pstart[k + 1] - L.pstart[k]) / 2;
    const int c0 = L.cum[k];
    if (L.cutround[k] < 0 && half < c0 + fc) {
      L.cutround[k] = round;
      L.include[k] = half > c0;
    }
    L.cum[k] = c0 + fc;
  }
  if (nc == 0) {
    // restart only while unvisited nodes remain (cum counts every visited node)
    if (mode == 2)
      L.restart[k] = L.cum[k] < L.pstart[k + 1] - L.pstart[k];
    else
      L.fend[k] = cur[L.pstart[k] + fc - 1];
  }
  L.fcnt[k] = nc;
}

// (g) mode 2: a piece whose component is exhausted restarts at its smallest
// unvisited node (one warp per piece scans its sorted node list)
__global__ void restart_kernel(Level L, int* nxt, int round) {
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= L.K || !L.restart[k]) return;
  const int end = L.pstart[k + 1];
  int c = L.cursor[k];
  int found = -1;
  while (c < end) {
    const int i = c + lane;
    const bool un = i < end && L.dist[L.plist[i]] < 0;
    const unsigned b = __ballot_sync(0xffffffffu, un);
    if (b) {
      found = c + __ffs(b) - 1;
      break;
    }
    c += 32;
  }
  if (lane == 0) {
    L.restart[k] = 0;
    if (found >= 0) {
      const int u = L.plist[found];
      nxt[L.pstart[k]] = u;
      L.dist[u] = round + 1;
      L.fcnt[k] = 1;
      L.cursor[k] = found + 1;
    } else {
      L.cursor[k] = end;
    }
  }
}

// ---- one breadth-first search per launch: a persistent cooperative kernel.
// Every round runs the phases above separated by grid-wide barriers; the
// piece prefix and the chunk prefix are recomputed by every CTA in shared
// memory, so a round costs four barriers and no host round trip.
namespace cg = cooperative_groups;

// exclusive block scan of src[0:cnt) into dst[0:cnt], dst[cnt] = total
__device__ void block_scan(const int* src, int cnt, int* dst) {
  __shared__ int wsum[kT / 32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < cnt; base += kT) {
    const int i = base + threadIdx.x;
    const int v = i < cnt ? src[i] : 0;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int q = 0; q < kT / 32; ++q) {
      if (q < w) wpre += wsum[q];
      tot += wsum[q];
    }
    if (i < cnt) dst[i] = carry + wpre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) dst[cnt] = carry;
  __syncthreads();
}

constexpr int kCoopMaxG = 1024;

// A frontier entry's neighbours are handled by a group of kLanes lanes (one
// neighbour each, the enriched graph's degree is ~8-16), so a round's
// dependent loads are a few latencies, not one per neighbour.
constexpr int kLanes = 16;

__global__ void __launch_bounds__(kT) bfs_coop_kernel(Level L, int* fa, int* fb, int mode) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int svp[kStageMax];
  __shared__ int sbt[kCoopMaxG + 1];
  __shared__ int cs[kT / kLanes];
  __shared__ int carry;
  const int G = gridDim.x;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = G * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int sub = threadIdx.x % kLanes;                 // lane within the entry's group
  const int grp = threadIdx.x / kLanes;                 // group within the CTA
  const unsigned gmask = 0xffffu << (lane & 16);        // the group's lanes in the warp
  const int ggroups = gthreads / kLanes, ggid = gtid / kLanes;
  int* cur = fa;
  int* nxt = fb;
  for (int round = 0;; ++round) {
    // A: piece prefix of the frontier sizes (every CTA, shared memory)
    block_scan(L.fcnt, L.K, svp);
    const int total = svp[L.K];
    if (total == 0) break;  // uniform: every CTA read the same fcnt
    // B: discovery, one neighbour per lane
    for (int e = ggid; e < total; e += ggroups) {
      const int k = find_piece(svp, L.K, e);
      const int u = cur[L.pstart[k] + (e - svp[k])];
      const long long a1 = L.off[u + 1];
      for (long long a = L.off[u] + sub; a < a1; a += kLanes) {
        const int v = L.adj[a];
        if (L.piece[v] == k && L.dist[v] < 0) atomicMin(&L.disc[v], e);
      }
    }
    grid.sync();
    // C: per entry counts, offsets inside the CTA's chunk
    const int chunk = (total + G - 1) / G;
    const int e0 = min(total, blockIdx.x * chunk), e1 = min(total, e0 + chunk);
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = e0; base < e1; base += kT / kLanes) {
      const int e = base + grp;
      int c = 0;
      if (e < e1) {
        const int k = find_piece(svp, L.K, e);
        const int u = cur[L.pstart[k] + (e - svp[k])];
        const long long a1 = L.off[u + 1];
        for (long long a = L.off[u] + sub; a < a1; a += kLanes) {
          const int v = L.adj[a];
          c += (L.piece[v] == k && L.dist[v] < 0 && L.disc[v] == e);
        }
      }
      for (int o = kLanes / 2; o; o >>= 1) c += __shfl_xor_sync(gmask, c, o);
      if (sub == 0) cs[grp] = c;
      __syncthreads();
      if (sub == 0 && e < e1) {
        int pre = 0;
        for (int q = 0; q < grp; ++q) pre += cs[q];
        L.offs[e] = carry + pre;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int q = 0; q < kT / kLanes; ++q) t += cs[q];
        carry += t;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) L.btot[blockIdx.x] = carry;
    grid.sync();
    // D: chunk prefix (every CTA), E: the next frontier in (entry,
    // adjacency) order: a lane's slot = the flagged lanes before it
    block_scan(L.btot, G, sbt);
    auto g = [&](int e) { return e >= total ? sbt[G] : sbt[e / chunk] + L.offs[e]; };
    for (int e = ggid; e < total; e += ggroups) {
      const int k = find_piece(svp, L.K, e);
      const int u = cur[L.pstart[k] + (e - svp[k])];
      int pos = L.pstart[k] + g(e) - g(svp[k]);
      const long long a0 = L.off[u], a1 = L.off[u + 1];
      for (long long a = a0; a < a1; a += kLanes) {
        const long long my = a + sub;
        int v = -1;
        bool f = false;
        if (my < a1) {
          v = L.adj[my];
          f = L.piece[v] == k && L.dist[v] < 0 && L.disc[v] == e;
        }
        const unsigned b = __ballot_sync(gmask, f) & gmask;
        if (f) {
          const unsigned below = b & ((1u << lane) - 1u);
          nxt[pos + __popc(below)] = v;
          L.dist[v] = round + 1;
        }
        pos += __popc(b);
      }
    }
    // F: per piece bookkeeping (reads only this round's offsets)
    for (int k = gtid; k < L.K; k += gthreads) {
      const int fc = L.fcnt[k];
      if (fc == 0) continue;
      const int nc = g(svp[k + 1]) - g(svp[k]);
      const int size = L.pstart[k + 1] - L.pstart[k];
      if (mode == 2) {
        const int half = size / 2;
        const int c0 = L.cum[k];
        if (L.cutround[k] < 0 && half < c0 + fc) {
          L.cutround[k] = round;
          L.include[k] = half > c0;
        }
        L.cum[k] = c0 + fc;
      }
      if (nc == 0) {
        if (mode == 2)
          L.restart[k] = L.cum[k] < size;
        else
          L.fend[k] = cur[L.pstart[k] + fc - 1];
      }
      L.fcnt[k] = nc;
    }
    grid.sync();
    // G: component restarts (mode 2), one warp per piece
    if (mode == 2) {
      const int gw = gtid >> 5, nw = gthreads >> 5;
      for (int k = gw; k < L.K; k += nw) {
        if (!L.restart[k]) continue;
        const int end = L.pstart[k + 1];
        int c = L.cursor[k];
        int found = -1;
        while (c < end) {
          const int i = c + lane;
          const bool un = i < end && L.dist[L.plist[i]] < 0;
          const unsigned bb = __ballot_sync(0xffffffffu, un);
          if (bb) {
            found = c + __ffs(bb) - 1;
            break;
          }
          c += 32;
        }
        if (lane == 0) {
          L.restart[k] = 0;
          if (found >= 0) {
            const int u = L.plist[found];
            nxt[L.pstart[k]] = u;
            L.dist[u] = round + 1;
            L.fcnt[k] = 1;
            L.cursor[k] = found + 1;
          } else {
            L.cursor[k] = end;
          }
        }
        __syncwarp();
      }
      grid.sync();
    }
    int* t = cur;
    cur = nxt;
    nxt = t;
  }
}

// per BFS: reset the visit state of the active pieces' nodes and seed src[k]
__global__ void bfs_reset_kernel(Level L) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < L.n; u += gridDim.x * blockDim.x) {
    const int k = L.piece[u];
    if (k >= 0 && L.active[k]) {
      L.dist[u] = -1;
      L.disc[u] = INT_MAX;
    }
  }
}
__global__ void bfs_seed_kernel(Level L, const int* src, int* cur, int mode) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L.K) return;
  L.restart[k] = 0;
  if (!L.active[k]) {
    L.fcnt[k] = 0;
    return;
  }
  const int s = src[k];
  cur[L.pstart[k]] = s;
  L.dist[s] = 0;
  L.fcnt[k] = 1;
  L.fend[k] = s;
  if (mode == 2) {
    L.cursor[k] = L.pstart[k];
    L.cum[k] = 0;
    L.cutround[k] = -1;
    L.include[k] = 0;
  }
}

// first minimum-degree node of each active piece (pseudo_peripheral's start)
__global__ void start_kernel(const int* piece, const int* active, const long long* off, int n,
                             unsigned long long* best) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    const int k = piece[u];
    if (k < 0 || !active[k]) continue;
    const unsigned long long key =
        (static_cast<unsigned long long>(off[u + 1] - off[u]) << 32) | static_cast<unsigned>(u);
    atomicMin(&best[k], key);
  }
}
__global__ void start_unpack_kernel(const unsigned long long* best, int K, int* src) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < K) src[k] = static_cast<int>(best[k] & 0xffffffffull);
}
__global__ void origin_kernel(const int* f1, const int* f2, int K, int* src) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < K) src[k] = min(f1[k], f2[k]);
}

// left (1) / right (0) by the cut round, then the separator (2): right nodes
// with a left neighbour in the same piece (bisect, graph.cpp:147-170)
__global__ void label_kernel(Level L, char* lab) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < L.n; u += gridDim.x * blockDim.x) {
    const int k = L.piece[u];
    if (k < 0 || !L.active[k]) continue;
    const int r = L.dist[u], cr = L.cutround[k];
    lab[u] = (r < cr || (r == cr && L.include[k])) ? 1 : 0;
  }
}
__global__ void separator_kernel(Level L, char* lab, int* counts) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < L.n; u += gridDim.x * blockDim.x) {
    const int k = L.piece[u];
    if (k < 0 || !L.active[k]) continue;
    if (lab[u] == 1) {
      atomicAdd(&counts[3 * k], 1);
      continue;
    }
    bool sep = false;
    for (long long a = L.off[u]; a < L.off[u + 1] && !sep; ++a) {
      const int v = L.adj[a];
      sep = L.piece[v] == k && lab[v] == 1;
    }
    if (sep) {
      lab[u] = 2;
      atomicAdd(&counts[3 * k + 2], 1);
    } else {
      atomicAdd(&counts[3 * k + 1], 1);
    }
  }
}
// next level's piece ids: a split piece's left half -> child base, right ->
// base + 1, separator -> -1; leaves and degenerate splits keep one child
__global__ void relabel_kernel(int n, int* piece, const char* lab, const int* active,
                               const int* split, const int* base) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    const int k = piece[u];
    if (k < 0) continue;
    if (!active[k] || !split[k]) {
      piece[u] = base[k];
      continue;
    }
    const char l = lab[u];
    piece[u] = l == 1 ? base[k] : l == 0 ? base[k] + 1 : -1;
  }
}

__global__ void iota_kernel(int n, int* a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}
// sort keys: piece id, separator last
__global__ void sortkey_kernel(int n, const int* piece, unsigned* key, unsigned sep_key) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    key[i] = piece[i] < 0 ? sep_key : static_cast<unsigned>(piece[i]);
}
// piece ranges in the sorted list
__global__ void bounds_kernel(int n, const unsigned* skey, int K, int* pstart) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned k = skey[i];
    const unsigned prev = i == 0 ? 0xffffffffu : skey[i - 1];
    if (k != prev) {
      // every key between prev + 1 and k starts here (empty pieces: none)
      const unsigned lo = i == 0 ? 0u : prev + 1;
      for (unsigned q = lo; q <= k && q <= static_cast<unsigned>(K); ++q) pstart[q] = i;
    }
    if (i == n - 1)
      for (unsigned q = k + 1; q <= static_cast<unsigned>(K); ++q) pstart[q] = n;
  }
}

// a borrowed device array with DevBuf's accessor
struct Borrowed {
  const void* p;
  template <class T> T* as() const { return static_cast<T*>(const_cast<void*>(p)); }
};

}  // namespace

// Core on device arrays: piece (n ints, out) = final piece id of every node
// in depth-first leaf order, -1 for the separator; returns the piece count.
int nested_dissection_core(Ctx* ctx, int n, const long long* d_off_p, const int* d_adj_p,
                           int target_blocks, int* piece_out) {
  cudaStream_t s = ctx->stream;
  if (target_blocks < 1 || target_blocks > std::max(n, 1))
    throw Error(1, "nested_dissection: target_blocks out of range");
  MSCG_CUDA(cudaMemsetAsync(piece_out, 0, sizeof(int) * std::max(n, 1), s));
  if (target_blocks == 1 || n <= 1) return 1;
  int depth = 0;
  while ((1 << depth) < target_blocks) ++depth;
  static const bool verbose = getenv("MSCG_VERBOSE") != nullptr;
  using clk = std::chrono::steady_clock;
  auto tl = clk::now();
  const Borrowed d_off{d_off_p}, d_adj{d_adj_p};
  const Borrowed piece{piece_out};
  DevBuf dist(sizeof(int) * n), disc(sizeof(int) * n),
      fa(sizeof(int) * n), fb(sizeof(int) * n), offs(sizeof(int) * n), lab(n),
      plist(sizeof(int) * n), ids(sizeof(int) * n), key(sizeof(unsigned) * n),
      skey(sizeof(unsigned) * n);
  const int G = 2 * ctx->sm_count;  // entry-chunk grid of the round kernels
  // the cooperative search: as many CTAs as are co-resident (<= kCoopMaxG)
  int Gc = 0;
  {
    int per_sm = 0, coop = 0, dev = 0;
    MSCG_CUDA(cudaGetDevice(&dev));
    MSCG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    MSCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_coop_kernel, kT, 0));
    static const bool no_coop = getenv("MSCG_ND_NOCOOP") != nullptr;
    if (coop && per_sm > 0 && !no_coop) Gc = std::min(kCoopMaxG, std::min(per_sm, 2) * ctx->sm_count);
  }
  const int Gn = 4 * ctx->sm_count; // node-sweep grid
  DevBuf btot(sizeof(int) * (G + 1));
  // cub sort workspace
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key.as<unsigned>(), skey.as<unsigned>(),
                                  ids.as<int>(), plist.as<int>(), n, 0, 32, s);
  DevBuf sort_tmp(std::max<size_t>(sort_bytes, 16));
  int K = 1;
  std::vector<int> h_active(1, 1), h_sizes(1, n);
  // sort nodes by piece (stable: ascending ids within a piece), separator last
  auto sort_by_piece = [&](int K_, int* d_pstart) {
    // key = piece id, separator = K_ (after every piece)
    sortkey_kernel<<<Gn, kT, 0, s>>>(n, piece.as<int>(), key.as<unsigned>(),
                                     static_cast<unsigned>(K_));
    iota_kernel<<<Gn, kT, 0, s>>>(n, ids.as<int>());
    int bits = 1;
    while ((1u << bits) <= static_cast<unsigned>(K_)) ++bits;
    size_t sb = sort_tmp.bytes;
    MSCG_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, sb, key.as<unsigned>(),
                                              skey.as<unsigned>(), ids.as<int>(),
                                              plist.as<int>(), n, 0, bits, s));
    if (d_pstart) bounds_kernel<<<Gn, kT, 0, s>>>(n, skey.as<unsigned>(), K_, d_pstart);
    ctx->launches += 3;
  };
  long long total_rounds = 0;
  for (int d = 0; d < depth; ++d) {
    DevBuf pstart(sizeof(int) * (K + 1)), active(sizeof(int) * K), fcnt(sizeof(int) * K),
        vpre(sizeof(int) * (K + 1)), fend(sizeof(int) * K), f1(sizeof(int) * K),
        src(sizeof(int) * K), cursor(sizeof(int) * K), cum(sizeof(int) * K),
        cutround(sizeof(int) * K), include(sizeof(int) * K), restart(sizeof(int) * K),
        best(sizeof(unsigned long long) * K), counts(sizeof(int) * 3 * K), split(sizeof(int) * K),
        base(sizeof(int) * K);
    // pieces of size <= 1 are leaves (dissect, graph.cpp:183-186)
    bool any = false;
    for (int k = 0; k < K; ++k) {
      if (h_sizes[k] <= 1) h_active[k] = 0;
      any = any || h_active[k];
    }
    if (!any) break;
    MSCG_CUDA(cudaMemcpyAsync(active.p, h_active.data(), sizeof(int) * K, cudaMemcpyHostToDevice, s));
    sort_by_piece(K, pstart.as<int>());
    Level L;
    L.n = n;
    L.K = K;
    L.off = d_off.as<long long>();
    L.adj = d_adj.as<int>();
    L.piece = piece.as<int>();
    L.plist = plist.as<int>();
    L.pstart = pstart.as<int>();
    L.active = active.as<int>();
    L.dist = dist.as<int>();
    L.disc = disc.as<int>();
    L.fcnt = fcnt.as<int>();
    L.vpre = vpre.as<int>();
    L.offs = offs.as<int>();
    L.btot = btot.as<int>();
    L.fend = fend.as<int>();
    L.cursor = cursor.as<int>();
    L.cum = cum.as<int>();
    L.cutround = cutround.as<int>();
    L.include = include.as<int>();
    L.restart = restart.as<int>();
    const int Kb = (K + kT - 1) / kT;
    // start: first minimum-degree node of each piece
    MSCG_CUDA(cudaMemsetAsync(best.p, 0xff, best.bytes, s));
    start_kernel<<<Gn, kT, 0, s>>>(piece.as<int>(), active.as<int>(), d_off.as<long long>(), n,
                                   best.as<unsigned long long>());
    start_unpack_kernel<<<Kb, kT, 0, s>>>(best.as<unsigned long long>(), K, src.as<int>());
    ctx->launches += 2;
    auto bfs = [&](int mode) {
      int* cur = fa.as<int>();
      int* nxt = fb.as<int>();
      bfs_reset_kernel<<<Gn, kT, 0, s>>>(L);
      bfs_seed_kernel<<<Kb, kT, 0, s>>>(L, src.as<int>(), cur, mode);
      ctx->launches += 2;
      if (Gc > 0 && K + 1 <= kStageMax) {
        int md = mode;
        void* args[] = {&L, &cur, &nxt, &md};
        MSCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bfs_coop_kernel), Gc, kT,
                                              args, 0, s));
        ctx->launches++;
        return;
      }
      int round = 0;
      for (;;) {
        for (int r = 0; r < kPoll; ++r, ++round) {
          vprefix_kernel<<<1, kT, 0, s>>>(L);
          expand_kernel<<<G, kT, 0, s>>>(L, cur);
          count_kernel<<<G, kT, 0, s>>>(L, cur);
          chunk_prefix_kernel<<<1, 32, 0, s>>>(L.btot, G);
          write_kernel<<<G, kT, 0, s>>>(L, cur, nxt, round);
          bookkeep_kernel<<<Kb, kT, 0, s>>>(L, cur, round, mode, G);
          ctx->launches += 6;
          if (mode == 2) {
            restart_kernel<<<(K * 32 + kT - 1) / kT, kT, 0, s>>>(L, nxt, round);
            ctx->launches++;
          }
          std::swap(cur, nxt);
        }
        // frontier total after the last round
        vprefix_kernel<<<1, kT, 0, s>>>(L);
        int tot = 0;
        MSCG_CUDA(cudaMemcpyAsync(&tot, vpre.as<int>() + K, sizeof(int), cudaMemcpyDeviceToHost, s));
        MSCG_CUDA(cudaStreamSynchronize(s));
        if (tot == 0) break;
      }
      total_rounds += round;
    };
    bfs(0);  // from the start, first component: f1
    MSCG_CUDA(cudaMemcpyAsync(f1.p, fend.p, sizeof(int) * K, cudaMemcpyDeviceToDevice, s));
    MSCG_CUDA(cudaMemcpyAsync(src.p, fend.p, sizeof(int) * K, cudaMemcpyDeviceToDevice, s));
    bfs(1);  // from f1: f2
    origin_kernel<<<Kb, kT, 0, s>>>(f1.as<int>(), fend.as<int>(), K, src.as<int>());
    bfs(2);  // from min(f1, f2), every component: the cut round
    label_kernel<<<Gn, kT, 0, s>>>(L, lab.as<char>());
    MSCG_CUDA(cudaMemsetAsync(counts.p, 0, counts.bytes, s));
    separator_kernel<<<Gn, kT, 0, s>>>(L, lab.as<char>(), counts.as<int>());
    ctx->launches += 3;
    std::vector<int> hc(3 * K);
    MSCG_CUDA(cudaMemcpyAsync(hc.data(), counts.p, sizeof(int) * 3 * K, cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaStreamSynchronize(s));
    // children in left-to-right order; degenerate splits stay whole as leaves
    std::vector<int> h_split(K, 0), h_base(K), n_active, n_sizes;
    int nk = 0;
    for (int k = 0; k < K; ++k) {
      h_base[k] = nk;
      if (h_active[k] && hc[3 * k] > 0 && hc[3 * k + 1] > 0) {
        h_split[k] = 1;
        n_active.push_back(1);
        n_sizes.push_back(hc[3 * k]);
        n_active.push_back(1);
        n_sizes.push_back(hc[3 * k + 1]);
        nk += 2;
      } else {
        n_active.push_back(0);
        n_sizes.push_back(h_sizes[k]);
        nk += 1;
      }
    }
    MSCG_CUDA(cudaMemcpyAsync(split.p, h_split.data(), sizeof(int) * K, cudaMemcpyHostToDevice, s));
    MSCG_CUDA(cudaMemcpyAsync(base.p, h_base.data(), sizeof(int) * K, cudaMemcpyHostToDevice, s));
    relabel_kernel<<<Gn, kT, 0, s>>>(n, piece.as<int>(), lab.as<char>(), active.as<int>(),
                                     split.as<int>(), base.as<int>());
    ctx->launches++;
    MSCG_CUDA(cudaStreamSynchronize(s));  // the per-level buffers go out of scope
    K = nk;
    h_active = std::move(n_active);
    h_sizes = std::move(n_sizes);
    if (verbose) {
      const auto now = clk::now();
      fprintf(stderr, "nested_dissection_device: level %d, %d pieces next, %lld rounds so far, %.3f s\n",
              d, K, total_rounds, std::chrono::duration<double>(now - tl).count());
      tl = now;
    }
  }
  MSCG_CUDA(cudaStreamSynchronize(s));
  return K;
}

void nested_dissection_device(Ctx* ctx, int n, const int64_t* h_off, const int* h_adj,
                              int target_blocks, std::vector<std::vector<int>>& blocks,
                              std::vector<int>& separator) {
  if (target_blocks < 1 || target_blocks > std::max(n, 1))
    throw Error(1, "nested_dissection: target_blocks out of range");
  blocks.clear();
  separator.clear();
  if (target_blocks == 1 || n <= 1) {
    std::vector<int> all(n);
    for (int i = 0; i < n; ++i) all[i] = i;
    blocks.push_back(std::move(all));
    return;
  }
  cudaStream_t s = ctx->stream;
  const long long ne = h_off[n];
  DevBuf d_off(sizeof(long long) * (n + 1)), d_adj(sizeof(int) * std::max<long long>(1, ne));
  MSCG_CUDA(cudaMemcpyAsync(d_off.p, h_off, sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, s));
  if (ne) MSCG_CUDA(cudaMemcpyAsync(d_adj.p, h_adj, sizeof(int) * ne, cudaMemcpyHostToDevice, s));
  DevBuf piece(sizeof(int) * n);
  const int K = nested_dissection_core(ctx, n, d_off.as<long long>(), d_adj.as<int>(),
                                       target_blocks, piece.as<int>());
  std::vector<int> hp(n);
  MSCG_CUDA(cudaMemcpyAsync(hp.data(), piece.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  // blocks: pieces in order, each ascending; separator ascending
  blocks.resize(K);
  for (int u = 0; u < n; ++u) (hp[u] < 0 ? separator : blocks[hp[u]]).push_back(u);
}

}  // namespace mscg
