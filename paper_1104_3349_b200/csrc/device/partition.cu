// partition_saddle (Interleaved) on the device (reference
// proj/src/partitioned_matrix.cpp:71-203 with nested_dissection,
// proj/src/graph.cpp:136-230), and the SURVEY 8(d)
// interface anchoring:
//   1. attached(q): the first-block nodes coupled to second-block unknown q
//      (both C[i, p+q] and C[p+q, j]), sorted and unique (:112-124);
//   2. the enriched graph: the (1,1) off-diagonal pattern plus a clique on
//      every attached(q), symmetrised, each adjacency sorted and unique
//      (:104-140);
//   3. nested dissection of it (csrc/device/dissect.cu);
//   4. every second-block unknown follows the block of its first attached
//      node that is not in the separator (:146-175); the forward map is
//      [block 0 nodes, block 0 unknowns, block 1 ..., separator, the rest],
//      each group ascending — one stable radix sort by group;
//   5. C' = P C P^T (rows gathered, columns renumbered and sorted per row)
//      and the block-diagonal invariant (:197-201) checked on the device.
// Everything reproduces the host build (csrc/host/partition.cpp) and hence
// the reference bit for bit; the tests compare the permutations and C'.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "host/setup.hpp"

namespace mscg {

int nested_dissection_core(Ctx* ctx, int n, const long long* d_off, const int* d_adj,
                           int target_blocks, int* piece_out);

namespace {

constexpr int kT = 256;

template <class T>
T* up(DevBuf& b, const std::vector<T>& h, cudaStream_t s) {
  b = DevBuf(sizeof(T) * std::max<size_t>(1, h.size()));
  if (!h.empty()) MSCG_CUDA(cudaMemcpyAsync(b.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
  return b.as<T>();
}

long long exclusive_scan(Ctx* ctx, const long long* in, long long* out, int n) {
  // out[0..n] = exclusive prefix, out[n] = total (in has n entries)
  cudaStream_t s = ctx->stream;
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n + 1, s);
  DevBuf tmp(std::max<size_t>(tb, 16));
  MSCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n + 1, s));
  long long tot = 0;
  MSCG_CUDA(cudaMemcpyAsync(&tot, out + n, sizeof(long long), cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  return tot;
}

// (1) attached lists: counts, then entries
__global__ void att_count_kernel(int n, int p, const int* rp, const int* ci, long long* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < p) {
      for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] >= p) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (ci[k] - p)), 1ull);
    } else {
      long long c = 0;
      for (int k = rp[i]; k < rp[i + 1]; ++k) c += ci[k] < p;
      if (c) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (i - p)), static_cast<unsigned long long>(c));
    }
  }
}
__global__ void att_fill_kernel(int n, int p, const int* rp, const int* ci, const long long* off,
                                long long* pos, int* att) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < p) {
      for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] >= p) {
          const int q = ci[k] - p;
          att[off[q] + atomicAdd(reinterpret_cast<unsigned long long*>(pos + q), 1ull)] = i;
        }
    } else {
      const int q = i - p;
      for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] < p) att[off[q] + atomicAdd(reinterpret_cast<unsigned long long*>(pos + q), 1ull)] = ci[k];
    }
  }
}
// per segment of a sorted list: drop duplicates in place, length -> len
__global__ void dedupe_kernel(int nseg, const long long* off, int* a, long long* len) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nseg; q += gridDim.x * blockDim.x) {
    const long long b = off[q], e = off[q + 1];
    long long w = b;
    for (long long k = b; k < e; ++k)
      if (k == b || a[k] != a[k - 1]) a[w++] = a[k];
    len[q] = w - b;
  }
}

// (2) enriched graph: raw counts and entries
__global__ void graph_count_kernel(int p, const int* rp, const int* ci, int ng,
                                   const long long* aoff, const long long* alen, const int* att,
                                   long long* cnt) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < p; i += nt)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k];
      if (j < p && j != i) {
        atomicAdd(reinterpret_cast<unsigned long long*>(cnt + i), 1ull);
        atomicAdd(reinterpret_cast<unsigned long long*>(cnt + j), 1ull);
      }
    }
  for (int q = tid; q < ng; q += nt) {
    const long long m = alen[q];
    for (long long a = 0; a < m; ++a)
      atomicAdd(reinterpret_cast<unsigned long long*>(cnt + att[aoff[q] + a]),
                static_cast<unsigned long long>(m - 1));
  }
}
__global__ void graph_fill_kernel(int p, const int* rp, const int* ci, int ng,
                                  const long long* aoff, const long long* alen, const int* att,
                                  const long long* off, long long* pos, int* raw) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  auto put = [&](int u, int v) {
    raw[off[u] + atomicAdd(reinterpret_cast<unsigned long long*>(pos + u), 1ull)] = v;
  };
  for (int i = tid; i < p; i += nt)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k];
      if (j < p && j != i) {
        put(i, j);
        put(j, i);
      }
    }
  for (int q = tid; q < ng; q += nt) {
    const long long m = alen[q];
    const int* nodes = att + aoff[q];
    for (long long a = 0; a < m; ++a)
      for (long long b = 0; b < m; ++b)
        if (a != b) put(nodes[a], nodes[b]);
  }
}
// the deduplicated head of each raw segment -> the packed adjacency
__global__ void compact_kernel(int nseg, const long long* roff, const int* raw, const long long* off,
                               int* adj) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nseg; u += gridDim.x * blockDim.x) {
    const long long m = off[u + 1] - off[u];
    for (long long k = 0; k < m; ++k) adj[off[u] + k] = raw[roff[u] + k];
  }
}

// (4) second-block unknowns: the block of the first attached node outside
// the separator; then the group keys of the forward map
__global__ void key_kernel(int n, int p, const int* piece, const long long* aoff,
                           const long long* alen, const int* att, int K, unsigned* key) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < p) {
      const int k = piece[i];
      key[i] = k >= 0 ? 2u * k : 2u * K;
    } else {
      const int q = i - p;
      int blk = -1;
      for (long long a = 0; a < alen[q]; ++a) {
        const int k = piece[att[aoff[q] + a]];
        if (k >= 0) {
          blk = k;
          break;
        }
      }
      key[i] = blk >= 0 ? 2u * blk + 1u : 2u * K + 1u;
    }
  }
}
__global__ void iota_kernel(int n, int* a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}
// group boundaries of the sorted keys: gstart[g] = first position of key g
__global__ void group_bounds_kernel(int n, const unsigned* sk, int ngroups, int* gstart) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned k = sk[i];
    const long long prev = i == 0 ? -1 : static_cast<long long>(sk[i - 1]);
    for (long long g = prev + 1; g <= static_cast<long long>(k) && g <= ngroups; ++g) gstart[g] = i;
    if (i == n - 1)
      for (long long g = static_cast<long long>(k) + 1; g <= ngroups; ++g) gstart[g] = n;
  }
}

// (5) C' = P C P^T: row lengths, then rows gathered with renumbered columns,
// insertion-sorted (rows are short)
__global__ void inv_kernel(int n, const int* fwd, int* inv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) inv[fwd[i]] = i;
}
__global__ void rowlen_kernel(int n, const int* rp, const int* fwd, long long* len) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    len[i] = rp[fwd[i] + 1] - rp[fwd[i]];
}
__global__ void permute_kernel(int n, const int* rp, const int* ci, const double* v, const int* fwd,
                               const int* inv, const long long* orp, int* oci, double* ov) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = fwd[i];
    const long long w0 = orp[i];
    int m = 0;
    for (int k = rp[o]; k < rp[o + 1]; ++k, ++m) {
      const int c = inv[ci[k]];
      const double x = v[k];
      long long j = w0 + m;
      while (j > w0 && oci[j - 1] > c) {
        oci[j] = oci[j - 1];
        ov[j] = ov[j - 1];
        --j;
      }
      oci[j] = c;
      ov[j] = x;
    }
  }
}
// entries of C'[0:p, 0:p] coupling different blocks (must be none)
__global__ void coupled_kernel(int p, const long long* rp, const int* ci, const int* bown,
                               unsigned long long* bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x)
    for (long long k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] < p && bown[ci[k]] != bown[i]) atomicAdd(bad, 1ull);
}
__global__ void bown_kernel(int p, const int* gstart, int K, int* bown) {
  // position i < p belongs to block b when it lies in groups 2b or 2b+1
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
    int lo = 0, hi = K;  // block b covers [gstart[2b], gstart[2b + 2])
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (gstart[2 * mid] <= i)
        lo = mid;
      else
        hi = mid;
    }
    bown[i] = lo;
  }
}
// anchoring keys: interface velocity v -> 2v, a pressure whose
// first interface-velocity neighbour is v -> 2v + 1, the rest -> 2 nsep
__global__ void anchor_key_kernel(int n, int p, int nsep, const long long* rp, const int* ci,
                                  unsigned* key) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n - p; q += gridDim.x * blockDim.x) {
    if (q < nsep) {
      key[q] = 2u * q;
      continue;
    }
    int best = -1;
    for (long long k = rp[p + q]; k < rp[p + q + 1]; ++k) {
      const int c = ci[k] - p;
      if (c >= 0 && c < nsep) {
        best = c;
        break;
      }
    }
    key[q] = best >= 0 ? 2u * best + 1u : 2u * nsep;
  }
}
__global__ void anchor_fwd_kernel(int n, int p, const int* sorted_q, int* fwd) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    fwd[i] = i < p ? i : p + sorted_q[i - p];
}
__global__ void compose_kernel(int n, const int* perm, const int* fwd, int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = perm[fwd[i]];
}

int bits_for(unsigned maxkey) {
  int b = 1;
  while (b < 32 && (1ull << b) <= maxkey) ++b;
  return b;
}

// stable sort of 0..n-1 by key (ascending), values out
void sort_ids(Ctx* ctx, int n, unsigned* key, unsigned maxkey, int* ids_out, unsigned* skey) {
  cudaStream_t s = ctx->stream;
  DevBuf ids(sizeof(int) * std::max(n, 1));
  iota_kernel<<<4 * ctx->sm_count, kT, 0, s>>>(n, ids.as<int>());
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, key, skey, ids.as<int>(), ids_out, n, 0,
                                  bits_for(maxkey), s);
  DevBuf tmp(std::max<size_t>(tb, 16));
  MSCG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key, skey, ids.as<int>(), ids_out, n, 0,
                                            bits_for(maxkey), s));
  ctx->launches += 2;
}

// C' = P C P^T on the device (permute_symmetric)
void permute_device(Ctx* ctx, int n, const int* rp, const int* ci, const double* v,
                    const int* fwd, DevBuf& orp, DevBuf& oci, DevBuf& ov) {
  cudaStream_t s = ctx->stream;
  const int G = 4 * ctx->sm_count;
  DevBuf inv(sizeof(int) * std::max(n, 1)), len(sizeof(long long) * (n + 1));
  inv_kernel<<<G, kT, 0, s>>>(n, fwd, inv.as<int>());
  rowlen_kernel<<<G, kT, 0, s>>>(n, rp, fwd, len.as<long long>());
  orp = DevBuf(sizeof(long long) * (n + 1));
  const long long nnz = exclusive_scan(ctx, len.as<long long>(), orp.as<long long>(), n);
  oci = DevBuf(sizeof(int) * std::max<long long>(1, nnz));
  ov = DevBuf(sizeof(double) * std::max<long long>(1, nnz));
  permute_kernel<<<G, kT, 0, s>>>(n, rp, ci, v, fwd, inv.as<int>(), orp.as<long long>(),
                                  oci.as<int>(), ov.as<double>());
  ctx->launches += 3;
}

__global__ void narrow_kernel(int n, const long long* a, int* b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
    b[i] = static_cast<int>(a[i]);
}

}  // namespace

host::Partitioned partition_saddle_device(Ctx* ctx, const host::Csr& c, int p, int target_blocks,
                                          bool anchored) {
  if (c.nrows != c.ncols || p < 1 || p > c.nrows)
    throw Error(1, "partition_saddle: bad split");
  using clk = std::chrono::steady_clock;
  static const bool verbose = getenv("MSCG_VERBOSE") != nullptr;
  const auto t0 = clk::now();
  cudaStream_t s = ctx->stream;
  const int n = c.nrows, ng = n - p;
  const int G = 4 * ctx->sm_count;
  DevBuf drp, dci, dv;
  const int* rp = up(drp, c.rp, s);
  const int* ci = up(dci, c.ci, s);
  const double* v = up(dv, c.v, s);
  // (1) attached lists
  DevBuf acnt(sizeof(long long) * (ng + 1)), aoff(sizeof(long long) * (ng + 1)),
      apos(sizeof(long long) * (ng + 1)), alen(sizeof(long long) * std::max(ng, 1));
  MSCG_CUDA(cudaMemsetAsync(acnt.p, 0, acnt.bytes, s));
  MSCG_CUDA(cudaMemsetAsync(apos.p, 0, apos.bytes, s));
  att_count_kernel<<<G, kT, 0, s>>>(n, p, rp, ci, acnt.as<long long>());
  const long long natt = exclusive_scan(ctx, acnt.as<long long>(), aoff.as<long long>(), ng);
  DevBuf att(sizeof(int) * std::max<long long>(1, natt)), att2(sizeof(int) * std::max<long long>(1, natt));
  att_fill_kernel<<<G, kT, 0, s>>>(n, p, rp, ci, aoff.as<long long>(), apos.as<long long>(),
                                   att.as<int>());
  {
    size_t tb = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, tb, att.as<int>(), att2.as<int>(), natt, ng,
                                       aoff.as<long long>(), aoff.as<long long>() + 1, s);
    DevBuf tmp(std::max<size_t>(tb, 16));
    MSCG_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, att.as<int>(), att2.as<int>(), natt,
                                                 ng, aoff.as<long long>(),
                                                 aoff.as<long long>() + 1, s));
  }
  dedupe_kernel<<<G, kT, 0, s>>>(ng, aoff.as<long long>(), att2.as<int>(), alen.as<long long>());
  ctx->launches += 3;
  // (2) enriched graph
  DevBuf gcnt(sizeof(long long) * (p + 1)), groff(sizeof(long long) * (p + 1)),
      gpos(sizeof(long long) * (p + 1)), glen(sizeof(long long) * (p + 1)),
      goff(sizeof(long long) * (p + 1));
  MSCG_CUDA(cudaMemsetAsync(gcnt.p, 0, gcnt.bytes, s));
  MSCG_CUDA(cudaMemsetAsync(gpos.p, 0, gpos.bytes, s));
  graph_count_kernel<<<G, kT, 0, s>>>(p, rp, ci, ng, aoff.as<long long>(), alen.as<long long>(),
                                      att2.as<int>(), gcnt.as<long long>());
  const long long nraw = exclusive_scan(ctx, gcnt.as<long long>(), groff.as<long long>(), p);
  DevBuf raw(sizeof(int) * std::max<long long>(1, nraw)), raw2(sizeof(int) * std::max<long long>(1, nraw));
  graph_fill_kernel<<<G, kT, 0, s>>>(p, rp, ci, ng, aoff.as<long long>(), alen.as<long long>(),
                                     att2.as<int>(), groff.as<long long>(), gpos.as<long long>(),
                                     raw.as<int>());
  {
    size_t tb = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, tb, raw.as<int>(), raw2.as<int>(), nraw, p,
                                       groff.as<long long>(), groff.as<long long>() + 1, s);
    DevBuf tmp(std::max<size_t>(tb, 16));
    MSCG_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, raw.as<int>(), raw2.as<int>(), nraw,
                                                 p, groff.as<long long>(),
                                                 groff.as<long long>() + 1, s));
  }
  raw = DevBuf();
  dedupe_kernel<<<G, kT, 0, s>>>(p, groff.as<long long>(), raw2.as<int>(), glen.as<long long>());
  const long long ne = exclusive_scan(ctx, glen.as<long long>(), goff.as<long long>(), p);
  DevBuf adj(sizeof(int) * std::max<long long>(1, ne));
  compact_kernel<<<G, kT, 0, s>>>(p, groff.as<long long>(), raw2.as<int>(), goff.as<long long>(),
                                  adj.as<int>());
  ctx->launches += 5;
  raw2 = DevBuf();
  MSCG_CUDA(cudaStreamSynchronize(s));
  const auto t1 = clk::now();
  // (3) nested dissection
  DevBuf piece(sizeof(int) * p);
  const int K = nested_dissection_core(ctx, p, goff.as<long long>(), adj.as<int>(), target_blocks,
                                       piece.as<int>());
  const auto t2 = clk::now();
  adj = DevBuf();
  // (4) forward map by group
  DevBuf key(sizeof(unsigned) * n), skey(sizeof(unsigned) * n), fwd(sizeof(int) * n),
      gstart(sizeof(int) * (2 * K + 3));
  key_kernel<<<G, kT, 0, s>>>(n, p, piece.as<int>(), aoff.as<long long>(), alen.as<long long>(),
                              att2.as<int>(), K, key.as<unsigned>());
  sort_ids(ctx, n, key.as<unsigned>(), 2u * K + 1u, fwd.as<int>(), skey.as<unsigned>());
  group_bounds_kernel<<<G, kT, 0, s>>>(n, skey.as<unsigned>(), 2 * K + 2, gstart.as<int>());
  ctx->launches += 2;
  std::vector<int> gs(2 * K + 3);
  MSCG_CUDA(cudaMemcpyAsync(gs.data(), gstart.p, sizeof(int) * gs.size(), cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  host::Partitioned out;
  for (int b = 0; b < K; ++b) out.d_ranges.push_back({gs[2 * b], gs[2 * b + 2]});
  out.p = gs[2 * K];
  out.separator_size = gs[2 * K + 1] - gs[2 * K];
  // (5) C' = P C P^T, block-diagonal check
  DevBuf orp, oci, ov;
  permute_device(ctx, n, rp, ci, v, fwd.as<int>(), orp, oci, ov);
  {
    DevBuf bown(sizeof(int) * std::max(out.p, 1)), bad(sizeof(unsigned long long));
    MSCG_CUDA(cudaMemsetAsync(bad.p, 0, bad.bytes, s));
    bown_kernel<<<G, kT, 0, s>>>(out.p, gstart.as<int>(), K, bown.as<int>());
    coupled_kernel<<<G, kT, 0, s>>>(out.p, orp.as<long long>(), oci.as<int>(), bown.as<int>(),
                                    bad.as<unsigned long long>());
    unsigned long long hb = 0;
    MSCG_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 2;
    if (hb)
      throw Error(1, "partition_saddle: interior blocks remained coupled (" + std::to_string(hb) +
                         " entries)");
  }
  DevBuf perm = std::move(fwd);
  const int pp = out.p, nsep = out.separator_size;
  if (anchored) {
    // SURVEY 8(d) interface anchoring: a symmetric permutation of the (2,2)
    // side, composed with the partition's
    DevBuf qkey(sizeof(unsigned) * std::max(n - pp, 1)), sq(sizeof(unsigned) * std::max(n - pp, 1)),
        qs(sizeof(int) * std::max(n - pp, 1)), afwd(sizeof(int) * n), comp(sizeof(int) * n);
    anchor_key_kernel<<<G, kT, 0, s>>>(n, pp, nsep, orp.as<long long>(), oci.as<int>(),
                                       qkey.as<unsigned>());
    sort_ids(ctx, n - pp, qkey.as<unsigned>(), 2u * nsep, qs.as<int>(), sq.as<unsigned>());
    anchor_fwd_kernel<<<G, kT, 0, s>>>(n, pp, qs.as<int>(), afwd.as<int>());
    // the permutation kernels take int32 row offsets
    DevBuf orp32(sizeof(int) * (n + 1));
    narrow_kernel<<<G, kT, 0, s>>>(n, orp.as<long long>(), orp32.as<int>());
    DevBuf arp, aci, av;
    permute_device(ctx, n, orp32.as<int>(), oci.as<int>(), ov.as<double>(), afwd.as<int>(), arp, aci, av);
    compose_kernel<<<G, kT, 0, s>>>(n, perm.as<int>(), afwd.as<int>(), comp.as<int>());
    ctx->launches += 4;
    orp = std::move(arp);
    oci = std::move(aci);
    ov = std::move(av);
    perm = std::move(comp);
  }
  // back to the host problem
  std::vector<long long> hrp(n + 1);
  MSCG_CUDA(cudaMemcpyAsync(hrp.data(), orp.p, sizeof(long long) * (n + 1), cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  const long long nnz = hrp[n];
  out.C = host::Csr(n, n);
  for (int i = 0; i <= n; ++i) out.C.rp[i] = static_cast<int>(hrp[i]);
  out.C.ci.resize(nnz);
  out.C.v.resize(nnz);
  out.perm.resize(n);
  if (nnz) {
    MSCG_CUDA(cudaMemcpyAsync(out.C.ci.data(), oci.p, sizeof(int) * nnz, cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaMemcpyAsync(out.C.v.data(), ov.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
  }
  MSCG_CUDA(cudaMemcpyAsync(out.perm.data(), perm.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  if (verbose) {
    const auto t3 = clk::now();
    fprintf(stderr,
            "partition_saddle_device: enriched graph %d nodes %lld edges %.3f s, dissection %.3f s, "
            "permutation%s %.3f s\n",
            p, ne, std::chrono::duration<double>(t1 - t0).count(),
            std::chrono::duration<double>(t2 - t1).count(), anchored ? " + anchoring" : "",
            std::chrono::duration<double>(t3 - t2).count());
  }
  return out;
}

}  // namespace mscg
