// Host problem layer, part 2: interleaved saddle partition by nested
// dissection, and the SURVEY §8(d) interface anchoring.
//
// Reproduces the reference ordering exactly:
//   partition_saddle (Interleaved)  proj/src/partitioned_matrix.cpp:100-202
//   nested_dissection / dissect     proj/src/graph.cpp:178-230
//   bisect / pseudo_peripheral      proj/src/graph.cpp:94-176
//   bfs_levels                      proj/src/graph.cpp:70-92
// The reference allocates O(n) scratch per bisection and recurses
// sequentially (172 s at cfg5).  Here the dissection tree is
// expanded level by level, the pieces of a level are bisected concurrently
// with per-thread epoch-stamped scratch, and leaves keep their left-to-right
// (= depth-first) order, so the block list and separator are identical.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <thread>

#include "setup.hpp"

namespace mscg::host {

int hardware_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 1 : static_cast<int>(h);
}

template <class F>
static void parallel_for(int n, int threads, F&& f) {
  if (threads <= 1 || n <= 1) {
    for (int i = 0; i < n; ++i) f(i, 0);
    return;
  }
  const int t = std::min(threads, n);
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int w = 0; w < t; ++w)
    pool.emplace_back([&, w] {
      for (int i = next++; i < n; i = next++) f(i, w);
    });
  for (auto& th : pool) th.join();
}

Csr permute_symmetric(const Csr& a, const std::vector<int>& fwd,
                      const std::vector<int>& inv) {
  const int n = a.nrows;
  Csr out(n, n);
  for (int i = 0; i < n; ++i) out.rp[i + 1] = out.rp[i] + (a.rp[fwd[i] + 1] - a.rp[fwd[i]]);
  out.ci.resize(a.nnz());
  out.v.resize(a.nnz());
  parallel_for(std::max(1, n / 65536 + 1), hardware_threads(), [&](int chunk, int) {
    const int lo = chunk * 65536, hi = std::min(n, lo + 65536);
    std::vector<std::pair<int, double>> tmp;
    for (int i = lo; i < hi; ++i) {
      const int o = fwd[i];
      tmp.clear();
      for (int k = a.rp[o]; k < a.rp[o + 1]; ++k) tmp.push_back({inv[a.ci[k]], a.v[k]});
      std::sort(tmp.begin(), tmp.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      int w = out.rp[i];
      for (auto& [c, v] : tmp) {
        out.ci[w] = c;
        out.v[w++] = v;
      }
    }
  });
  return out;
}

namespace {

// Undirected adjacency (symmetrised closure of the enriched pattern,
// graph.cpp:8-30), sorted, no self loops.
struct Graph {
  int n = 0;
  std::vector<int64_t> off;
  std::vector<int> adj;
  int deg(int u) const { return static_cast<int>(off[u + 1] - off[u]); }
};

// Per-thread scratch.  st[v] packs (piece epoch << 32 | visited epoch) so the
// BFS membership and visited tests are one random access per edge.
struct Scratch {
  std::vector<uint64_t> st;
  std::vector<int> left;
  int epoch = 0;
  explicit Scratch(int n) : st(n, 0), left(n, 0) {}
};

struct LevelOrder {
  std::vector<int> order, level;
};

// bfs_levels (graph.cpp:70-92).  When only_first is set, stop after the
// start's component (all pseudo_peripheral needs).  Visit order and levels
// are the reference's: FIFO queue, neighbours in adjacency order; levels are
// read off the queue's level boundaries.  The queue runs ahead with software
// prefetches (adjacency lists kPfAdj nodes ahead, their neighbours' state
// kPfSt nodes ahead): the walk is bound by random accesses to st[].
void bfs_levels(const Graph& g, const std::vector<int>& nodes, Scratch& s,
                int mem_ep, int start, bool only_first, LevelOrder& lo) {
  constexpr std::size_t kPfAdj = 16, kPfSt = 6;
  const uint32_t ep = static_cast<uint32_t>(++s.epoch);
  const uint64_t mem_hi = static_cast<uint64_t>(static_cast<uint32_t>(mem_ep)) << 32;
  uint64_t* st = s.st.data();
  const int64_t* off = g.off.data();
  const int* adj = g.adj.data();
  lo.order.clear();
  lo.level.clear();
  auto run = [&](int src) {
    std::size_t head = lo.order.size();
    st[src] = mem_hi | ep;
    lo.order.push_back(src);
    int level = 0;
    std::size_t level_end = head + 1;
    while (head < lo.order.size()) {
      if (head == level_end) {
        ++level;
        level_end = lo.order.size();
      }
      if (head + kPfAdj < lo.order.size()) __builtin_prefetch(adj + off[lo.order[head + kPfAdj]]);
      if (head + kPfSt < lo.order.size()) {
        const int w = lo.order[head + kPfSt];
        for (int64_t k = off[w]; k < off[w + 1]; ++k) __builtin_prefetch(st + adj[k]);
      }
      const int u = lo.order[head++];
      lo.level.push_back(level);
      for (int64_t k = off[u]; k < off[u + 1]; ++k) {
        const int v = adj[k];
        const uint64_t sv = st[v];
        if ((sv & 0xffffffff00000000ull) == mem_hi && static_cast<uint32_t>(sv) != ep) {
          st[v] = mem_hi | ep;
          lo.order.push_back(v);
        }
      }
    }
  };
  if (start >= 0) run(start);
  if (only_first) return;
  for (int u : nodes)
    if (static_cast<uint32_t>(st[u]) != ep) run(u);
}

struct Split {
  std::vector<int> left, right, sep;
  bool degenerate = false;
};

// bisect (graph.cpp:136-176) with pseudo_peripheral (graph.cpp:94-117).
Split bisect(const Graph& g, const std::vector<int>& nodes, Scratch& s) {
  const int mem_ep = ++s.epoch;
  const uint64_t mem_hi = static_cast<uint64_t>(static_cast<uint32_t>(mem_ep)) << 32;
  for (int u : nodes) s.st[u] = mem_hi;  // member, not visited
  int start = nodes.front();
  int best = g.deg(start);
  for (int u : nodes)
    if (g.deg(u) < best) {
      best = g.deg(u);
      start = u;
    }
  LevelOrder lo;
  lo.order.reserve(nodes.size());
  lo.level.reserve(nodes.size());
  bfs_levels(g, nodes, s, mem_ep, start, true, lo);
  const int f1 = lo.order.back();
  bfs_levels(g, nodes, s, mem_ep, f1, true, lo);
  const int f2 = lo.order.back();
  const int origin = std::min(f1, f2);
  bfs_levels(g, nodes, s, mem_ep, origin, false, lo);

  std::size_t cut = nodes.size() / 2;
  while (cut < lo.order.size() && cut > 0 && lo.level[cut] == lo.level[cut - 1] &&
         lo.level[cut] != 0)
    ++cut;
  Split r;
  const int lep = ++s.epoch;
  const int sep_ep = ++s.epoch;
  for (std::size_t i = 0; i < cut && i < lo.order.size(); ++i) s.left[lo.order[i]] = lep;
  std::size_t nleft = std::min(cut, lo.order.size()), nsep = 0;
  for (std::size_t i = cut; i < lo.order.size(); ++i) {
    const int u = lo.order[i];
    if (i + 6 < lo.order.size()) {
      const int w = lo.order[i + 6];
      for (int64_t k = g.off[w]; k < g.off[w + 1]; ++k) __builtin_prefetch(&s.left[g.adj[k]]);
    }
    for (int64_t k = g.off[u]; k < g.off[u + 1]; ++k)
      if (s.left[g.adj[k]] == lep) {
        s.left[u] = sep_ep;
        ++nsep;
        break;
      }
  }
  // the piece's node list is ascending, so one pass over it yields the three
  // sorted sides without sorting
  r.left.reserve(nleft);
  r.sep.reserve(nsep);
  r.right.reserve(nodes.size() - nleft - nsep);
  for (int u : nodes) {
    const int m = s.left[u];
    (m == lep ? r.left : m == sep_ep ? r.sep : r.right).push_back(u);
  }
  r.degenerate = r.left.empty() || r.right.empty();
  return r;
}

struct Piece {
  std::vector<int> nodes;
  bool leaf = false;
};

// nested_dissection (graph.cpp:198-230): returns blocks (in depth-first leaf
// order) and the sorted separator.
void nested_dissection(const Graph& g, int target_blocks, int threads,
                       std::vector<std::vector<int>>& blocks,
                       std::vector<int>& separator) {
  if (target_blocks < 1 || target_blocks > std::max(g.n, 1))
    throw std::invalid_argument("nested_dissection: target_blocks out of range");
  blocks.clear();
  separator.clear();
  if (target_blocks == 1 || g.n <= 1) {
    std::vector<int> all(g.n);
    for (int i = 0; i < g.n; ++i) all[i] = i;
    blocks.push_back(std::move(all));
    return;
  }
  int depth = 0;
  while ((1 << depth) < target_blocks) ++depth;
  static const bool verbose = getenv("MSCG_VERBOSE") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  std::vector<Piece> pieces(1);
  pieces[0].nodes.resize(g.n);
  for (int i = 0; i < g.n; ++i) pieces[0].nodes[i] = i;
  const int nthreads = std::max(1, std::min(threads, 16));
  std::vector<std::unique_ptr<Scratch>> scratch(nthreads);
  for (int d = 0; d < depth; ++d) {
    std::vector<Split> splits(pieces.size());
    std::vector<int> todo;
    for (std::size_t i = 0; i < pieces.size(); ++i) {
      if (pieces[i].leaf) continue;
      if (pieces[i].nodes.size() <= 1) {
        pieces[i].leaf = true;
        continue;
      }
      todo.push_back(static_cast<int>(i));
    }
    parallel_for(static_cast<int>(todo.size()), nthreads, [&](int t, int w) {
      if (!scratch[w]) scratch[w] = std::make_unique<Scratch>(g.n);
      splits[todo[t]] = bisect(g, pieces[todo[t]].nodes, *scratch[w]);
    });
    std::vector<Piece> next;
    next.reserve(pieces.size() * 2);
    for (std::size_t i = 0; i < pieces.size(); ++i) {
      Piece& pc = pieces[i];
      if (pc.leaf) {
        next.push_back(std::move(pc));
        continue;
      }
      Split& sp = splits[i];
      if (sp.degenerate) {
        pc.leaf = true;
        next.push_back(std::move(pc));
        continue;
      }
      separator.insert(separator.end(), sp.sep.begin(), sp.sep.end());
      next.push_back(Piece{std::move(sp.left), false});
      next.push_back(Piece{std::move(sp.right), false});
    }
    pieces = std::move(next);
    if (verbose) {
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "nested_dissection: level %d, %zu pieces, %.3f s\n", d, todo.size(),
              std::chrono::duration<double>(now - tl).count());
      tl = now;
    }
  }
  std::sort(separator.begin(), separator.end());
  for (auto& pc : pieces) blocks.push_back(std::move(pc.nodes));
}

}  // namespace

void nested_dissection_host(int n, const int64_t* off, const int* adj, int target_blocks,
                            int threads, std::vector<std::vector<int>>& blocks,
                            std::vector<int>& separator) {
  Graph g;
  g.n = n;
  g.off.assign(off, off + n + 1);
  g.adj.assign(adj, adj + off[n]);
  nested_dissection(g, target_blocks, threads <= 0 ? hardware_threads() : threads, blocks,
                    separator);
}

void undirected_graph(int n, const int* rp, const int* ci, std::vector<int64_t>& off,
                      std::vector<int>& adj) {
  // build_graph (graph.cpp:8-30) as the reference computes it: node i's list
  // is its own off-diagonal row pattern plus the rows j > i that list i.
  // (The reference assigns undirected[i] = out[i] at step i, overwriting the
  // entries earlier rows pushed, so the "undirected" lists are symmetric only
  // for structurally symmetric patterns — such as the saddle systems here.)
  std::vector<int64_t> cnt(n + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] != i) {
        ++cnt[i + 1];
        if (ci[k] < i) ++cnt[ci[k] + 1];
      }
  for (int i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int> raw(cnt[n]);
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (int i = 0; i < n; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] != i) {
        raw[pos[i]++] = ci[k];
        if (ci[k] < i) raw[pos[ci[k]]++] = i;
      }
  off.assign(n + 1, 0);
  adj.clear();
  for (int i = 0; i < n; ++i) {
    auto b = raw.begin() + cnt[i], e = raw.begin() + cnt[i + 1];
    std::sort(b, e);
    e = std::unique(b, e);
    adj.insert(adj.end(), b, e);
    off[i + 1] = static_cast<int64_t>(adj.size());
  }
}

Partitioned partition_saddle(const Csr& c, int p, int target_blocks, int threads,
                             const Dissector& dissect) {
  if (c.nrows != c.ncols || p < 1 || p > c.nrows)
    throw std::invalid_argument("partition_saddle: bad split");
  if (threads <= 0) threads = hardware_threads();
  const int n = c.nrows;
  const int ng = n - p;
  const auto t_start = std::chrono::steady_clock::now();

  // attached[q]: first-block nodes coupled to second-block unknown q
  // (partitioned_matrix.cpp:112-124), as a sorted, unique CSR list.
  std::vector<int64_t> aoff(ng + 1, 0);
  for (int i = 0; i < p; ++i)
    for (int k = c.rp[i]; k < c.rp[i + 1]; ++k)
      if (c.ci[k] >= p) ++aoff[c.ci[k] - p + 1];
  for (int q = 0; q < ng; ++q)
    for (int k = c.rp[p + q]; k < c.rp[p + q + 1]; ++k)
      if (c.ci[k] < p) ++aoff[q + 1];
  for (int q = 0; q < ng; ++q) aoff[q + 1] += aoff[q];
  std::vector<int> att(aoff[ng]);
  {
    std::vector<int64_t> pos(aoff.begin(), aoff.end() - 1);
    for (int i = 0; i < p; ++i)
      for (int k = c.rp[i]; k < c.rp[i + 1]; ++k)
        if (c.ci[k] >= p) att[pos[c.ci[k] - p]++] = i;
    for (int q = 0; q < ng; ++q)
      for (int k = c.rp[p + q]; k < c.rp[p + q + 1]; ++k)
        if (c.ci[k] < p) att[pos[q]++] = c.ci[k];
  }
  std::vector<int64_t> alen(ng);
  for (int q = 0; q < ng; ++q) {
    auto b = att.begin() + aoff[q], e = att.begin() + aoff[q + 1];
    std::sort(b, e);
    alen[q] = std::unique(b, e) - b;
  }

  // Enriched graph: (1,1) pattern plus cliques of first-block nodes sharing
  // a second-block column (partitioned_matrix.cpp:104-140), symmetrised.
  Graph g;
  g.n = p;
  std::vector<int64_t> cnt(p + 1, 0);
  for (int i = 0; i < p; ++i)
    for (int k = c.rp[i]; k < c.rp[i + 1]; ++k) {
      const int j = c.ci[k];
      if (j < p && j != i) {
        ++cnt[i + 1];
        ++cnt[j + 1];
      }
    }
  for (int q = 0; q < ng; ++q) {
    const int64_t m = alen[q];
    for (int64_t a = 0; a < m; ++a) cnt[att[aoff[q] + a] + 1] += m - 1;
  }
  for (int i = 0; i < p; ++i) cnt[i + 1] += cnt[i];
  std::vector<int> raw(cnt[p]);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int i = 0; i < p; ++i)
      for (int k = c.rp[i]; k < c.rp[i + 1]; ++k) {
        const int j = c.ci[k];
        if (j < p && j != i) {
          raw[pos[i]++] = j;
          raw[pos[j]++] = i;
        }
      }
    for (int q = 0; q < ng; ++q) {
      const int64_t m = alen[q];
      const int* nodes = att.data() + aoff[q];
      for (int64_t a = 0; a < m; ++a)
        for (int64_t b = 0; b < m; ++b)
          if (a != b) raw[pos[nodes[a]]++] = nodes[b];
    }
  }
  std::vector<int> ulen(p);
  parallel_for((p + 65535) / 65536, threads, [&](int chunk, int) {
    const int lo = chunk * 65536, hi = std::min(p, lo + 65536);
    for (int i = lo; i < hi; ++i) {
      auto b = raw.begin() + cnt[i], e = raw.begin() + cnt[i + 1];
      std::sort(b, e);
      ulen[i] = static_cast<int>(std::unique(b, e) - b);
    }
  });
  g.off.assign(p + 1, 0);
  for (int i = 0; i < p; ++i) g.off[i + 1] = g.off[i] + ulen[i];
  g.adj.resize(g.off[p]);
  for (int i = 0; i < p; ++i)
    std::copy(raw.begin() + cnt[i], raw.begin() + cnt[i] + ulen[i], g.adj.begin() + g.off[i]);
  std::vector<int>().swap(raw);

  static const bool verbose = getenv("MSCG_VERBOSE") != nullptr;
  const auto tg = std::chrono::steady_clock::now();
  if (verbose)
    fprintf(stderr, "partition_saddle: enriched graph %d nodes, %lld edges, %.3f s\n", p,
            static_cast<long long>(g.off[p]),
            std::chrono::duration<double>(tg - t_start).count());
  std::vector<std::vector<int>> blocks;
  std::vector<int> separator;
  if (dissect)
    dissect(g.n, g.off.data(), g.adj.data(), target_blocks, blocks, separator);
  else
    nested_dissection(g, target_blocks, threads, blocks, separator);
  const auto tn = std::chrono::steady_clock::now();

  // Second-block unknowns follow their interior couplings
  // (partitioned_matrix.cpp:146-175).
  const int nblocks = static_cast<int>(blocks.size());
  std::vector<int> owner(p, -1);
  for (int b = 0; b < nblocks; ++b)
    for (int u : blocks[b]) owner[u] = b;
  for (auto& b : blocks) std::sort(b.begin(), b.end());
  std::vector<std::vector<int>> tail(nblocks);
  std::vector<int> g_side;
  for (int q = 0; q < ng; ++q) {
    int blk = -1;
    for (int64_t a = 0; a < alen[q]; ++a) {
      const int v = att[aoff[q] + a];
      if (owner[v] >= 0) {
        blk = owner[v];
        break;
      }
    }
    (blk < 0 ? g_side : tail[blk]).push_back(p + q);
  }

  Partitioned out;
  std::vector<int> fwd;
  fwd.reserve(n);
  for (int b = 0; b < nblocks; ++b) {
    const int begin = static_cast<int>(fwd.size());
    fwd.insert(fwd.end(), blocks[b].begin(), blocks[b].end());
    fwd.insert(fwd.end(), tail[b].begin(), tail[b].end());
    out.d_ranges.push_back({begin, static_cast<int>(fwd.size())});
  }
  out.p = static_cast<int>(fwd.size());
  fwd.insert(fwd.end(), separator.begin(), separator.end());
  fwd.insert(fwd.end(), g_side.begin(), g_side.end());
  out.separator_size = static_cast<int>(separator.size());
  std::vector<int> inv(n, -1);
  for (int k = 0; k < n; ++k) {
    if (fwd[k] < 0 || fwd[k] >= n || inv[fwd[k]] != -1)
      throw std::runtime_error("partition_saddle: forward map is not a bijection");
    inv[fwd[k]] = k;
  }
  out.C = permute_symmetric(c, fwd, inv);
  out.perm = std::move(fwd);

  // Block-diagonal invariant (partitioned_matrix.cpp:197-201).
  std::vector<int> bown(out.p, -1);
  for (int b = 0; b < nblocks; ++b)
    for (int i = out.d_ranges[b].first; i < out.d_ranges[b].second; ++i) bown[i] = b;
  int64_t bad = 0;
  for (int i = 0; i < out.p; ++i)
    for (int k = out.C.rp[i]; k < out.C.rp[i + 1]; ++k) {
      const int j = out.C.ci[k];
      if (j < out.p && bown[i] != bown[j]) ++bad;
    }
  if (bad)
    throw std::runtime_error("partition_saddle: interior blocks remained coupled (" +
                             std::to_string(bad) + " entries)");
  if (verbose)
    fprintf(stderr, "partition_saddle: dissection %.3f s, permutation %.3f s\n",
            std::chrono::duration<double>(tn - tg).count(),
            std::chrono::duration<double>(std::chrono::steady_clock::now() - tn).count());
  return out;
}

void anchor_interface(Partitioned& pm) {
  const int n = pm.n(), p = pm.p, ng = pm.n_g(), nsep = pm.separator_size;
  std::vector<std::vector<int>> after(nsep);
  std::vector<int> rest;
  for (int q = nsep; q < ng; ++q) {
    int best = -1;
    for (int k = pm.C.rp[p + q]; k < pm.C.rp[p + q + 1]; ++k) {
      const int c = pm.C.ci[k] - p;
      if (c >= 0 && c < nsep) {
        best = c;  // columns sorted: first interface-velocity column is smallest
        break;
      }
    }
    (best >= 0 ? after[best] : rest).push_back(q);
  }
  std::vector<int> fwd(n);
  for (int i = 0; i < p; ++i) fwd[i] = i;
  int w = p;
  for (int v = 0; v < nsep; ++v) {
    fwd[w++] = p + v;
    for (int q : after[v]) fwd[w++] = p + q;
  }
  for (int q : rest) fwd[w++] = p + q;
  std::vector<int> inv(n);
  for (int k = 0; k < n; ++k) inv[fwd[k]] = k;
  pm.C = permute_symmetric(pm.C, fwd, inv);
  std::vector<int> composed(n);
  for (int k = 0; k < n; ++k) composed[k] = pm.perm[fwd[k]];
  pm.perm = std::move(composed);
}

}  // namespace mscg::host
