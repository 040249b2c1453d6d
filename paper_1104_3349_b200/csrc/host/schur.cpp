// Host problem layer, part 3: aggregates over the interface numbering and
// the mini-Schur-complement approximation S^ (setup, once).
//
//   equal_sizes              proj/src/aggregates.cpp:132-141
//   aggregate_by_numbering   proj/src/aggregates.cpp:36-48
//   build_msc (MSCN/MSCNR/LUM, numbering aggregates)
//                            proj/src/schur_approx.cpp:88-161
// MSCN/MSCNR need an exact LU of each aggregate's D-side companion block;
// that is done here with the reference's dense LU (dense_matrix.cpp:85-123)
// and sparse multi-RHS triangular solve (factorization.cpp:160-199), in the
// reference's operation order, so S^ is bit-identical.  This is setup work
// over blocks of size sz; the device path starts at the factorisation of
// the interior blocks and of S^ (csrc/device/).
#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <thread>

#include "setup.hpp"

namespace mscg::host {

std::vector<int> equal_sizes(int n_g, int sz) {
  if (sz < 1 || n_g < 1) throw std::invalid_argument("equal_sizes: sz and n_g must be positive");
  sz = std::min(sz, n_g);
  const int k = std::max(1, n_g / sz);
  std::vector<int> sizes(k, sz);
  sizes.back() = n_g - sz * (k - 1);
  return sizes;
}

std::vector<int> anchored_sizes(const Partitioned& pm, int sz) {
  const int ng = pm.n_g(), p = pm.p;
  if (sz <= 0) sz = std::max(1, ng / 8);
  std::vector<char> is_p(ng, 0);
  for (int q = 0; q < ng; ++q) {
    bool diag = false;
    for (int k = pm.C.rp[p + q]; k < pm.C.rp[p + q + 1]; ++k)
      if (pm.C.ci[k] == p + q) {
        diag = true;
        break;
      }
    is_p[q] = !diag;
  }
  std::vector<int> sizes;
  int cur = 0;
  for (int q = 0; q < ng; ++q) {
    ++cur;
    const bool next_is_p = (q + 1 < ng) && is_p[q + 1];
    if (cur >= sz && !next_is_p && q + 1 < ng) {
      sizes.push_back(cur);
      cur = 0;
    }
  }
  if (cur > 0) sizes.push_back(cur);
  return sizes;
}

Variant variant_from_name(const std::string& name) {
  if (name == "mscn") return Variant::Mscn;
  if (name == "mscnr") return Variant::Mscnr;
  if (name == "lum") return Variant::Lum;
  if (name == "omscn") return Variant::Omscn;
  if (name == "omscnr") return Variant::Omscnr;
  if (name == "olum") return Variant::Olum;
  throw std::invalid_argument("unknown or unsupported MSC variant: " + name);
}

bool variant_overlapped(Variant v) {
  return v == Variant::Omscn || v == Variant::Omscnr || v == Variant::Olum;
}
bool variant_rowsum(Variant v) { return v == Variant::Mscnr || v == Variant::Omscnr; }
bool variant_lumped(Variant v) { return v == Variant::Lum || v == Variant::Olum; }

static const char* variant_str(Variant v) {
  switch (v) {
    case Variant::Mscn: return "mscn";
    case Variant::Mscnr: return "mscnr";
    case Variant::Lum: return "lum";
    case Variant::Omscn: return "omscn";
    case Variant::Omscnr: return "omscnr";
    case Variant::Olum: return "olum";
  }
  return "?";
}

std::vector<int> overlap_widths(int n_g, const std::vector<int>& sizes, int sz, int overlap) {
  std::vector<int> w(sizes.size(), overlap < 0 ? sz : overlap);
  if (!w.empty()) w.back() = 0;
  int end = 0;
  for (size_t i = 0; i < w.size(); ++i) {
    end += sizes[i];
    int bound = std::min(sizes[i] - 1, n_g - end);
    if (i + 1 == w.size()) bound = 0;
    w[i] = std::min(w[i], bound);
  }
  return w;
}

void aggregate_spans(const Partitioned& pm, const std::vector<int>& sizes, Variant v,
                     const std::vector<int>& widths, std::vector<std::pair<int, int>>& ranges,
                     std::vector<std::pair<int, int>>& spans) {
  const int ng = pm.n_g(), p = pm.p;
  int total = 0;
  for (int s : sizes) {
    if (s < 1) throw std::invalid_argument("aggregates: sizes must be >= 1");
    total += s;
  }
  if (sizes.empty() || total != ng)
    throw std::invalid_argument("aggregates: sizes sum to " + std::to_string(total) +
                                ", expected " + std::to_string(ng));
  ranges.clear();
  spans.clear();
  int b = 0;
  for (int s : sizes) {
    ranges.push_back({b, b + s});
    b += s;
  }
  const int k = static_cast<int>(sizes.size());
  const bool have = !widths.empty();
  if (have) {  // aggregate_overlapped (aggregates.cpp:50-85)
    if (static_cast<int>(widths.size()) != k)
      throw std::invalid_argument("aggregate_overlapped: one width per aggregate");
    for (int i = 0; i < k; ++i) {
      const int w = widths[i];
      if (w < 0 || (i + 1 == k && w != 0))
        throw std::invalid_argument("aggregate_overlapped: widths must be >= 0 and end with 0");
      if (w >= sizes[i])
        throw std::invalid_argument("aggregate_overlapped: width " + std::to_string(w) +
                                    " of aggregate " + std::to_string(i) + " violates w < size");
      if (ranges[i].second + w > ng)
        throw std::invalid_argument("aggregate_overlapped: overlapped span of aggregate " +
                                    std::to_string(i) + " exceeds the block");
    }
  }
  // check_agg_compatible (schur_approx.cpp:56-85)
  const bool want = variant_overlapped(v);
  if (want != have)
    throw std::invalid_argument(std::string("build_msc: variant ") + variant_str(v) +
                                (want ? " needs an overlapped aggregate set"
                                      : " needs a non-overlapped aggregate set"));
  for (int i = 0; i < k; ++i) spans.push_back({ranges[i].first, ranges[i].second + (have ? widths[i] : 0)});
  if (!variant_lumped(v)) {
    for (int i = 0; i < k; ++i)
      if (spans[i].second > p)
        throw std::invalid_argument("build_msc: aggregate " + std::to_string(i) +
                                    " has a D-side index outside the (1,1) block");
  }
}

Csr merge_msc(int ng, const std::vector<std::pair<int, int>>& ranges,
              const std::vector<std::pair<int, int>>& spans,
              const std::vector<const double*>& local) {
  // Row r collects, for every aggregate whose span holds r (a contiguous
  // run of aggregates ending at r's owner), that aggregate's owned columns
  // in ascending order: the row-major order from_triplets sorts into.
  Csr s(ng, ng);
  const int k = static_cast<int>(ranges.size());
  int own = 0;
  for (int r = 0; r < ng; ++r) {
    while (own + 1 < k && ranges[own].second <= r) ++own;
    int first = own;
    while (first > 0 && spans[first - 1].second > r) --first;
    for (int i = first; i <= own; ++i) {
      const auto [sb, se] = spans[i];
      if (r < sb || r >= se) continue;
      const int m = se - sb;
      const double* a = local[i];
      for (int c = ranges[i].first; c < ranges[i].second; ++c) {
        const double v = a[static_cast<size_t>(r - sb) * m + (c - sb)];
        if (v != 0.0) {
          s.ci.push_back(c);
          s.v.push_back(v);
        }
      }
    }
    s.rp[r + 1] = static_cast<int>(s.ci.size());
  }
  return s;
}

namespace {

struct Dense {
  int r = 0, c = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
};

// A[rows, cols] for a contiguous row range and a contiguous column range
// (extract_submatrix, sparse_matrix.cpp:146-172, for numbering aggregates).
Dense dense_range(const Csr& a, int rb, int re, int cb, int ce) {
  Dense d(re - rb, ce - cb);
  for (int i = rb; i < re; ++i)
    for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
      if (a.ci[k] >= cb && a.ci[k] < ce) d(i - rb, a.ci[k] - cb) = a.v[k];
  return d;
}

struct SparseRows {
  std::vector<std::vector<std::pair<int, double>>> rows;
};

struct LuFactors {
  SparseRows L, U;
  std::vector<int> perm;
};

// dense_lu (dense_matrix.cpp:85-123) re-stored sparse (factorization.cpp:11-32).
LuFactors factor_exact(Dense a, int agg) {
  const int n = a.r;
  LuFactors f;
  f.perm.resize(n);
  for (int i = 0; i < n; ++i) f.perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = std::abs(a(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a(i, k)) > best) {
        best = std::abs(a(i, k));
        piv = i;
      }
    if (best == 0.0)
      throw SingularError("build_msc: singular D block of aggregate " + std::to_string(agg) +
                              " (dense_lu: zero pivot at index " + std::to_string(k) + ")",
                          k);
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(a(k, j), a(piv, j));
      std::swap(f.perm[k], f.perm[piv]);
    }
    const double pivot = a(k, k);
    for (int i = k + 1; i < n; ++i) {
      const double lik = a(i, k) / pivot;
      a(i, k) = lik;
      if (lik == 0.0) continue;
      for (int j = k + 1; j < n; ++j) a(i, j) -= lik * a(k, j);
    }
  }
  f.L.rows.resize(n);
  f.U.rows.resize(n);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < i; ++j)
      if (a(i, j) != 0.0) f.L.rows[i].push_back({j, a(i, j)});
    for (int j = i; j < n; ++j)
      if (a(i, j) != 0.0) f.U.rows[i].push_back({j, a(i, j)});
  }
  return f;
}

// Multi-RHS solve (factorization.cpp:160-199).
Dense solve(const LuFactors& f, const Dense& b) {
  const int n = b.r, m = b.c;
  Dense x(n, m);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) x(i, j) = b(f.perm[i], j);
  for (int i = 0; i < n; ++i)
    for (auto [c, lik] : f.L.rows[i])
      for (int j = 0; j < m; ++j) x(i, j) -= lik * x(c, j);
  for (int i = n - 1; i >= 0; --i) {
    double diag = 0.0;
    for (auto [c, uik] : f.U.rows[i]) {
      if (c == i) {
        diag = uik;
        continue;
      }
      for (int j = 0; j < m; ++j) x(i, j) -= uik * x(c, j);
    }
    for (int j = 0; j < m; ++j) x(i, j) /= diag;
  }
  return x;
}

}  // namespace

SchurApprox build_msc(const Partitioned& pm, const std::vector<int>& sizes, Variant v,
                      int threads, const std::vector<int>& widths) {
  const int ng = pm.n_g(), p = pm.p;
  SchurApprox out;
  aggregate_spans(pm, sizes, v, widths, out.ranges, out.spans);
  out.overlapped = variant_overlapped(v);
  const int k = static_cast<int>(sizes.size());
  std::vector<Dense> local(k);
  if (threads <= 0) threads = hardware_threads();
  std::atomic<int> next{0};
  std::exception_ptr err;
  std::mutex err_mu;
  int err_idx = k;
  auto work = [&] {
    for (int i = next++; i < k; i = next++) {
      try {
        const auto [sb, se] = out.spans[i];
        const int m = se - sb;
        // G = C[p:, p:]; D = C[:p, :p]; E = C[:p, p:]; F = C[p:, :p].
        Dense s = dense_range(pm.C, p + sb, p + se, p + sb, p + se);
        if (!variant_lumped(v)) {
          LuFactors dlu = factor_exact(dense_range(pm.C, sb, se, sb, se), i);
          Dense e = dense_range(pm.C, sb, se, p + sb, p + se);
          Dense rhs;
          if (variant_rowsum(v)) {
            // E_ii compressed to diag(E_ii * 1) (schur_approx.cpp:112-126).
            rhs = Dense(m, m);
            for (int r = 0; r < m; ++r) {
              double acc = 0.0;
              for (int t = pm.C.rp[sb + r]; t < pm.C.rp[sb + r + 1]; ++t) {
                const int c = pm.C.ci[t];
                if (c >= p + sb && c < p + se) acc += pm.C.v[t] * 1.0;
              }
              rhs(r, r) = acc;
            }
          } else {
            rhs = std::move(e);
          }
          Dense x = solve(dlu, rhs);
          // correction = F_ii x (dense_matrix.cpp:62-77), then S - correction.
          Dense corr(m, m);
          for (int r = 0; r < m; ++r)
            for (int t = pm.C.rp[p + sb + r]; t < pm.C.rp[p + sb + r + 1]; ++t) {
              const int c = pm.C.ci[t];
              if (c < sb || c >= se) continue;
              const double aik = pm.C.v[t];
              for (int j = 0; j < m; ++j) corr(r, j) += aik * x(c - sb, j);
            }
          for (size_t t = 0; t < s.a.size(); ++t) s.a[t] = s.a[t] - corr.a[t];
        }
        local[i] = std::move(s);
      } catch (...) {
        // Deterministic: report the lowest failing aggregate, as the
        // reference's sequential build_msc (workers = 1) does.
        std::lock_guard<std::mutex> lk(err_mu);
        if (i < err_idx) {
          err_idx = i;
          err = std::current_exception();
        }
      }
    }
  };
  {
    std::vector<std::thread> pool;
    const int t = std::max(1, std::min(threads, k));
    for (int w = 1; w < t; ++w) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  }
  if (err) std::rethrow_exception(err);

  // Sequential merge (schur_approx.cpp:141-160).
  std::vector<const double*> lp(k);
  for (int i = 0; i < k; ++i) lp[i] = local[i].a.data();
  out.s_hat = merge_msc(ng, out.ranges, out.spans, lp);
  return out;
}

}  // namespace mscg::host
