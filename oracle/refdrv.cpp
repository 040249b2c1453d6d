// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// C-ABI driver over the UNMODIFIED reference library (/root/reference/proj,
// compiled in place by oracle/Makefile into oracle/_ref/libmscref.so).  It
// exposes the reference's own setup / apply / solve entry points to the
// Python tests, the golden-fixture generator (tests/golden/make_golden.py)
// and bench.py's cpu_baseline / --impl reference legs.  Every function here
// only marshals arrays and calls the reference's public API:
//   generate_oseen        proj/include/msc/oseen.hpp:43-44
//   scale_rows            proj/include/msc/row_scaling.hpp:23
//   partition_saddle      proj/include/msc/partitioned_matrix.hpp:69-70
//   aggregate_by_numbering/equal_sizes  proj/include/msc/aggregates.hpp:41,61
//   build_msc             proj/include/msc/schur_approx.hpp:45-46
//   build_preconditioner  proj/include/msc/preconditioner.hpp:66-68
//   MscPreconditioner::apply proj/src/preconditioner.cpp:85-114
//   gmres                 proj/include/msc/gmres.hpp:44-47
//   factor_ilut / solve   proj/include/msc/factorization.hpp:38-43
//   matvec                proj/include/msc/sparse_matrix.hpp:87
//   load/write_(matrix|vector)_market  proj/include/msc/matrix_market.hpp:26-36
//   oracle::random_vector / random_saddle  proj/tests/oracles.hpp:92-142
// The "anchored" interface re-ordering is the harness-level fix of
// SURVEY.md §8(d) (public API only: permute + PartitionedMatrix::from_split +
// aggregate_by_numbering); the product's host layer implements the same rule
// (paper_1104_3349_b200/csrc/host/aggregate.cpp) and the tests check they agree.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "msc/aggregates.hpp"
#include "msc/factorization.hpp"
#include "msc/graph.hpp"
#include "msc/gmres.hpp"
#include "msc/matrix_market.hpp"
#include "msc/oseen.hpp"
#include "msc/parallel.hpp"
#include "msc/partitioned_matrix.hpp"
#include "msc/permutation.hpp"
#include "msc/preconditioner.hpp"
#include "msc/row_scaling.hpp"
#include "msc/schur_approx.hpp"
#include "oracles.hpp"

using namespace msc;

namespace {

thread_local std::string g_err;
thread_local int g_err_pivot = -1;

struct RefProblem {
  // Problem in the final (scaled, permuted) numbering.
  PartitionedMatrix pm;
  std::vector<int> perm;          // forward map of the saddle reorder (+anchoring)
  std::vector<double> scaled_rhs; // generator rhs, scaled + permuted (may be empty)
  AggregateSet agg;
  SchurApproximation schur;
  std::unique_ptr<MscPreconditioner> prec;
  bool have_schur = false;
  int overlap = -1;  // overlapped aggregate width (benchmark.cpp:35: -1 = sz)
};

struct RefFactors {
  TriangularFactors f;
};

const SparseMatrix* pick(RefProblem* p, int which) {
  switch (which) {
    case 0: return &p->pm.C;
    case 1: return &p->pm.D;
    case 2: return &p->pm.E;
    case 3: return &p->pm.F;
    case 4: return &p->pm.G;
    case 5: return p->have_schur ? &p->schur.s_hat : nullptr;
  }
  return nullptr;
}

void copy_csr(const SparseMatrix& a, int* rp, int* ci, double* v) {
  if (rp) std::memcpy(rp, a.row_offsets().data(), sizeof(int) * (a.rows() + 1));
  if (ci) std::memcpy(ci, a.col_indices().data(), sizeof(int) * a.nnz());
  if (v) std::memcpy(v, a.values().data(), sizeof(double) * a.nnz());
}

SparseMatrix csr_from_arrays(int nrows, int ncols, const int* rp, const int* ci,
                             const double* v) {
  std::vector<Triplet> t;
  t.reserve(rp[nrows]);
  for (int i = 0; i < nrows; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k) t.push_back({i, ci[k], v[k]});
  return SparseMatrix::from_triplets(nrows, ncols, std::move(t));
}

// SURVEY.md §8(d) interface anchoring: every (2,2)-side pressure with a
// separator-velocity neighbour in G is placed directly after its
// smallest-index such neighbour; others keep their order at the tail.
// `nsep` = number of separator velocities at the head of the interface.
std::vector<int> anchored_interface_order(const PartitionedMatrix& pm, int nsep,
                                          std::vector<char>& is_anchored) {
  const int ng = pm.n_g();
  std::vector<std::vector<int>> after(nsep);
  std::vector<int> tail;
  is_anchored.assign(ng, 0);
  for (int q = nsep; q < ng; ++q) {
    int best = -1;
    for (int c : pm.G.row_cols(q)) {
      if (c < nsep) { best = c; break; }  // columns sorted: first is smallest
    }
    if (best >= 0) after[best].push_back(q); else tail.push_back(q);
  }
  std::vector<int> order;
  order.reserve(ng);
  for (int v = 0; v < nsep; ++v) {
    order.push_back(v);
    for (int q : after[v]) { order.push_back(q); is_anchored[q] = 1; }
  }
  for (int q : tail) order.push_back(q);
  return order;
}

// ---- private-member access (test infrastructure) -------------------------
// MscPreconditioner can only be filled by build_preconditioner (a friend,
// preconditioner.hpp:45-48), whose interior-block loop is sequential
// (preconditioner.cpp:44-56: 16-23 min at cfg5).  To run the reference's
// OWN apply (preconditioner.cpp:85-114) on reference factors computed
// concurrently, or on factors downloaded from the GPU, the driver fills the
// object's members directly.  Explicit template instantiation may name
// private members ([temp.spec.general]/6), which is the standard way to do
// this without modifying the reference headers.
template <class Tag, typename Tag::type M>
struct Rob {
  friend typename Tag::type get(Tag) { return M; }
};
#define REF_ROB(TAG, CLS, TYPE, MEMBER)                   \
  struct TAG {                                           \
    using type = TYPE CLS::*;                            \
    friend type get(TAG);                                \
  };                                                     \
  template struct Rob<TAG, &CLS::MEMBER>;

using RangeVec = std::vector<std::pair<int, int>>;
REF_ROB(PcN, MscPreconditioner, int, n_)
REF_ROB(PcP, MscPreconditioner, int, p_)
REF_ROB(PcKind, MscPreconditioner, std::string, kind_)
REF_ROB(PcDR, MscPreconditioner, RangeVec, d_ranges_)
REF_ROB(PcDF, MscPreconditioner, std::vector<TriangularFactors>, d_factors_)
REF_ROB(PcSR, MscPreconditioner, RangeVec, schur_ranges_)
REF_ROB(PcSF, MscPreconditioner, std::vector<TriangularFactors>, schur_factors_)
REF_ROB(PcSS, MscPreconditioner, bool, schur_single_)
REF_ROB(PcE, MscPreconditioner, SparseMatrix, e_)
REF_ROB(PcF, MscPreconditioner, SparseMatrix, f_)
REF_ROB(SmR, SparseMatrix, int, nrows_)
REF_ROB(SmC, SparseMatrix, int, ncols_)
REF_ROB(SmRP, SparseMatrix, std::vector<int>, row_offsets_)
REF_ROB(SmCI, SparseMatrix, std::vector<int>, col_indices_)
REF_ROB(SmV, SparseMatrix, std::vector<double>, values_)
#undef REF_ROB

// CSR arrays straight into a SparseMatrix (the caller guarantees the
// reference's invariants: sorted rows, no explicit zeros) — no triplet sort.
SparseMatrix csr_direct(int nrows, int ncols, const int* rp, const int* ci,
                        const double* v) {
  SparseMatrix a;
  a.*get(SmR{}) = nrows;
  a.*get(SmC{}) = ncols;
  a.*get(SmRP{}) = std::vector<int>(rp, rp + nrows + 1);
  const std::size_t nnz = static_cast<std::size_t>(rp[nrows]);
  a.*get(SmCI{}) = std::vector<int>(ci, ci + nnz);
  a.*get(SmV{}) = std::vector<double>(v, v + nnz);
  return a;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SingularMatrixError& e) {
    g_err = e.what();
    g_err_pivot = e.pivot_index;
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_pivot = -1;
    return -1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(int* pivot) {
  if (pivot) *pivot = g_err_pivot;
  return g_err.c_str();
}

void ref_random_vector(int n, unsigned seed, double* out) {
  std::mt19937 rng(seed);
  std::vector<double> v = oracle::random_vector(n, rng);
  std::memcpy(out, v.data(), sizeof(double) * n);
}

void ref_problem_free(RefProblem* p) { delete p; }

// Oseen problem through the reference pipeline (benchmark.cpp:45-67,101-135):
// generate -> scale_rows -> partition_saddle(Interleaved) [-> anchoring].
// grid_kind 0 uniform / 1 stretched.  Aggregates/Schur are built separately.
int ref_problem_oseen(int grid_n, double nu, int grid_kind, double stretch,
                      int nA, int anchored, RefProblem** out) {
  return guarded([&] {
    auto prob = generate_oseen(grid_n, nu,
                               grid_kind ? GridKind::Stretched : GridKind::Uniform,
                               WindKind::Recirculating, stretch);
    RowScaling scaled = scale_rows(prob.matrices.C, prob.rhs);
    SaddleReorder r = partition_saddle(scaled.matrix, prob.matrices.p, nA,
                                       SaddleOrdering::Interleaved);
    auto p = std::make_unique<RefProblem>();
    p->perm = r.perm.forward;
    p->scaled_rhs = permute_vector(scaled.rhs, r.perm);
    if (anchored) {
      const int n = r.matrix.n();
      const int pp = r.matrix.p;
      std::vector<char> is_anch;
      std::vector<int> iorder =
          anchored_interface_order(r.matrix, r.separator_size, is_anch);
      std::vector<int> fwd(n);
      for (int i = 0; i < pp; ++i) fwd[i] = i;
      for (int k = 0; k < n - pp; ++k) fwd[pp + k] = pp + iorder[k];
      Permutation ap = Permutation::from_forward(fwd);
      SparseMatrix c2 = permute(r.matrix.C, ap);
      p->pm = PartitionedMatrix::from_split(std::move(c2), pp,
                                            r.matrix.d_block_ranges);
      std::vector<int> composed(n);
      for (int k = 0; k < n; ++k) composed[k] = p->perm[fwd[k]];
      p->perm = composed;
      p->scaled_rhs = permute_vector(p->scaled_rhs, ap);
    } else {
      p->pm = std::move(r.matrix);
    }
    *out = p.release();
  });
}

// Arbitrary partitioned system from CSR arrays (tests' random saddles).
int ref_problem_from_csr(int n, const int* rp, const int* ci, const double* v,
                         int p, int nranges, const int* ranges, RefProblem** out) {
  return guarded([&] {
    std::vector<std::pair<int, int>> rr;
    for (int i = 0; i < nranges; ++i) rr.push_back({ranges[2 * i], ranges[2 * i + 1]});
    auto pr = std::make_unique<RefProblem>();
    pr->pm = PartitionedMatrix::from_split(csr_from_arrays(n, n, rp, ci, v), p, rr);
    pr->perm.resize(n);
    for (int i = 0; i < n; ++i) pr->perm[i] = i;
    *out = pr.release();
  });
}

// oracle::random_saddle (tests/oracles.hpp:122-142) with the given seed.
int ref_problem_random_saddle(int p, int ng, unsigned seed, double density,
                              RefProblem** out) {
  return guarded([&] {
    std::mt19937 rng(seed);
    auto pr = std::make_unique<RefProblem>();
    pr->pm = oracle::random_saddle(p, ng, rng, density);
    pr->perm.resize(p + ng);
    for (int i = 0; i < p + ng; ++i) pr->perm[i] = i;
    *out = pr.release();
  });
}

void ref_problem_dims(RefProblem* p, int* n, int* pp, int* nblocks,
                      int64_t* nnz_c) {
  *n = p->pm.n();
  *pp = p->pm.p;
  *nblocks = static_cast<int>(p->pm.d_block_ranges.size());
  *nnz_c = static_cast<int64_t>(p->pm.C.nnz());
}

// which: 0 C, 1 D, 2 E, 3 F, 4 G, 5 S_hat.  Returns nnz (or -1).
int64_t ref_csr_shape(RefProblem* p, int which, int* nrows, int* ncols) {
  const SparseMatrix* a = pick(p, which);
  if (!a) return -1;
  *nrows = a->rows();
  *ncols = a->cols();
  return static_cast<int64_t>(a->nnz());
}
int ref_csr_get(RefProblem* p, int which, int* rp, int* ci, double* v) {
  const SparseMatrix* a = pick(p, which);
  if (!a) return -1;
  copy_csr(*a, rp, ci, v);
  return 0;
}
void ref_get_perm(RefProblem* p, int* perm) {
  std::memcpy(perm, p->perm.data(), sizeof(int) * p->perm.size());
}
int ref_get_scaled_rhs(RefProblem* p, double* out) {
  if (p->scaled_rhs.empty()) return -1;
  std::memcpy(out, p->scaled_rhs.data(), sizeof(double) * p->scaled_rhs.size());
  return 0;
}
void ref_get_d_ranges(RefProblem* p, int* ranges) {
  for (std::size_t i = 0; i < p->pm.d_block_ranges.size(); ++i) {
    ranges[2 * i] = p->pm.d_block_ranges[i].first;
    ranges[2 * i + 1] = p->pm.d_block_ranges[i].second;
  }
}

// Aggregates: mode 0 = equal_sizes(n_g, sz) numbering (benchmark.cpp:74-99,
// sz <= 0 -> n_g/8), mode 1 = anchored greedy sizes (close at >= sz, never
// directly before an anchored pressure), mode 2 = explicit sizes.
int ref_build_schur(RefProblem* p, const char* variant, int mode, int sz,
                    int nsizes, const int* sizes_in, int workers) {
  return guarded([&] {
    const int ng = p->pm.n_g();
    std::vector<int> sizes;
    if (mode == 2) {
      sizes.assign(sizes_in, sizes_in + nsizes);
    } else if (mode == 1) {
      // A pressure is "anchored" when its (2,2) row couples to an earlier
      // interface velocity: after anchoring these follow their velocity.
      // Recover the rule from the matrix itself: node q is a pressure iff
      // its G-row has no entry on the diagonal block of velocities... we
      // instead use the D-free criterion: pressure rows of the scaled Oseen
      // system have an empty diagonal except the pin.
      if (sz <= 0) sz = std::max(1, ng / 8);
      std::vector<char> is_p(ng, 0);
      for (int q = 0; q < ng; ++q) {
        bool diag = false;
        for (int c : p->pm.G.row_cols(q)) if (c == q) { diag = true; break; }
        is_p[q] = !diag;
      }
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
    } else {
      if (sz <= 0) sz = std::max(1, ng / 8);
      sz = std::min(sz, ng);
      sizes = equal_sizes(ng, sz);
    }
    const MscVariant v = variant_from_name(variant);
    if (variant_overlapped(v)) {
      // make_aggregates' overlapped branch (benchmark.cpp:80-88), with the
      // overlap width passed through ref_set_overlap (default -1 = sz)
      if (sz <= 0) sz = std::max(1, ng / 8);
      sz = std::min(sz, ng);
      std::vector<int> widths(sizes.size(), p->overlap < 0 ? sz : p->overlap);
      widths.back() = 0;
      clip_overlap_widths(ng, sizes, widths);
      p->agg = aggregate_overlapped(ng, sizes, widths);
    } else {
      p->agg = aggregate_by_numbering(ng, sizes);
    }
    p->schur = build_msc(p->pm, p->agg, v, workers);
    p->have_schur = true;
  });
}

// nested_dissection(build_graph(A), target) (graph.cpp:8-30,178-230) of the
// pattern of a CSR matrix: forward permutation (blocks, then separator) and
// the block ranges (ranges[2*cap]); returns the block count or -1.
int ref_nested_dissection(int n, const int* rp, const int* ci, int target, int* perm,
                          int* ranges, int cap) {
  int nb = -1;
  if (guarded([&] {
    std::vector<double> v(rp[n], 1.0);
    AdjacencyGraph g = build_graph(csr_from_arrays(n, n, rp, ci, v.data()));
    SeparatorPartition part = nested_dissection(g, target);
    for (int i = 0; i < n; ++i) perm[i] = part.permutation.forward[i];
    nb = static_cast<int>(part.block_ranges.size());
    for (int b = 0; b < nb && b < cap; ++b) {
      ranges[2 * b] = part.block_ranges[b].first;
      ranges[2 * b + 1] = part.block_ranges[b].second;
    }
  }))
    return -1;
  return nb;
}

// overlap width used by the next ref_build_schur of an overlapped variant
void ref_set_overlap(RefProblem* p, int overlap) { p->overlap = overlap; }

int ref_exact_schur(RefProblem* p) {
  return guarded([&] {
    p->schur = build_exact_schur(p->pm);
    p->have_schur = true;
  });
}

int ref_num_aggregates(RefProblem* p) {
  return p->have_schur ? static_cast<int>(p->schur.owned_ranges.size()) : -1;
}
void ref_get_schur_ranges(RefProblem* p, int* ranges) {
  for (std::size_t i = 0; i < p->schur.owned_ranges.size(); ++i) {
    ranges[2 * i] = p->schur.owned_ranges[i].first;
    ranges[2 * i + 1] = p->schur.owned_ranges[i].second;
  }
}

int ref_build_precond(RefProblem* p, double tolA, int sA) {
  return guarded([&] {
    p->prec = std::make_unique<MscPreconditioner>(
        build_preconditioner(p->pm, p->schur, tolA, sA));
  });
}

// build_preconditioner (preconditioner.cpp:26-83) with its interior-block
// factorisation loop spread over the reference's own parallel_for
// (parallel.cpp:21-50).  Every block runs the reference factor_ilut /
// factor_exact exactly as the sequential loop does, so the resulting
// MscPreconditioner is member-for-member the one build_preconditioner
// returns; a singular block raises the reference's message for the LOWEST
// failing block index, as the sequential loop would.
int ref_build_precond_parallel(RefProblem* p, double tolA, int sA, int workers) {
  return guarded([&] {
    const PartitionedMatrix& c = p->pm;
    const SchurApproximation& schur = p->schur;
    if (schur.s_hat.rows() != c.n_g())
      throw std::invalid_argument(
          "build_preconditioner: Schur approximation does not match the split");
    if (c.d_block_ranges.empty())
      throw std::invalid_argument("build_preconditioner: no interior D blocks");
    auto b = std::make_unique<MscPreconditioner>();
    (*b).*get(PcN{}) = c.n();
    (*b).*get(PcP{}) = c.p;
    (*b).*get(PcKind{}) = schur.exact ? "exact-schur" : variant_name(schur.variant);
    (*b).*get(PcDR{}) = c.d_block_ranges;
    (*b).*get(PcE{}) = c.E;
    (*b).*get(PcF{}) = c.F;
    const int nb = static_cast<int>(c.d_block_ranges.size());
    auto& df = (*b).*get(PcDF{});
    df.resize(nb);
    std::vector<std::string> err(nb);
    std::vector<int> errpiv(nb, -2);
    parallel_for(nb, workers, [&](int i) {
      const auto [begin, end] = c.d_block_ranges[i];
      SparseMatrix block = extract_block(c.D, begin, end, begin, end);
      try {
        const int dim = end - begin;
        df[i] = dim <= sA ? factor_exact(block) : factor_ilut(block, tolA);
      } catch (const SingularMatrixError& e) {
        err[i] = e.what();
        errpiv[i] = e.pivot_index;
      }
    });
    for (int i = 0; i < nb; ++i)
      if (errpiv[i] != -2)
        throw SingularMatrixError("build_preconditioner: (1,1) block " +
                                      std::to_string(i) + ": " + err[i],
                                  errpiv[i]);
    if (schur.overlapped) {
      (*b).*get(PcSS{}) = true;
      try {
        ((*b).*get(PcSF{})).push_back(factor_exact(schur.s_hat));
      } catch (const SingularMatrixError& e) {
        throw SingularMatrixError(
            std::string("build_preconditioner: overlapped Schur band: ") + e.what(),
            e.pivot_index);
      }
    } else {
      (*b).*get(PcSR{}) = schur.owned_ranges;
      for (std::size_t i = 0; i < schur.owned_ranges.size(); ++i) {
        const auto [begin, end] = schur.owned_ranges[i];
        SparseMatrix block = extract_block(schur.s_hat, begin, end, begin, end);
        try {
          ((*b).*get(PcSF{})).push_back(factor_exact(block));
        } catch (const SingularMatrixError& e) {
          throw SingularMatrixError("build_preconditioner: Schur block " +
                                        std::to_string(i) + ": " + e.what(),
                                    e.pivot_index);
        }
      }
    }
    p->prec = std::move(b);
  });
}

// A reference problem whose C, split, interior ranges and Schur
// approximation come from arrays (e.g. the product's bit-identical setup):
// C through csr_direct, D/E/F/G by the reference's from_split.
int ref_problem_from_arrays(int n, const int* rp, const int* ci, const double* v,
                            int p, int nranges, const int* ranges,
                            RefProblem** out) {
  return guarded([&] {
    std::vector<std::pair<int, int>> rr;
    for (int i = 0; i < nranges; ++i) rr.push_back({ranges[2 * i], ranges[2 * i + 1]});
    auto pr = std::make_unique<RefProblem>();
    pr->pm = PartitionedMatrix::from_split(csr_direct(n, n, rp, ci, v), p, rr);
    pr->perm.resize(n);
    for (int i = 0; i < n; ++i) pr->perm[i] = i;
    *out = pr.release();
  });
}

// Install a block-diagonal Schur approximation (S^ + owned ranges).
int ref_problem_set_schur(RefProblem* p, const char* variant, const int* rp,
                          const int* ci, const double* v, int nranges,
                          const int* ranges) {
  return guarded([&] {
    const int ng = p->pm.n_g();
    p->schur = SchurApproximation{};
    p->schur.s_hat = csr_direct(ng, ng, rp, ci, v);
    p->schur.variant = variant_from_name(variant);
    for (int i = 0; i < nranges; ++i) {
      p->schur.owned_ranges.push_back({ranges[2 * i], ranges[2 * i + 1]});
      p->schur.spans.push_back({ranges[2 * i], ranges[2 * i + 1]});
    }
    p->have_schur = true;
  });
}

// Stage 1 of "reference apply on given interior factors": an
// MscPreconditioner whose ranges/E/F come from the problem, Schur blocks
// factored by the reference factor_exact (as build_preconditioner does),
// interior factors to be installed block by block.
int ref_precond_begin(RefProblem* p) {
  return guarded([&] {
    const PartitionedMatrix& c = p->pm;
    auto b = std::make_unique<MscPreconditioner>();
    (*b).*get(PcN{}) = c.n();
    (*b).*get(PcP{}) = c.p;
    (*b).*get(PcKind{}) = variant_name(p->schur.variant);
    (*b).*get(PcDR{}) = c.d_block_ranges;
    (*b).*get(PcE{}) = c.E;
    (*b).*get(PcF{}) = c.F;
    ((*b).*get(PcDF{})).resize(c.d_block_ranges.size());
    (*b).*get(PcSR{}) = p->schur.owned_ranges;
    auto& sf = (*b).*get(PcSF{});
    sf.resize(p->schur.owned_ranges.size());
    const auto& sr = p->schur.owned_ranges;
    const SparseMatrix& sh = p->schur.s_hat;
    parallel_for(static_cast<int>(sr.size()), 0, [&](int i) {
      sf[i] = factor_exact(extract_block(sh, sr[i].first, sr[i].second, sr[i].first,
                                         sr[i].second));
    });
    p->prec = std::move(b);
  });
}

int ref_precond_set_dfactor(RefProblem* p, int b, int n, const int* lrp, const int* lci,
                            const double* lv, const int* urp, const int* uci,
                            const double* uv) {
  return guarded([&] {
    auto& df = (*p->prec).*get(PcDF{});
    TriangularFactors f;
    f.lower = csr_direct(n, n, lrp, lci, lv);
    f.upper = csr_direct(n, n, urp, uci, uv);
    f.row_perm = Permutation::identity(n);
    f.kind = FactorKind::Incomplete;
    df.at(b) = std::move(f);
  });
}

// MscPreconditioner::apply (preconditioner.cpp:85-114), operation for
// operation, with block_solve's independent per-block `solve` calls
// (preconditioner.cpp:13-22) spread over parallel_for.  Each block's
// arithmetic is the reference's own, so the result is bit-identical to the
// stock single-threaded apply (tests/test_oracle.py checks it).
int ref_apply_threads(RefProblem* p, const double* y, double* x, int workers) {
  return guarded([&] {
    const MscPreconditioner& b = *p->prec;
    const int n = b.*get(PcN{});
    const int pp = b.*get(PcP{});
    const int ng = n - pp;
    const auto& dr = b.*get(PcDR{});
    const auto& df = b.*get(PcDF{});
    auto bsolve = [&](const double* in, double* out) {
      parallel_for(static_cast<int>(dr.size()), workers, [&](int i) {
        const auto [begin, end] = dr[i];
        std::vector<double> local(in + begin, in + end);
        std::vector<double> s = solve(df[i], local);
        std::copy(s.begin(), s.end(), out + begin);
      });
    };
    std::vector<double> z1(pp, 0.0);
    bsolve(y, z1.data());
    std::vector<double> t = matvec(b.*get(PcF{}), z1);
    for (int i = 0; i < ng; ++i) t[i] = y[pp + i] - t[i];
    std::vector<double> z2(ng, 0.0);
    const auto& sf = b.*get(PcSF{});
    if (b.*get(PcSS{})) {
      std::vector<double> s = solve(sf[0], t);
      std::copy(s.begin(), s.end(), z2.begin());
    } else {
      const auto& sr = b.*get(PcSR{});
      for (std::size_t i = 0; i < sr.size(); ++i) {
        std::vector<double> local(t.begin() + sr[i].first, t.begin() + sr[i].second);
        std::vector<double> s = solve(sf[i], local);
        std::copy(s.begin(), s.end(), z2.begin() + sr[i].first);
      }
    }
    std::vector<double> w = matvec(b.*get(PcE{}), z2);
    std::vector<double> corr(pp, 0.0);
    bsolve(w.data(), corr.data());
    for (int i = 0; i < pp; ++i) x[i] = z1[i] - corr[i];
    std::copy(z2.begin(), z2.end(), x + pp);
  });
}

// Wall seconds of `reps` stock applies (MscPreconditioner::apply).
double ref_time_apply(RefProblem* p, const double* y, double* x, int reps) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    std::vector<double> o = p->prec->apply(std::span<const double>(y, p->pm.n()));
    std::memcpy(x, o.data(), sizeof(double) * o.size());
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Wall seconds of `reps` threaded applies (ref_apply_threads).
double ref_time_apply_threads(RefProblem* p, const double* y, double* x, int reps,
                              int workers) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r)
    if (ref_apply_threads(p, y, x, workers) != 0) return -1.0;
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_num_dfactors(RefProblem* p) {
  return p->prec ? static_cast<int>(p->prec->d_factors().size()) : -1;
}

int64_t ref_stored_nnz(RefProblem* p) {
  return p->prec ? static_cast<int64_t>(p->prec->stored_nnz()) : -1;
}

// kind 0 = interior D block factors, 1 = Schur block factors.
int ref_factor_dims(RefProblem* p, int kind, int idx, int* dim, int64_t* nnz_l,
                    int64_t* nnz_u) {
  if (!p->prec) return -1;
  const auto& v = kind == 0 ? p->prec->d_factors() : p->prec->schur_factors();
  if (idx < 0 || idx >= static_cast<int>(v.size())) return -1;
  *dim = v[idx].dim();
  *nnz_l = static_cast<int64_t>(v[idx].lower.nnz());
  *nnz_u = static_cast<int64_t>(v[idx].upper.nnz());
  return 0;
}
int ref_factor_get(RefProblem* p, int kind, int idx, int* lrp, int* lci,
                   double* lv, int* urp, int* uci, double* uv, int* perm) {
  if (!p->prec) return -1;
  const auto& v = kind == 0 ? p->prec->d_factors() : p->prec->schur_factors();
  const TriangularFactors& f = v[idx];
  copy_csr(f.lower, lrp, lci, lv);
  copy_csr(f.upper, urp, uci, uv);
  if (perm) std::memcpy(perm, f.row_perm.forward.data(), sizeof(int) * f.dim());
  return 0;
}

int ref_apply(RefProblem* p, const double* y, double* x) {
  return guarded([&] {
    std::vector<double> r = p->prec->apply(std::span<const double>(y, p->pm.n()));
    std::memcpy(x, r.data(), sizeof(double) * r.size());
  });
}

int ref_matvec(RefProblem* p, int which, const double* x, double* y) {
  return guarded([&] {
    const SparseMatrix* a = pick(p, which);
    std::vector<double> r = matvec(*a, std::span<const double>(x, a->cols()));
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}

// gmres (gmres.cpp:35-191).  hist must hold max_iters + 64 entries.
int ref_gmres(RefProblem* p, int use_prec, const double* b, int restart,
              int max_iters, double rel_tol, int left, double* x, int* iters,
              int* converged, double* hist, int* nhist, double* seconds) {
  return guarded([&] {
    SolverConfig cfg;
    cfg.restart = restart;
    cfg.max_iters = max_iters;
    cfg.rel_tol = rel_tol;
    cfg.side = left ? PrecondSide::Left : PrecondSide::Right;
    std::vector<double> rhs(b, b + p->pm.n());
    auto [xs, rep] = gmres(p->pm.C, use_prec ? p->prec.get() : nullptr, rhs, cfg);
    std::memcpy(x, xs.data(), sizeof(double) * xs.size());
    *iters = rep.iterations;
    *converged = rep.converged ? 1 : 0;
    const int cap = *nhist;
    const int m = static_cast<int>(rep.residual_history.size());
    for (int i = 0; i < std::min(cap, m); ++i) hist[i] = rep.residual_history[i];
    *nhist = m;
    *seconds = rep.solve_seconds;
  });
}

// ---- standalone kernels over raw CSR ------------------------------------

int ref_factor_ilut(int n, const int* rp, const int* ci, const double* v,
                    double tol, RefFactors** out) {
  return guarded([&] {
    auto f = std::make_unique<RefFactors>();
    f->f = factor_ilut(csr_from_arrays(n, n, rp, ci, v), tol);
    *out = f.release();
  });
}
int ref_factor_exact(int n, const int* rp, const int* ci, const double* v,
                     RefFactors** out) {
  return guarded([&] {
    auto f = std::make_unique<RefFactors>();
    f->f = factor_exact(csr_from_arrays(n, n, rp, ci, v));
    *out = f.release();
  });
}
void ref_factors_free(RefFactors* f) { delete f; }
void ref_factors_dims(RefFactors* f, int* dim, int64_t* nnz_l, int64_t* nnz_u) {
  *dim = f->f.dim();
  *nnz_l = static_cast<int64_t>(f->f.lower.nnz());
  *nnz_u = static_cast<int64_t>(f->f.upper.nnz());
}
void ref_factors_get(RefFactors* f, int* lrp, int* lci, double* lv, int* urp,
                     int* uci, double* uv, int* perm) {
  copy_csr(f->f.lower, lrp, lci, lv);
  copy_csr(f->f.upper, urp, uci, uv);
  if (perm) std::memcpy(perm, f->f.row_perm.forward.data(), sizeof(int) * f->f.dim());
}
// Build factors directly from arrays (e.g. factors downloaded from the GPU,
// identical to the reference's) so that the reference `solve` can be timed
// without re-running its ILUT.
RefFactors* ref_factors_from_arrays(int n, const int* lrp, const int* lci,
                                    const double* lv, const int* urp,
                                    const int* uci, const double* uv,
                                    const int* perm) {
  auto f = std::make_unique<RefFactors>();
  f->f.lower = csr_from_arrays(n, n, lrp, lci, lv);
  f->f.upper = csr_from_arrays(n, n, urp, uci, uv);
  std::vector<int> fwd(n);
  for (int i = 0; i < n; ++i) fwd[i] = perm ? perm[i] : i;
  f->f.row_perm = Permutation::from_forward(fwd);
  return f.release();
}
// Same, straight from reference-invariant CSR arrays (no triplet sort).
RefFactors* ref_factors_from_csr(int n, const int* lrp, const int* lci, const double* lv,
                                 const int* urp, const int* uci, const double* uv) {
  auto f = std::make_unique<RefFactors>();
  f->f.lower = csr_direct(n, n, lrp, lci, lv);
  f->f.upper = csr_direct(n, n, urp, uci, uv);
  f->f.row_perm = Permutation::identity(n);
  f->f.kind = FactorKind::Incomplete;
  return f.release();
}

int ref_solve(RefFactors* f, const double* b, double* x) {
  return guarded([&] {
    std::vector<double> r = solve(f->f, std::span<const double>(b, f->f.dim()));
    std::memcpy(x, r.data(), sizeof(double) * r.size());
  });
}

// CPU baseline timing: `reps` sweeps of the reference `solve` over the given
// factor handles (one per sampled block), run with the reference's own
// parallel_for (parallel.cpp:21-50) on `workers` threads.  rhs/out hold
// sum(dim) doubles, concatenated per handle.  Returns wall seconds.
double ref_time_block_solves(int nf, RefFactors** fs, const double* rhs,
                             double* out, int reps, int workers) {
  std::vector<std::size_t> off(nf + 1, 0);
  for (int i = 0; i < nf; ++i) off[i + 1] = off[i] + fs[i]->f.dim();
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    parallel_for(nf, workers, [&](int i) {
      std::vector<double> x =
          solve(fs[i]->f, std::span<const double>(rhs + off[i], fs[i]->f.dim()));
      std::memcpy(out + off[i], x.data(), sizeof(double) * x.size());
    });
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_hardware_threads() {
  return static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
}

// Matrix Market I/O through the reference (matrix_market.cpp:20-142).
struct RefMat {
  SparseMatrix a;
};

// oracle::random_dd_sparse(n, density, mt19937(seed)) (tests/oracles.hpp:100-120).
RefMat* ref_random_dd_sparse(int n, double density, unsigned seed) {
  std::mt19937 rng(seed);
  return new RefMat{oracle::random_dd_sparse(n, density, rng)};
}

// The raw (unscaled, unpermuted) (1,1) block D of generate_oseen(grid, nu)
// on the uniform grid with the recirculating wind (acceptance.cpp:513-519).
int ref_oseen_raw_d(int grid_n, double nu, RefMat** out) {
  return guarded([&] {
    auto prob = generate_oseen(grid_n, nu, GridKind::Uniform, WindKind::Recirculating);
    *out = new RefMat{prob.matrices.D};
  });
}
int ref_mm_read(const char* path, RefMat** out) {
  return guarded([&] { *out = new RefMat{load_matrix_market(path)}; });
}
void ref_mat_dims(RefMat* m, int* nrows, int* ncols, int64_t* nnz) {
  *nrows = m->a.rows();
  *ncols = m->a.cols();
  *nnz = m->a.nnz();
}
void ref_mat_get(RefMat* m, int* rp, int* ci, double* v) { copy_csr(m->a, rp, ci, v); }
void ref_mat_free(RefMat* m) { delete m; }
int ref_mm_write(const char* path, int nrows, int ncols, const int* rp, const int* ci,
                 const double* v) {
  return guarded([&] { write_matrix_market(path, csr_from_arrays(nrows, ncols, rp, ci, v)); });
}
int ref_mm_read_vector(const char* path, int* n, double* v) {
  return guarded([&] {
    std::vector<double> x = load_vector_market(path);
    *n = static_cast<int>(x.size());
    if (v) std::memcpy(v, x.data(), sizeof(double) * x.size());
  });
}
int ref_mm_write_vector(const char* path, int n, const double* v) {
  return guarded([&] { write_vector_market(path, std::span<const double>(v, n)); });
}

}  // extern "C"
