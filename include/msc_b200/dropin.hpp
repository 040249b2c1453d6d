// msc_b200/dropin.hpp — header-only C++ drop-in for the reference's
// solve-phase API (/root/reference/proj/include/msc), implemented over the
// C ABI in mscg.h.  A reference user swaps
//
//     msc::MscPreconditioner b = msc::build_preconditioner(c, s, tolA, sA);
//     auto [x, rep] = msc::gmres(c.C, &b, rhs, cfg);
// for
//     msc_b200::GpuPreconditioner b = msc_b200::build_preconditioner(c, s, tolA, sA);
//     auto [x, rep] = msc_b200::gmres(c.C, &b, rhs, cfg);
//
// with the same argument meaning and the same exceptions
// (std::invalid_argument, msc::SingularMatrixError{pivot_index}).
// GpuPreconditioner derives from msc::Preconditioner, so it also plugs into
// any code that takes `const msc::Preconditioner*` — including the
// reference's own gmres (preconditioner.hpp:19-28: apply is const and safe
// to call concurrently; each call here is stream-ordered on the context).
//
// Requires the reference headers on the include path (this adapter reads
// their types) and links against libmscg.so.
#pragma once

#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "msc/gmres.hpp"
#include "msc/matrix_market.hpp"
#include "msc/preconditioner.hpp"
#include "msc/schur_approx.hpp"
#include "mscg.h"

namespace msc_b200 {

[[noreturn]] inline void raise(const mscg_status& st) {
  const std::string msg = st.message;
  switch (st.code) {
    case MSCG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case MSCG_ERR_SINGULAR: throw msc::SingularMatrixError(msg, st.pivot_index);
    case MSCG_ERR_IO: throw msc::IoError(msg);  // message already carries "(line N)"
    default: throw std::runtime_error(msg);
  }
}
inline void check(int rc, const mscg_status& st) {
  if (rc != MSCG_OK) raise(st);
}

// One device + stream; shared by everything built from it.
class Context {
 public:
  explicit Context(int device = 0) {
    mscg_status st{};
    check(mscg_ctx_create(device, &h_, &st), st);
  }
  ~Context() { mscg_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  mscg_ctx* get() const { return h_; }
  static Context& instance() {
    static Context ctx(0);
    return ctx;
  }

 private:
  mscg_ctx* h_ = nullptr;
};

// Device-resident MSC preconditioner (reference MscPreconditioner,
// preconditioner.hpp:34-64).
class GpuPreconditioner : public msc::Preconditioner {
 public:
  GpuPreconditioner(mscg_precond* h, std::string kind, int n) : h_(h), kind_(std::move(kind)), n_(n) {}
  ~GpuPreconditioner() override { mscg_precond_destroy(h_); }
  GpuPreconditioner(GpuPreconditioner&& o) noexcept : h_(o.h_), kind_(std::move(o.kind_)), n_(o.n_) {
    o.h_ = nullptr;
  }

  std::vector<double> apply(std::span<const double> y) const override {
    if (static_cast<int>(y.size()) != n_)
      throw std::invalid_argument("MscPreconditioner::apply: length mismatch");
    std::vector<double> x(n_);
    mscg_status st{};
    check(mscg_precond_apply(h_, y.data(), x.data(), MSCG_MEM_HOST, &st), st);
    return x;
  }
  std::string kind() const override { return kind_; }
  int dim() const override { return n_; }
  std::size_t stored_nnz() const override {
    return static_cast<std::size_t>(mscg_precond_stored_nnz(h_));
  }

  // d_factors()/schur_factors() accessors (preconditioner.hpp:41-44),
  // materialised from the device on demand.
  msc::TriangularFactors factors(int kind, int idx) const {
    mscg_status st{};
    int dim = 0;
    int64_t nl = 0, nu = 0;
    check(mscg_precond_factor(h_, kind, idx, &dim, &nl, &nu, nullptr, nullptr, nullptr, nullptr,
                              nullptr, nullptr, nullptr, &st),
          st);
    std::vector<int> lrp(dim + 1), lci(nl), urp(dim + 1), uci(nu), perm(dim);
    std::vector<double> lv(nl), uv(nu);
    check(mscg_precond_factor(h_, kind, idx, &dim, &nl, &nu, lrp.data(), lci.data(), lv.data(),
                              urp.data(), uci.data(), uv.data(), perm.data(), &st),
          st);
    auto csr = [dim](const std::vector<int>& rp, const std::vector<int>& ci,
                     const std::vector<double>& v) {
      std::vector<msc::Triplet> t;
      t.reserve(v.size());
      for (int i = 0; i < dim; ++i)
        for (int k = rp[i]; k < rp[i + 1]; ++k) t.push_back({i, ci[k], v[k]});
      return msc::SparseMatrix::from_triplets(dim, dim, std::move(t));
    };
    msc::TriangularFactors f;
    f.lower = csr(lrp, lci, lv);
    f.upper = csr(urp, uci, uv);
    f.row_perm = msc::Permutation::from_forward(std::move(perm));
    return f;
  }
  mscg_precond* get() const { return h_; }

 private:
  mscg_precond* h_;
  std::string kind_;
  int n_;
};

// build_preconditioner (preconditioner.hpp:66-68): block-diagonal Schur
// approximations factor per owned range, overlapped (banded) ones whole by
// one exact LU (schur_single_, preconditioner.cpp:58-67).
inline GpuPreconditioner build_preconditioner(const msc::PartitionedMatrix& c,
                                              const msc::SchurApproximation& schur,
                                              double tolA, int sA,
                                              Context& ctx = Context::instance()) {
  if (schur.s_hat.rows() != c.n_g())
    throw std::invalid_argument(
        "build_preconditioner: Schur approximation does not match the split");
  std::vector<int> dr, sr;
  for (auto [b, e] : c.d_block_ranges) {
    dr.push_back(b);
    dr.push_back(e);
  }
  for (auto [b, e] : schur.owned_ranges) {
    sr.push_back(b);
    sr.push_back(e);
  }
  mscg_precond* h = nullptr;
  mscg_status st{};
  check(mscg_precond_build(ctx.get(), c.n(), c.p, c.C.row_offsets().data(),
                           c.C.col_indices().data(), c.C.values().data(),
                           static_cast<int>(c.d_block_ranges.size()), dr.data(),
                           schur.s_hat.row_offsets().data(), schur.s_hat.col_indices().data(),
                           schur.s_hat.values().data(),
                           schur.overlapped ? MSCG_SCHUR_SINGLE
                                            : static_cast<int>(schur.owned_ranges.size()),
                           sr.data(), tolA, sA, &h, &st),
        st);
  return GpuPreconditioner(h, schur.exact ? "exact-schur" : msc::variant_name(schur.variant),
                           c.n());
}

// matvec (sparse_matrix.hpp:87) on the device; bit-identical to the CPU.
inline std::vector<double> matvec(const msc::SparseMatrix& a, std::span<const double> x,
                                  Context& ctx = Context::instance()) {
  if (static_cast<int>(x.size()) != a.cols())
    throw std::invalid_argument("matvec: x has length " + std::to_string(x.size()) +
                                ", expected " + std::to_string(a.cols()));
  mscg_csr* h = nullptr;
  mscg_status st{};
  check(mscg_csr_upload(ctx.get(), a.rows(), a.cols(), a.row_offsets().data(),
                        a.col_indices().data(), a.values().data(), &h, &st),
        st);
  std::vector<double> y(a.rows());
  const int rc = mscg_spmv(h, x.data(), y.data(), MSCG_MEM_HOST, &st);
  mscg_csr_destroy(h);
  check(rc, st);
  return y;
}

// gmres (gmres.hpp:44-47): right/left-preconditioned restarted GMRES with
// the reference's convergence rules; `prec` must be a GpuPreconditioner or
// null (no CPU fallback for other preconditioners).  Orthogonalisation is
// DCGS2 (two basis sweeps; same projections as the reference's MGS, rounding
// regrouped).  cfg.restart <= 500 (std::invalid_argument above: the Givens
// state is staged in shared memory).
inline std::pair<std::vector<double>, msc::SolveReport> gmres(
    const msc::SparseMatrix& a, const msc::Preconditioner* prec, const std::vector<double>& rhs,
    const msc::SolverConfig& cfg, Context& ctx = Context::instance()) {
  const auto* gp = dynamic_cast<const GpuPreconditioner*>(prec);
  if (prec && !gp)
    throw std::invalid_argument("gmres: only device (GpuPreconditioner) preconditioners");
  const int n = a.rows();
  if (a.cols() != n || static_cast<int>(rhs.size()) != n)
    throw std::invalid_argument("gmres: dimension mismatch");
  mscg_status st{};
  mscg_csr* h = nullptr;  // the operator as given (it need not be the preconditioner's C)
  check(mscg_csr_upload(ctx.get(), n, n, a.row_offsets().data(), a.col_indices().data(),
                        a.values().data(), &h, &st),
        st);
  mscg_gmres_config c{cfg.restart, cfg.max_iters, cfg.rel_tol,
                      cfg.side == msc::PrecondSide::Left ? 1 : 0, 2};
  mscg_gmres_report rep{};
  std::vector<double> x(n), hist(static_cast<size_t>(cfg.max_iters) + 64);
  const int rc = mscg_gmres(ctx.get(), h, gp ? gp->get() : nullptr, rhs.data(), x.data(),
                            MSCG_MEM_HOST, &c, &rep, hist.data(), static_cast<int>(hist.size()),
                            &st);
  mscg_csr_destroy(h);
  check(rc, st);
  msc::SolveReport r;
  r.iterations = rep.iterations;
  r.converged = rep.converged != 0;
  r.residual_history.assign(hist.begin(), hist.begin() + rep.history_len);
  r.solve_seconds = rep.solve_seconds;
  return {std::move(x), std::move(r)};
}

// load_matrix_market / write_matrix_market (matrix_market.hpp:28-31) through
// the library's parser and writer (same CSR, same file bytes, same IoError).
inline msc::SparseMatrix load_matrix_market(const std::filesystem::path& path) {
  mscg_status st{};
  int nr = 0, nc = 0;
  int64_t nnz = 0;
  check(mscg_mm_read(path.c_str(), &nr, &nc, &nnz, nullptr, nullptr, nullptr, &st), st);
  std::vector<int> rp(nr + 1), ci(nnz);
  std::vector<double> v(nnz);
  check(mscg_mm_read(path.c_str(), &nr, &nc, &nnz, rp.data(), ci.data(), v.data(), &st), st);
  std::vector<msc::Triplet> t;
  t.reserve(nnz);
  for (int i = 0; i < nr; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k) t.push_back({i, ci[k], v[k]});
  return msc::SparseMatrix::from_triplets(nr, nc, std::move(t));
}
inline void write_matrix_market(const std::filesystem::path& path, const msc::SparseMatrix& a) {
  mscg_status st{};
  check(mscg_mm_write(path.c_str(), a.rows(), a.cols(), a.row_offsets().data(),
                      a.col_indices().data(), a.values().data(), &st),
        st);
}

}  // namespace msc_b200
