// TEST INFRASTRUCTURE: the C++ drop-in (include/msc_b200/dropin.hpp) used
// exactly where the reference's own API is used, against the unmodified
// reference (compiled in place, oracle/_ref).  Mirrors the reference suites
// proj/tests/test_precond_solve.cpp and test_krylov.cpp:
//   * apply vs the dense three-factor inverse B (test_precond_solve.cpp:95-109)
//   * apply vs the reference MscPreconditioner on the Oseen cfg1 system
//   * the reference's OWN gmres driving the GPU preconditioner
//     (GpuPreconditioner is an msc::Preconditioner)
//   * msc_b200::gmres iteration count vs the reference (+-1)
//   * SingularMatrixError with the reference's message on the cfg3 system
// Prints "PASS <name>" / "FAIL <name>: detail"; exit status = failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "msc/gmres.hpp"
#include "msc/oseen.hpp"
#include "msc/partitioned_matrix.hpp"
#include "msc/row_scaling.hpp"
#include "msc/schur_approx.hpp"
#include "msc_b200/dropin.hpp"
#include "oracles.hpp"

using namespace msc;

static int failures = 0;
static void report(bool ok, const char* name, const std::string& detail = "") {
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name, detail.empty() ? "" : ": ", detail.c_str());
  if (!ok) ++failures;
}

static DenseMatrix dense_b(const PartitionedMatrix& c, const SparseMatrix& s_hat) {
  const int n = c.n(), p = c.p;
  DenseMatrix b(n, n);
  DenseMatrix d = to_dense(c.D), e = to_dense(c.E), f = to_dense(c.F);
  DenseMatrix corner = multiply(f, oracle::gauss_solve(d, e));
  DenseMatrix s = to_dense(s_hat);
  for (int i = 0; i < p; ++i) {
    for (int j = 0; j < p; ++j) b(i, j) = d(i, j);
    for (int j = 0; j < n - p; ++j) b(i, p + j) = e(i, j);
  }
  for (int i = 0; i < n - p; ++i) {
    for (int j = 0; j < p; ++j) b(p + i, j) = f(i, j);
    for (int j = 0; j < n - p; ++j) b(p + i, p + j) = corner(i, j) + s(i, j);
  }
  return b;
}

struct Cfg {
  PartitionedMatrix pm;
  std::vector<double> rhs;
};

static Cfg oseen(int grid, double nu, int nA, bool stretched = false, double stretch = 1.056) {
  OseenProblem prob = generate_oseen(grid, nu, stretched ? GridKind::Stretched : GridKind::Uniform,
                                     WindKind::Recirculating, stretch);
  RowScaling sc = scale_rows(prob.matrices.C, prob.rhs);
  SaddleReorder r = partition_saddle(sc.matrix, prob.matrices.p, nA, SaddleOrdering::Interleaved);
  return {r.matrix, permute_vector(sc.rhs, r.perm)};
}

int main() {
  // --- apply vs the dense three-factor inverse (exact factors) ---
  {
    std::mt19937 rng(37);
    PartitionedMatrix c = oracle::random_saddle(20, 8, rng, 0.3);
    SchurApproximation s = build_msc(c, aggregate_by_numbering(8, {4, 4}), MscVariant::Mscn);
    auto b = msc_b200::build_preconditioner(c, s, 0.0, 1 << 30);
    DenseMatrix bd = dense_b(c, s.s_hat);
    double worst = 0.0;
    for (int trial = 0; trial < 3; ++trial) {
      std::vector<double> y = oracle::random_vector(28, rng);
      worst = std::max(worst, oracle::rel_err(b.apply(y), oracle::gauss_solve(bd, y)));
    }
    report(worst < 1e-10, "apply_matches_dense_three_factor_inverse", std::to_string(worst));
  }
  // --- cfg1: apply, factors, gmres (ours and the reference's) ---
  {
    Cfg c = oseen(32, 0.1, 8);
    SchurApproximation s =
        build_msc(c.pm, aggregate_by_numbering(c.pm.n_g(), equal_sizes(c.pm.n_g(), c.pm.n_g() / 8)),
                  MscVariant::Lum);
    MscPreconditioner ref = build_preconditioner(c.pm, s, 1e-4, 0);
    auto gpu = msc_b200::build_preconditioner(c.pm, s, 1e-4, 0);
    std::mt19937 rng(0);
    std::vector<double> y = oracle::random_vector(c.pm.n(), rng);
    const double err = oracle::rel_err(gpu.apply(y), ref.apply(y));
    report(err < 1e-10, "cfg1_apply_vs_reference", std::to_string(err));
    report(gpu.stored_nnz() == ref.stored_nnz(), "cfg1_stored_nnz",
           std::to_string(gpu.stored_nnz()) + " vs " + std::to_string(ref.stored_nnz()));
    bool same = true;
    for (int bi = 0; bi < static_cast<int>(ref.d_factors().size()); ++bi) {
      TriangularFactors f = gpu.factors(0, bi);
      same = same && f.lower.same_pattern_and_values(ref.d_factors()[bi].lower) &&
             f.upper.same_pattern_and_values(ref.d_factors()[bi].upper);
    }
    report(same, "cfg1_ilut_factors_bit_identical");

    SolverConfig cfg;
    cfg.restart = 30;
    cfg.rel_tol = 1e-8;
    auto [xr, rr] = msc::gmres(c.pm.C, &ref, y, cfg);
    auto [xm, rm] = msc::gmres(c.pm.C, &gpu, y, cfg);  // reference GMRES, GPU preconditioner
    auto [xg, rg] = msc_b200::gmres(c.pm.C, &gpu, y, cfg);
    report(rr.converged && rm.converged && std::abs(rm.iterations - rr.iterations) <= 1,
           "reference_gmres_with_gpu_preconditioner",
           std::to_string(rm.iterations) + " vs " + std::to_string(rr.iterations));
    report(rg.converged && std::abs(rg.iterations - rr.iterations) <= 1 &&
               true_residual(c.pm.C, xg, y) <= 1e-8,
           "dropin_gmres_iterations",
           std::to_string(rg.iterations) + " vs " + std::to_string(rr.iterations));
    std::vector<double> mv = msc_b200::matvec(c.pm.C, y);
    report(mv == matvec(c.pm.C, y), "matvec_bit_identical");
  }
  // --- cfg1 with an overlapped Schur band (OMSCN): the drop-in factors the
  // band whole like the reference's schur_single_ (preconditioner.cpp:58-67)
  {
    Cfg c = oseen(32, 0.1, 8);
    const int ng = c.pm.n_g(), sz = ng / 8;
    std::vector<int> sizes = equal_sizes(ng, sz), widths(sizes.size(), sz);
    widths.back() = 0;
    clip_overlap_widths(ng, sizes, widths);
    SchurApproximation s =
        build_msc(c.pm, aggregate_overlapped(ng, sizes, widths), MscVariant::Omscn);
    MscPreconditioner ref = build_preconditioner(c.pm, s, 1e-4, 0);
    auto gpu = msc_b200::build_preconditioner(c.pm, s, 1e-4, 0);
    std::mt19937 rng(1);
    std::vector<double> y = oracle::random_vector(c.pm.n(), rng);
    const double err = oracle::rel_err(gpu.apply(y), ref.apply(y));
    report(s.overlapped && err < 1e-10, "omscn_band_apply_vs_reference", std::to_string(err));
    TriangularFactors f = gpu.factors(1, 0);
    report(ref.schur_factors().size() == 1 && f.dim() == ng &&
               f.upper.same_pattern_and_values(ref.schur_factors()[0].upper) &&
               f.lower.same_pattern_and_values(ref.schur_factors()[0].lower),
           "omscn_band_factor_bit_identical");
  }
  // --- cfg3 as written: identical SingularMatrixError ---
  {
    Cfg c = oseen(256, 0.002, 64, true, 1.1);
    SchurApproximation s =
        build_msc(c.pm, aggregate_by_numbering(c.pm.n_g(), equal_sizes(c.pm.n_g(), 795)),
                  MscVariant::Lum);
    std::string want, got;
    int pw = -1, pg = -2;
    try {
      build_preconditioner(c.pm, s, 1e-4, 0);
    } catch (const SingularMatrixError& e) {
      want = e.what();
      pw = e.pivot_index;
    }
    try {
      msc_b200::build_preconditioner(c.pm, s, 1e-4, 0);
    } catch (const SingularMatrixError& e) {
      got = e.what();
      pg = e.pivot_index;
    }
    report(!want.empty() && want == got && pw == pg, "cfg3_singular_error", got);
  }
  // --- input validation mirrors the reference ---
  {
    bool threw = false;
    try {
      SolverConfig bad;
      bad.restart = 0;
      msc_b200::gmres(SparseMatrix::identity(3), nullptr, std::vector<double>(3, 1.0), bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    report(threw, "gmres_bad_config_invalid_argument");
  }
  return failures;
}
