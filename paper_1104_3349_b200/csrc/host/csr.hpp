// Host-side CSR used by the one-off setup layer (problem assembly, saddle
// partitioning, aggregation, Schur approximation).  Same storage convention
// as the reference SparseMatrix (proj/include/msc/sparse_matrix.hpp:77-81):
// int32 row offsets and columns, fp64 values, columns strictly increasing
// per row, no stored zeros.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mscg::host {

struct Csr {
  int nrows = 0, ncols = 0;
  std::vector<int> rp{0};
  std::vector<int> ci;
  std::vector<double> v;

  Csr() = default;
  Csr(int r, int c) : nrows(r), ncols(c), rp(r + 1, 0) {}
  int64_t nnz() const { return static_cast<int64_t>(ci.size()); }
  int row_begin(int i) const { return rp[i]; }
  int row_end(int i) const { return rp[i + 1]; }
};

// Error carrying the zero-pivot index, mirrored onto the C-ABI status
// (reference SingularMatrixError, sparse_matrix.hpp:23-28).
struct SingularError : std::runtime_error {
  SingularError(const std::string& w, int piv) : std::runtime_error(w), pivot(piv) {}
  int pivot;
};

// A[rb:re, cb:ce) re-indexed from 0 (reference extract_block,
// sparse_matrix.cpp:127-144).  Rows are sorted so a plain filter suffices.
inline Csr extract_block(const Csr& a, int rb, int re, int cb, int ce) {
  Csr out(re - rb, ce - cb);
  for (int i = rb; i < re; ++i) {
    for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
      const int c = a.ci[k];
      if (c >= cb && c < ce) {
        out.ci.push_back(c - cb);
        out.v.push_back(a.v[k]);
      }
    }
    out.rp[i - rb + 1] = static_cast<int>(out.ci.size());
  }
  return out;
}

// Symmetric permutation result(i,j) = A(fwd[i], fwd[j]) (reference permute,
// permutation.cpp:30-45): per new row, columns re-sorted by new index.
Csr permute_symmetric(const Csr& a, const std::vector<int>& fwd,
                      const std::vector<int>& inv);

}  // namespace mscg::host
