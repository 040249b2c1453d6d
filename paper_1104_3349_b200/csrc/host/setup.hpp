// Host problem layer: one-off setup that produces the (interior blocks |
// interface) saddle system the device solve phase consumes.  Everything here
// reproduces the reference's matrices bit-for-bit ("must be
// reproduced bit-identically so that GPU and CPU see the same matrix").
#pragma once

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "csr.hpp"

namespace mscg::host {

struct OseenSystem {
  Csr C;                    // physics split: velocities [0,p), pressures [p,n)
  int p = 0;
  std::vector<double> rhs;  // generator rhs (leaky lid)
};

// generate_oseen(..., WindKind::Recirculating, stretch): proj/src/oseen.cpp:373-441.
OseenSystem generate_oseen(int grid_n, double nu, bool stretched, double stretch);
// Its argument checks and its grid (cell boundaries x, y and centres xc, yc;
// oseen.cpp:19-71) for the device assembly (csrc/device/oseen.cu).
void check_oseen_args(int grid_n, double nu, bool stretched, double stretch);
void oseen_grid(int grid_n, bool stretched, double stretch, std::vector<double>& x,
                std::vector<double>& y, std::vector<double>& xc, std::vector<double>& yc);

// scale_rows: proj/src/row_scaling.cpp:8-31 (in place).
void scale_rows(Csr& a, std::vector<double>& rhs);

// Partitioned system in the final numbering (reference PartitionedMatrix,
// proj/include/msc/partitioned_matrix.hpp:19-37, restricted to what the
// solve phase needs).
struct Partitioned {
  Csr C;
  int p = 0;
  std::vector<std::pair<int, int>> d_ranges;
  std::vector<int> perm;    // forward map: new index k holds original perm[k]
  int separator_size = 0;   // interface velocities (head of the interface)
  int n() const { return C.nrows; }
  int n_g() const { return C.nrows - p; }
};

// partition_saddle(c, p, target_blocks, Interleaved):
// proj/src/partitioned_matrix.cpp:71-203 with nested_dissection
// (proj/src/graph.cpp:136-230).  `threads` <= 0 picks the hardware count;
// the result does not depend on it.
Partitioned partition_saddle(const Csr& c, int p, int target_blocks, int threads = 0);

// SURVEY.md §8(d) interface anchoring: each interface pressure with an
// interface-velocity neighbour is moved directly after its smallest-index
// such neighbour (symmetric permutation of the (2,2) side only).
void anchor_interface(Partitioned& pm);

// Aggregate sizes.  equal_sizes: proj/src/aggregates.cpp:132-141;
// anchored_sizes: greedy, close once >= sz unless the next node is a
// pressure (an interface row without a diagonal entry).
std::vector<int> equal_sizes(int n_g, int sz);
std::vector<int> anchored_sizes(const Partitioned& pm, int sz);

enum class Variant { Mscn, Mscnr, Lum };
Variant variant_from_name(const std::string& name);

// build_msc for the non-overlapped numbering variants
// (proj/src/schur_approx.cpp:88-161): S^ as a block-diagonal CSR over the
// aggregate ranges.
struct SchurApprox {
  Csr s_hat;
  std::vector<std::pair<int, int>> ranges;
};
SchurApprox build_msc(const Partitioned& pm, const std::vector<int>& sizes,
                      Variant v, int threads = 0);

int hardware_threads();

// Matrix Market coordinate I/O (proj/src/matrix_market.cpp:20-142), the
// wire format shared with the reference; failures throw IoError with the
// reference's message text (proj/include/msc/matrix_market.hpp:16-24).
struct IoError : std::runtime_error {
  explicit IoError(const std::string& w) : std::runtime_error(w) {}
};
Csr load_matrix_market(const std::string& path);
void write_matrix_market(const std::string& path, const Csr& a);
std::vector<double> load_vector_market(const std::string& path);
void write_vector_market(const std::string& path, const double* v, int n);

}  // namespace mscg::host
