// Host problem layer: one-off setup that produces the (interior blocks |
// interface) saddle system the device solve phase consumes.  Everything here
// reproduces the reference's matrices bit-for-bit ("must be
// reproduced bit-identically so that GPU and CPU see the same matrix").
#pragma once

#include <cstdint>
#include <functional>
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
// `dissect` (optional) replaces the host nested dissection of the enriched
// graph (CSR with sorted adjacency): the device version
// (csrc/device/dissect.cu) plugs in here; the result must be the reference's
// blocks (depth-first order, each ascending) and sorted separator.
using Dissector = std::function<void(int n, const int64_t* off, const int* adj, int target,
                                     std::vector<std::vector<int>>& blocks,
                                     std::vector<int>& separator)>;
Partitioned partition_saddle(const Csr& c, int p, int target_blocks, int threads = 0,
                             const Dissector& dissect = {});

// nested_dissection (graph.cpp:178-230) on the host (level-parallel) of an
// undirected graph in CSR (sorted adjacency, no self loops), and build_graph
// (graph.cpp:8-30) of a square CSR pattern.
void nested_dissection_host(int n, const int64_t* off, const int* adj, int target_blocks,
                            int threads, std::vector<std::vector<int>>& blocks,
                            std::vector<int>& separator);
void undirected_graph(int n, const int* rp, const int* ci, std::vector<int64_t>& off,
                      std::vector<int>& adj);

// SURVEY.md §8(d) interface anchoring: each interface pressure with an
// interface-velocity neighbour is moved directly after its smallest-index
// such neighbour (symmetric permutation of the (2,2) side only).
void anchor_interface(Partitioned& pm);

// Aggregate sizes.  equal_sizes: proj/src/aggregates.cpp:132-141;
// anchored_sizes: greedy, close once >= sz unless the next node is a
// pressure (an interface row without a diagonal entry).
std::vector<int> equal_sizes(int n_g, int sz);
std::vector<int> anchored_sizes(const Partitioned& pm, int sz);

// MSC variants over numbering aggregates (schur_approx.cpp:11-52); the
// overlapped ones (O*) extend every aggregate's span by a width into the
// next (aggregate_overlapped, aggregates.cpp:50-85).
enum class Variant { Mscn, Mscnr, Lum, Omscn, Omscnr, Olum };
Variant variant_from_name(const std::string& name);
bool variant_overlapped(Variant v);
bool variant_rowsum(Variant v);
bool variant_lumped(Variant v);

// Overlap widths as benchmark.cpp:74-88 makes them: `overlap` for every
// aggregate (< 0: sz), the last 0, clipped to min(size - 1, n_g - end)
// (clip_overlap_widths, aggregates.cpp:143-156).
std::vector<int> overlap_widths(int n_g, const std::vector<int>& sizes, int sz, int overlap);

// build_msc (proj/src/schur_approx.cpp:88-161) over numbering aggregates:
// owned ranges from `sizes`, spans extended by `widths` (empty: none; the
// overlapped variants need them, aggregate_overlapped's checks apply).
// Each aggregate's dense S_ii lives on its span; the merge writes every
// owned column over its aggregate's whole span, so overlapped aggregates
// give a banded S^ (block diagonal otherwise).
struct SchurApprox {
  Csr s_hat;
  std::vector<std::pair<int, int>> ranges;  // owned ranges
  std::vector<std::pair<int, int>> spans;   // = ranges unless overlapped
  bool overlapped = false;
};
SchurApprox build_msc(const Partitioned& pm, const std::vector<int>& sizes,
                      Variant v, int threads = 0, const std::vector<int>& widths = {});
// The aggregate checks of aggregate_overlapped / check_agg_compatible
// (aggregates.cpp:50-85, schur_approx.cpp:56-85): owned ranges and spans.
void aggregate_spans(const Partitioned& pm, const std::vector<int>& sizes, Variant v,
                     const std::vector<int>& widths, std::vector<std::pair<int, int>>& ranges,
                     std::vector<std::pair<int, int>>& spans);
// The sequential merge (schur_approx.cpp:141-160) of per-aggregate dense
// blocks local[i] (span x span, row-major) into S^.
Csr merge_msc(int n_g, const std::vector<std::pair<int, int>>& ranges,
              const std::vector<std::pair<int, int>>& spans,
              const std::vector<const double*>& local);

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

namespace mscg {
struct Ctx;
// partition_saddle (Interleaved, partitioned_matrix.cpp:71-203) on the
// device (csrc/device/partition.cu) — attached lists, enriched graph, nested
// dissection, the second-block assignment, C' = P C P^T — and optionally
// the SURVEY 8(d) interface anchoring: identical to host::partition_saddle
// (+ host::anchor_interface).
host::Partitioned partition_saddle_device(Ctx* ctx, const host::Csr& c, int p, int target_blocks,
                                          bool anchored);
}  // namespace mscg
