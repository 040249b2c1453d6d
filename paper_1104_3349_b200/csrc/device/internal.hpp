// Internal C++ interfaces between the C ABI (csrc/capi.cpp) and the device
// code (csrc/device/*.cu).  Nothing here is exported.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

namespace mscg {

// Owning device allocation.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n);
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept;
  template <class T> T* as() const { return static_cast<T*>(p); }
  void reset();
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;        // stream every call is ordered on
  cudaStream_t owned_stream = nullptr;  // the context's own (destroyed with it)
  int sm_count = 148;
  int64_t launches = 0;
  int correction = -1;  // kCorr* for preconditioners built on this context (-1: default)
  // pinned staging for host<->device vector traffic
  double* pinned = nullptr;
  size_t pinned_elems = 0;
  double* stage(size_t elems);
  ~Ctx();
};

// Device CSR kept in SELL-64 (slices of 64 rows, column-major inside a
// slice): lane r of a warp owns rows 2r, 2r+1 and reads entry k of both as one
// 16-byte load, keeping the reference's row-sequential accumulation order.
struct DevCsr {
  Ctx* ctx = nullptr;
  int nrows = 0, ncols = 0;
  int64_t nnz = 0;
  int nslices = 0;
  DevBuf slice_ptr;    // int64[nslices+1] entry offsets
  DevBuf slice_width;  // int32[nslices]
  DevBuf col;          // int32 (-1 = padding)
  DevBuf val;          // fp64
  int64_t padded = 0;
};
std::unique_ptr<DevCsr> upload_csr(Ctx* ctx, int nrows, int ncols, const int* rp,
                                   const int* ci, const double* v);
// y = A x                        (mode 0)
// y = base - A x                 (mode 1)
// y = base + A x                 (mode 2; base may alias y)
void spmv(const DevCsr& a, const double* x, double* y, const double* base, int mode,
          cudaStream_t s);
// the same for rows [row_lo, row_hi) only
void spmv_rows(const DevCsr& a, const double* x, double* y, const double* base, int mode,
               int row_lo, int row_hi, cudaStream_t s);

// Per-block factors in the tiled solve layout (see trisolve.cu).  Rows of a
// block are grouped in tiles of kTile = 32 rows.  For tile t:
//  * L near window: columns 32(t-2) .. 32(t+1): tiles t-2, t-1 and the
//    strictly lower diagonal tile t;
//  * U near window: columns 32t .. 32(t+3): the strictly upper diagonal tile
//    t and tiles t+1, t+2 (stored layout below);
//  * far entries (L: columns < 32(t-2); U: columns >= 32(t+3)) in CSR with
//    block-local uint16 columns, every block's rows contiguous, row offsets
//    indexed by row0[b] + b + i (dim+1 per block, relative to loff/uoff[b]).
// The U diagonal is kept apart (udiag) together with its reciprocal.
// Absent entries are exact zeros in the near tiles (stored factor values are
// never zero), so the reference CSR is recoverable exactly.
constexpr int kTile = 32;
constexpr int kNearTiles = 3;
// Stored near tile (one TMA copy brings everything the chain needs, so the
// solver warp issues no global loads), in this order:
//  * per-row metadata: [kMetaDiag + j] = 1 / U_jj (U tiles), [kMetaSeg + j]
//    = far work items of row j (int in the low 32 bits);
//  * header: [kHdr] = ELL width W of this tile (or kDenseNbr), [kHdr + 1] =
//    bytes of the near item the solver issues kRing items later (the tile
//    stream carries its own copy sizes);
//  * the strictly triangular part of the INVERSE of the diagonal tile packed
//    by column (tri_l / tri_u): L_tt^-1 is unit lower triangular, U_tt^-1
//    upper triangular with diagonal 1 / U_jj (the metadata), so the tile's
//    32-step substitution chain becomes one 32-term dot product per row;
//  * the two neighbour tiles (L: t-2, t-1; U: t+1, t+2), as a 64-column
//    window, either
//      - ELL (W entries per row, W a multiple of 4, rows padded with zero
//        values): window columns as bytes, word [(e/4)*32 + j] holding
//        entries 4(e/4)..+3 of row j, then values as double2 pairs
//        [(e/2)*32 + j] — 36 W doubles; or
//      - dense (kDenseNbr, when ELL would not be smaller): 32 x 64
//        column-major, entry [k*32 + j].
// Only the used prefix of a tile is copied (kNbrOff + 36 W doubles for ELL).
// Past the largest copy (kTileElems) each slot keeps the diagonal tile's own
// strictly triangular part (kOrigOff, same packing), never read by the solve,
// from which the reference factors are recovered exactly.
constexpr int kMetaDiag = 0;
constexpr int kMetaSeg = kTile;
constexpr int kHdr = 2 * kTile;
constexpr int kTriOff = kHdr + 4;
constexpr int kTriElems = kTile * (kTile - 1) / 2;
// L: column k holds rows k+1..31; U: column k holds rows 0..k-1.
__host__ __device__ constexpr int tri_l(int j, int k) { return k * (2 * kTile - 1 - k) / 2 + j - k - 1; }
__host__ __device__ constexpr int tri_u(int j, int k) { return k * (k - 1) / 2 + j; }
constexpr int kNbrOff = kTriOff + kTriElems;
constexpr int kNbrElems = 2 * kTile * kTile;
constexpr int kTileElems = kNbrOff + kNbrElems;
constexpr int kOrigOff = kTileElems;
constexpr int kTileStride = kOrigOff + kTriElems;
constexpr int kDenseNbr = -1;
constexpr int kEllMax = ((kNbrElems / 36) / 4) * 4;  // widest ELL smaller than dense (56)
__host__ __device__ constexpr int ell_width(int maxrow) {
  return (maxrow + 3) / 4 * 4 > kEllMax ? kDenseNbr : (maxrow + 3) / 4 * 4;
}
__host__ __device__ constexpr int tile_elems(int w) {
  return w == kDenseNbr ? kTileElems : kNbrOff + 36 * w;
}
// ELL entry e of row j: value index and column byte index within the tile.
__host__ __device__ constexpr int ell_val(int w, int j, int e) {
  return kNbrOff + 4 * w + ((e >> 1) * kTile + j) * 2 + (e & 1);
}
__host__ __device__ constexpr int ell_colbyte(int j, int e) {
  return kNbrOff * 8 + ((e >> 2) * kTile + j) * 4 + (e & 3);
}
// Window padding column (a slot that is always solved before use): L: the
// last row of tile t-1; U: the first row of tile t+1.
constexpr int kPadColL = 2 * kTile - 1;
constexpr int kPadColU = 0;
// Near items in flight per solver (TMA ring depth).
constexpr int kRing = 2;
// Far entries of a row are cut into work items of kSeg entries (at most
// kMaxSeg per row; the last item takes the remainder).  Item lists per block
// and pass (L: rows ascending, U: rows descending) hold int4 {row, seg,
// begin, end} (far-entry offsets within the block).
constexpr int kSolveChunks = 8;
// Rows of one tile whose far lists are short (<= kShortRow entries) are
// grouped into one work item of at most kGroupEntries entries: a warp loads
// them in one round and sums each row in shared memory (one memory round trip
// for the group instead of one per row).  Item encoding: y = need << 8 |
// kMultiFlag | (rows - 1), x = first row (ascending), [z, w) = entries.
constexpr int kShortRow = 96;
constexpr int kGroupEntries = 128;
constexpr int kMultiFlag = 0x80;
constexpr int kSeg = 512;
constexpr int kMaxSeg = 4;
constexpr int kMaxNeed = 65536 / kTile;  // readiness counts are tiles of a block
__host__ __device__ inline int far_segments(int nfar) {
  const int s = (nfar + kSeg - 1) / kSeg;
  return s < kMaxSeg ? s : kMaxSeg;
}
// Pieces of a long row (more than kShortRow far entries) when the pack cuts
// rows by readiness (pack_tiled_kernel): at least `pieces`, at most kMaxSeg.
__host__ __device__ inline int far_pieces(int nfar, int pieces) {
  int s = far_segments(nfar);
  if (nfar > kShortRow && s < pieces) s = pieces;
  return s < kMaxSeg ? s : kMaxSeg;
}
struct FactorSet {
  int nblocks = 0;
  int total_rows = 0;
  int max_dim = 0;
  bool has_perm = false;
  std::vector<int> h_row0, h_dim;          // host copies
  std::vector<int64_t> h_loff, h_uoff;     // per block far-entry offsets (+1 total)
  std::vector<int64_t> h_toff;             // per block first tile (+1 total)
  std::vector<int64_t> h_nnz_l, h_nnz_u;   // true factor counts (U without diagonal)
  std::vector<char> h_exact;               // per block: exact LU (1) or ILUT (0)
  DevBuf row0, dim;                        // int32[nblocks]
  DevBuf loff, uoff;                       // int64[nblocks+1]
  DevBuf toff;                             // int64[nblocks+1]
  DevBuf lrp, urp;                         // int32[total_rows + nblocks]
  DevBuf lval, uval;                       // fp64 (far entries)
  DevBuf lcol, ucol;                       // uint16
  DevBuf ltile, utile;                     // fp64 [tiles][kTileStride] (copied prefix varies)
  DevBuf lwidth, uwidth;                   // int32[tiles]: ELL width or kDenseNbr
  // Far sums: every work item writes its own slot (per block and pass; a
  // row's slots are consecutive from lslot/uslot[row]), max_slots per block.
  DevBuf lslot, uslot;                     // int32[total_rows]
  int max_slots = 0;
  std::vector<int> h_lwidth, h_uwidth;
  std::vector<int64_t> h_lioff, h_uioff;   // per block far work-item offsets (+1)
  DevBuf lioff, uioff;                     // int64[nblocks+1] (capacity)
  DevBuf lnum, unum;                       // int32[nblocks] items in use
  DevBuf litems, uitems;                   // int32 (row << 3 | seg)
  DevBuf udiag, urdiag;                    // fp64[total_rows]
  DevBuf perm;                             // int32[total_rows] (local), if has_perm
  DevBuf order;                            // int32[nblocks] launch order, all blocks (LPT)
  DevBuf order_chunked;                    // the same per chunk (positions h_chunk[c]..)
  // The blocks are cut into kSolveChunks contiguous chunks (block index
  // ranges h_chunk[c] .. h_chunk[c+1]); `order` lists each chunk's blocks
  // longest first (LPT) at the same positions, so a chunk can be solved on
  // its own (host-buffer applies overlap the copies of one chunk with the
  // solve of another).
  std::vector<int> h_chunk;
  // side stream for the last partial wave of a whole-set solve (trisolve.cu)
  mutable std::mutex tail_mu;
  mutable cudaStream_t tail_stream = nullptr;
  mutable cudaEvent_t tail_ev[2] = {nullptr, nullptr};
  ~FactorSet();
  int64_t nnz_l() const;
  int64_t nnz_u() const;
  int64_t far_l() const { return h_loff.empty() ? 0 : h_loff.back(); }
  int64_t far_u() const { return h_uoff.empty() ? 0 : h_uoff.back(); }
  int64_t tiles() const { return h_toff.empty() ? 0 : h_toff.back(); }
};

// Block descriptor for factorisation input: rows [row0, row0+dim) of a CSR
// matrix whose block-local columns are [col0, col0+dim).
struct BlockSpec {
  int row0, dim, col0;
};

struct FactorTimes {
  double ilut_s = 0, lu_s = 0, pack_s = 0, corr_s = 0;
};

// Factor all blocks of `a_rp/a_ci/a_v` (device CSR arrays, int32) listed in
// `blocks`: ILUT(tol) where exact[b] == 0, dense partial-pivoting LU where
// exact[b] == 1.  Throws Error(SINGULAR) naming the first failing block.
// `what` prefixes error messages ("(1,1) block" / "Schur block").
std::unique_ptr<FactorSet> factor_blocks(Ctx* ctx, const int* a_rp, const int* a_ci,
                                         const double* a_v,
                                         const std::vector<BlockSpec>& blocks,
                                         const std::vector<char>& exact, double tol,
                                         const char* what, FactorTimes* times);

// x_b = U_b^-1 L_b^-1 P_b rhs_b for every block b, launched as one kernel
// (one CTA per block).  out = x, or out = sub - x when sub != nullptr.
// order/norder (optional): solve only the blocks order[0 .. norder) (device
// list), in that order.
void block_trisolve(const FactorSet& fs, const double* rhs, double* out,
                    const double* sub, cudaStream_t s, long long* trace = nullptr,
                    int chunk = -1, const int* order = nullptr, int norder = 0);
// Raise a kernel's dynamic shared-memory limit once per kernel and size.
void ensure_smem(const void* kern, size_t smem);

// Explicit interior correction (correct.cu): W_b = D_b^-1 E_b[:, cols_b] per
// interior block as a dense column-major panel, so the apply's second half
// x1 = z1 - D^-1 (E z2) becomes x1_b = z1_b - W_b z2[cols_b] (one streaming
// pass over W instead of an E SpMV and a second pass over the factors).
constexpr int kCorrOff = 0, kCorrOn = 1, kCorrAuto = 2;
int correction_mode_default();  // MSCG_CORRECTION=off|on|auto (default auto)
struct Correction {
  int nblocks = 0, kmax = 0;
  int64_t entries = 0;         // sum over blocks of dim_b * k_b
  const int* row0 = nullptr;   // the FactorSet's (borrowed)
  const int* dim = nullptr;
  DevBuf woff;                 // int64[nblocks+1] panel offsets
  DevBuf wcoff;                // int32[nblocks+1] column-list offsets
  DevBuf wcols;                // int32 interface columns per block, ascending
  DevBuf wval;                 // fp64 panels
  DevBuf items;                // int2 {block, first row} (slices of `slice` rows)
  int slice = 512;
  bool split = false;          // correct_split_kernel (few rows)
  std::vector<int> h_item_chunk;  // item range of block chunk c
  double build_s = 0;
};
// E rows numbered like D's rows (e_rp has D.total_rows + 1 entries), columns
// = interface index.  r/o scratch: D.total_rows doubles each.  Returns null
// when mode is off, or auto and the panels would not save bytes / memory.
std::unique_ptr<Correction> build_correction(Ctx* ctx, const FactorSet& D, const int* e_rp,
                                             const int* e_ci, const double* e_v, int mode,
                                             double* r_scratch, double* o_scratch);
// out_b = z1_b - W_b x2[cols_b] for all blocks (chunk < 0) or block chunk c.
void apply_correction(const Correction& c, const double* x2, const double* z1, double* out,
                      int chunk, cudaStream_t s);

// A shard owns the interior blocks [b0, b1) (rows [row_lo, row_hi)) of a
// preconditioner split across ranks.  Its D holds only those
// blocks, E only those rows and F only those columns, so one apply is
//   rank:      z1_r = D_r^-1 y1_r,  tpart = F_r z1_r          (apply_shard_begin)
//   exchange:  tsum = sum over ranks of tpart                 (caller: all-reduce)
//   rank:      z2 = S^-1 (y2 - tsum), x1_r = z1_r - D_r^-1 E_r z2   (apply_shard_end)
// with S replicated.  Vectors keep the global length; each rank touches its
// interior rows and the (replicated) interface rows only.
struct Shard {
  bool on = false;
  int b0 = 0, b1 = 0, row_lo = 0, row_hi = 0;
  std::unique_ptr<DevCsr> Cr;  // C[row_lo:row_hi, :]
  std::unique_ptr<DevCsr> G;   // C[p:n, p:n]
};

struct Precond {
  Ctx* ctx = nullptr;
  int n = 0, p = 0;
  std::unique_ptr<DevCsr> C, E, F;
  std::unique_ptr<FactorSet> D, S;
  std::unique_ptr<Correction> corr;  // explicit D^-1 E panels (null: two solves)
  int64_t stored_nnz = 0;
  FactorTimes times;
  Shard shard;
  // Build-time and shard scratch (a shard's z1 lives from apply_shard_begin
  // to apply_shard_end, so a shard is one apply at a time by contract).
  DevBuf z1, t, w;
  // Use the explicit correction panels when built (false: the reference's
  // E SpMV + second interior solve, for measurement and cross-checks).
  bool use_corr = true;
  // x = B^-1 y on stream s.  The apply's own vectors (z1, t, w) come from a
  // per-stream scratch set: calls on one stream are ordered by the stream,
  // calls on different streams get different sets, so concurrent applies
  // from several threads are safe (preconditioner.hpp:17-18).
  void apply(const double* y_dev, double* x_dev, cudaStream_t s, cudaEvent_t* ev = nullptr);
  // x = B^-1 y with y, x in page-locked host memory: the interior rows move
  // in kSolveChunks pieces on side streams so that each piece's copy overlaps
  // the solve of the others.  d_y, d_x: device scratch of n doubles.
  void apply_host(const double* y_host, double* x_host, double* d_y, double* d_x,
                  cudaStream_t s);
  // y = C x with x, y page-locked host memory: an interior row of C only
  // reads its own block's and the interface's columns, so each block
  // chunk's rows are multiplied as soon as that chunk of x (and the
  // interface part, copied first) has arrived, and leave while later
  // chunks are still in flight.  d_x, d_y: device scratch of n doubles.
  // When the interior ranges are coupled (entries of C[0:p, 0:p] outside
  // their block: PartitionedMatrix::from_split accepts such splits and the
  // preconditioner keeps only the diagonal blocks) the whole x is copied
  // before any row is multiplied.
  bool d_coupled = false;
  void spmv_host(const double* x_host, double* y_host, double* d_x, double* d_y,
                 cudaStream_t s);
  ~Precond();
  void apply_shard_begin(const double* y_dev, double* tpart_dev, cudaStream_t s);
  void apply_shard_end(const double* y_dev, const double* tsum_dev, double* x_dev,
                       cudaStream_t s);
  // y1_r = C[rows_r, :] x;  y2part = F_r x1_r (+ G x2 when with_g): the
  // interface rows of C x are the sum of y2part over ranks.
  void spmv_shard(const double* x_dev, double* y_dev, double* y2part_dev, bool with_g,
                  cudaStream_t s);

 private:
  void ensure_side_streams();
  void chunk_rows(int c, int& lo, int& hi) const;
  struct Scratch {
    DevBuf z1, t, w;
  };
  Scratch& scratch_for(cudaStream_t s);
  std::mutex scratch_mu;
  std::vector<std::pair<cudaStream_t, std::unique_ptr<Scratch>>> scratch;
  cudaStream_t side[kSolveChunks] = {};
  cudaEvent_t ev_in[kSolveChunks] = {}, ev_out[kSolveChunks] = {}, ev_mid = nullptr;
};

// Build the whole preconditioner (block_begin = 0, block_end = -1) or the
// shard owning interior blocks [block_begin, block_end).  schur_single: S^
// is an overlapped band, factored whole by one exact LU (the reference's
// schur_single_, preconditioner.cpp:58-67; s_ranges unused).
std::unique_ptr<Precond> build_precond(Ctx* ctx, int n, int p, const int* c_rp,
                                       const int* c_ci, const double* c_v,
                                       const std::vector<std::pair<int, int>>& d_ranges,
                                       const int* s_rp, const int* s_ci,
                                       const double* s_v,
                                       const std::vector<std::pair<int, int>>& s_ranges,
                                       double tol_a, int s_a, int block_begin = 0,
                                       int block_end = -1, bool schur_single = false);

// build_msc for numbering aggregates (ranges over the interface numbering)
// on the device: S^ returned as a host CSR (n_g x n_g, block diagonal),
// bit-identical to the reference.  Throws Error(SINGULAR) naming the first
// aggregate whose D block is singular.
constexpr int kMscMscn = 0, kMscMscnr = 1, kMscLum = 2;
// nested_dissection (proj/src/graph.cpp:178-230) of an undirected graph
// (CSR, sorted adjacency, no self loops) on the device: blocks in the
// reference's depth-first leaf order (each ascending) and the sorted
// separator, identical to the reference (csrc/device/dissect.cu).
void nested_dissection_device(Ctx* ctx, int n, const int64_t* off, const int* adj,
                              int target_blocks, std::vector<std::vector<int>>& blocks,
                              std::vector<int>& separator);

// ranges: owned ranges; spans: each aggregate's working range (= ranges,
// or extended into the next aggregate for the overlapped variants, whose
// banded S^ is merged on the host in the reference's order).
void build_msc_device(Ctx* ctx, int n, int p, const int* c_rp, const int* c_ci, const double* c_v,
                      const std::vector<std::pair<int, int>>& ranges,
                      const std::vector<std::pair<int, int>>& spans, int variant,
                      std::vector<int>& s_rp, std::vector<int>& s_ci, std::vector<double>& s_v);

// generate_oseen's assembly + scale_rows on the device (one thread per row,
// bit-identical; grid from the host): returns the scaled CSR and rhs.
void oseen_assemble_device(Ctx* ctx, int n, const std::vector<double>& x,
                           const std::vector<double>& y, const std::vector<double>& xc,
                           const std::vector<double>& yc, double nu, std::vector<int>& rp,
                           std::vector<int>& ci, std::vector<double>& v,
                           std::vector<double>& rhs, int& p_out);

// Download one block's factors in the reference layout.
void download_factor(const FactorSet& fs, int idx, std::vector<int>& lrp,
                     std::vector<int>& lci, std::vector<double>& lv,
                     std::vector<int>& urp, std::vector<int>& uci,
                     std::vector<double>& uv, std::vector<int>& perm);

struct GmresConfig {
  int restart = 300, max_iters = 3000;
  double rel_tol = 1e-9;
  bool left = false;
  int orth = 2;  // 0 MGS, 1 CGS2, 2 DCGS2
};
struct GmresResult {
  int iterations = 0;
  bool converged = false;
  std::vector<double> history;
  double seconds = 0, final_true = 0;
};
GmresResult gmres(Ctx* ctx, const DevCsr& a, Precond* pc, const double* b_dev,
                  double* x_dev, const GmresConfig& cfg);
double true_residual(Ctx* ctx, const DevCsr& a, const double* x_dev, const double* b_dev);
// Distributed GMRES over preconditioner shards (one rank per process):
// comm.allreduce(count, user) must sum buf[0:count] over the ranks in stream
// order on the context stream.  b, x: global-length device vectors (x gets
// the rank's own interior rows and the interface; other rows zero).
struct DistComm {
  int rank = 0, size = 1;
  double* buf = nullptr;
  int cap = 0;
  void (*allreduce)(int count, void* user) = nullptr;
  void* user = nullptr;
};
GmresResult gmres_shard(Ctx* ctx, Precond* shard, const double* b_dev, double* x_dev,
                        const GmresConfig& cfg, const DistComm& comm);

}  // namespace mscg
