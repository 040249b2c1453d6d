// C ABI (include/mscg.h) over the host setup layer and the device solve phase.
// Maps C++ exceptions to mscg_status with the reference's error categories:
// std::invalid_argument -> MSCG_ERR_INVALID_ARGUMENT, SingularMatrixError ->
// MSCG_ERR_SINGULAR (+ block, pivot_index), CUDA failures -> MSCG_ERR_CUDA.
#include "mscg.h"

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "device/common.cuh"
#include "device/internal.hpp"
#include "host/setup.hpp"

struct mscg_ctx {
  mscg::Ctx ctx;
  std::mutex mu;
  mscg::DevBuf scratch;  // device vectors of host-mode calls (guarded by mu)
};
struct mscg_csr {
  std::unique_ptr<mscg::DevCsr> owned;
  mscg::DevCsr* a = nullptr;
  mscg_ctx* ctx = nullptr;
  mscg::Precond* owner = nullptr;  // set for a preconditioner's own C (saddle layout known)
};
struct mscg_precond {
  std::unique_ptr<mscg::Precond> pc;
  mscg_ctx* ctx = nullptr;
  mscg_csr matrix;  // borrowed view of pc->C
};
struct mscg_factors {
  std::unique_ptr<mscg::FactorSet> fs;
  mscg_ctx* ctx = nullptr;
};
struct mscg_problem {
  mscg::host::Partitioned pm;
  std::vector<double> scaled_rhs;
  bool have_schur = false;
  mscg::host::SchurApprox schur;
  std::vector<int> d_ranges_flat, s_ranges_flat;
};

namespace {

void set_status(mscg_status* st, int code, const std::string& msg, int block = -1, int piv = -1) {
  if (!st) return;
  st->code = code;
  st->block = block;
  st->pivot_index = piv;
  std::strncpy(st->message, msg.c_str(), sizeof(st->message) - 1);
  st->message[sizeof(st->message) - 1] = 0;
}

template <class F>
int guard(mscg_status* st, F&& f) {
  try {
    f();
    set_status(st, MSCG_OK, "");
    return MSCG_OK;
  } catch (const mscg::Error& e) {
    set_status(st, e.code, e.what(), e.block, e.pivot);
    return e.code;
  } catch (const mscg::host::SingularError& e) {
    set_status(st, MSCG_ERR_SINGULAR, e.what(), -1, e.pivot);
    return MSCG_ERR_SINGULAR;
  } catch (const std::invalid_argument& e) {
    set_status(st, MSCG_ERR_INVALID_ARGUMENT, e.what());
    return MSCG_ERR_INVALID_ARGUMENT;
  } catch (const mscg::host::IoError& e) {
    set_status(st, MSCG_ERR_IO, e.what());
    return MSCG_ERR_IO;
  } catch (const std::bad_alloc& e) {
    set_status(st, MSCG_ERR_OUT_OF_MEMORY, "host out of memory");
    return MSCG_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_status(st, MSCG_ERR_RUNTIME, e.what());
    return MSCG_ERR_RUNTIME;
  }
}

void flatten(const std::vector<std::pair<int, int>>& r, std::vector<int>& out) {
  out.clear();
  for (auto [b, e] : r) {
    out.push_back(b);
    out.push_back(e);
  }
}

std::vector<std::pair<int, int>> pairs(int n, const int* flat) {
  std::vector<std::pair<int, int>> r;
  for (int i = 0; i < n; ++i) r.push_back({flat[2 * i], flat[2 * i + 1]});
  return r;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Run `f(dev_in, dev_out)` with host or device vectors.
template <class F>
void with_vectors(mscg_ctx* c, const double* in, size_t nin, double* out, size_t nout, int mem,
                  F&& f) {
  cudaStream_t s = c->ctx.stream;
  if (mem == MSCG_MEM_DEVICE) {
    f(in, out);
    return;
  }
  std::lock_guard<std::mutex> lk(c->mu);
  const size_t need = sizeof(double) * (std::max<size_t>(1, nin) + std::max<size_t>(1, nout));
  if (c->scratch.bytes < need) c->scratch = mscg::DevBuf(need);  // grow-only
  double* const d_in = c->scratch.as<double>();
  double* const d_out = d_in + std::max<size_t>(1, nin);
  // Page-locked caller buffers are copied directly; pageable ones go
  // through the context's pinned staging buffer.
  const bool pin_in = is_pinned(in), pin_out = is_pinned(out);
  double* stage = (pin_in && pin_out) ? nullptr : c->ctx.stage(std::max(nin, nout));
  const double* src = in;
  if (!pin_in) {
    std::memcpy(stage, in, sizeof(double) * nin);
    src = stage;
  }
  MSCG_CUDA(cudaMemcpyAsync(d_in, src, sizeof(double) * nin, cudaMemcpyHostToDevice, s));
  f(d_in, d_out);
  MSCG_CUDA(cudaMemcpyAsync(pin_out ? out : stage, d_out, sizeof(double) * nout,
                            cudaMemcpyDeviceToHost, s));
  MSCG_CUDA(cudaStreamSynchronize(s));
  if (!pin_out) std::memcpy(out, stage, sizeof(double) * nout);
}

}  // namespace

extern "C" {

int mscg_abi_version(void) { return MSCG_ABI_VERSION; }

int mscg_ctx_create(int device, mscg_ctx** out, mscg_status* st) {
  return guard(st, [&] {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      throw mscg::Error(MSCG_ERR_CUDA, std::string("no CUDA device available (") +
                                           cudaGetErrorString(e) + "); this library has no CPU path");
    if (device < 0 || device >= count) throw std::invalid_argument("mscg_ctx_create: bad device");
    auto c = std::make_unique<mscg_ctx>();
    c->ctx.device = device;
    MSCG_CUDA(cudaSetDevice(device));
    MSCG_CUDA(cudaStreamCreateWithFlags(&c->ctx.owned_stream, cudaStreamNonBlocking));
    c->ctx.stream = c->ctx.owned_stream;
    MSCG_CUDA(cudaDeviceGetAttribute(&c->ctx.sm_count, cudaDevAttrMultiProcessorCount, device));
    *out = c.release();
  });
}

void mscg_ctx_destroy(mscg_ctx* ctx) { delete ctx; }

int mscg_ctx_set_stream(mscg_ctx* ctx, void* stream, int use_own, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx) throw std::invalid_argument("mscg_ctx_set_stream: null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    MSCG_CUDA(cudaStreamSynchronize(ctx->ctx.stream));
    ctx->ctx.stream = use_own ? ctx->ctx.owned_stream : static_cast<cudaStream_t>(stream);
  });
}
void* mscg_ctx_stream(mscg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->ctx.stream) : nullptr; }
int mscg_ctx_synchronize(mscg_ctx* ctx, mscg_status* st) {
  return guard(st, [&] { MSCG_CUDA(cudaStreamSynchronize(ctx->ctx.stream)); });
}
int64_t mscg_ctx_launches(mscg_ctx* ctx) { return ctx ? ctx->ctx.launches : 0; }
int mscg_ctx_set_correction(mscg_ctx* ctx, int mode, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx) throw std::invalid_argument("mscg_ctx_set_correction: null context");
    if (mode < -1 || mode > MSCG_CORRECTION_AUTO)
      throw std::invalid_argument("mscg_ctx_set_correction: mode must be -1, 0, 1 or 2");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->ctx.correction = mode;
  });
}

// ---- host problem layer ---------------------------------------------------

int mscg_problem_oseen(int grid_n, double nu, int stretched, double stretch, int n_a,
                       int anchored, int threads, mscg_problem** out, mscg_status* st) {
  return guard(st, [&] {
    using clk = std::chrono::steady_clock;
    auto pb = std::make_unique<mscg_problem>();
    const auto t0 = clk::now();
    mscg::host::OseenSystem sys = mscg::host::generate_oseen(grid_n, nu, stretched != 0, stretch);
    const auto t1 = clk::now();
    mscg::host::scale_rows(sys.C, sys.rhs);
    const auto t2 = clk::now();
    pb->pm = mscg::host::partition_saddle(sys.C, sys.p, n_a, threads);
    const auto t3 = clk::now();
    if (anchored) mscg::host::anchor_interface(pb->pm);
    const auto t4 = clk::now();
    if (getenv("MSCG_VERBOSE")) {
      auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
      fprintf(stderr, "problem_oseen: generate %.3f s, scale %.3f s, partition %.3f s, anchor %.3f s\n",
              sec(t0, t1), sec(t1, t2), sec(t2, t3), sec(t3, t4));
    }
    pb->scaled_rhs.resize(sys.rhs.size());
    for (size_t k = 0; k < sys.rhs.size(); ++k) pb->scaled_rhs[k] = sys.rhs[pb->pm.perm[k]];
    flatten(pb->pm.d_ranges, pb->d_ranges_flat);
    *out = pb.release();
  });
}

int mscg_problem_oseen_device(mscg_ctx* ctx, int grid_n, double nu, int stretched,
                              double stretch, int n_a, int anchored, int threads,
                              mscg_problem** out, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx) throw std::invalid_argument("generate_oseen: null context");
    mscg::host::check_oseen_args(grid_n, nu, stretched != 0, stretch);
    auto pb = std::make_unique<mscg_problem>();
    std::vector<double> x, y, xc, yc;
    mscg::host::oseen_grid(grid_n, stretched != 0, stretch, x, y, xc, yc);
    mscg::host::OseenSystem sys;
    {
      std::lock_guard<std::mutex> lk(ctx->mu);
      mscg::oseen_assemble_device(&ctx->ctx, grid_n, x, y, xc, yc, nu, sys.C.rp, sys.C.ci,
                                  sys.C.v, sys.rhs, sys.p);
    }
    sys.C.nrows = sys.C.ncols = static_cast<int>(sys.C.rp.size()) - 1;
    // nested dissection on the device too;
    // MSCG_DISSECT=host keeps the host version (comparisons)
    static const bool host_nd = [] {
      const char* e = getenv("MSCG_DISSECT");
      return e && std::string(e) == "host";
    }();
    if (host_nd) {
      pb->pm = mscg::host::partition_saddle(sys.C, sys.p, n_a, threads);
      if (anchored) mscg::host::anchor_interface(pb->pm);
    } else {
      // the whole partition (and anchoring) on the device
      std::lock_guard<std::mutex> lk(ctx->mu);
      pb->pm = mscg::partition_saddle_device(&ctx->ctx, sys.C, sys.p, n_a, anchored != 0);
    }
    pb->scaled_rhs.resize(sys.rhs.size());
    for (size_t k = 0; k < sys.rhs.size(); ++k) pb->scaled_rhs[k] = sys.rhs[pb->pm.perm[k]];
    flatten(pb->pm.d_ranges, pb->d_ranges_flat);
    *out = pb.release();
  });
}

int mscg_nested_dissection(mscg_ctx* ctx, int n, const int* rp, const int* ci, int target,
                           int threads, int* perm, int* nblocks, int* ranges, int cap,
                           mscg_status* st) {
  return guard(st, [&] {
    if (n < 0 || !rp || !perm || !nblocks) throw std::invalid_argument("nested_dissection: bad arguments");
    std::vector<int64_t> off;
    std::vector<int> adj;
    mscg::host::undirected_graph(n, rp, ci, off, adj);
    std::vector<std::vector<int>> blocks;
    std::vector<int> sep;
    if (ctx) {
      std::lock_guard<std::mutex> lk(ctx->mu);
      mscg::nested_dissection_device(&ctx->ctx, n, off.data(), adj.data(), target, blocks, sep);
    } else {
      if (target < 1 || target > std::max(n, 1))
        throw std::invalid_argument("nested_dissection: target_blocks out of range");
      mscg::host::nested_dissection_host(n, off.data(), adj.data(), target, threads, blocks, sep);
    }
    int w = 0, b = 0;
    for (const auto& blk : blocks) {
      if (ranges && b < cap) {
        ranges[2 * b] = w;
        ranges[2 * b + 1] = w + static_cast<int>(blk.size());
      }
      for (int u : blk) perm[w++] = u;
      ++b;
    }
    for (int u : sep) perm[w++] = u;
    *nblocks = b;
  });
}

int mscg_problem_from_csr(int n, const int* rp, const int* ci, const double* v, int p,
                          int nranges, const int* ranges, mscg_problem** out, mscg_status* st) {
  return guard(st, [&] {
    if (n < 0 || p < 0 || p > n) throw std::invalid_argument("PartitionedMatrix: split out of range");
    auto pb = std::make_unique<mscg_problem>();
    mscg::host::Csr& c = pb->pm.C;
    c = mscg::host::Csr(n, n);
    c.rp.assign(rp, rp + n + 1);
    c.ci.assign(ci, ci + rp[n]);
    c.v.assign(v, v + rp[n]);
    pb->pm.p = p;
    if (nranges > 0) pb->pm.d_ranges = pairs(nranges, ranges);
    else pb->pm.d_ranges = {{0, p}};
    pb->pm.perm.resize(n);
    for (int i = 0; i < n; ++i) pb->pm.perm[i] = i;
    flatten(pb->pm.d_ranges, pb->d_ranges_flat);
    *out = pb.release();
  });
}

void mscg_problem_destroy(mscg_problem* pb) { delete pb; }

void mscg_problem_dims(const mscg_problem* pb, int* n, int* p, int* nblocks, int64_t* nnz_c,
                       int* separator_size) {
  if (n) *n = pb->pm.n();
  if (p) *p = pb->pm.p;
  if (nblocks) *nblocks = static_cast<int>(pb->pm.d_ranges.size());
  if (nnz_c) *nnz_c = pb->pm.C.nnz();
  if (separator_size) *separator_size = pb->pm.separator_size;
}

int mscg_problem_csr(const mscg_problem* pb, int which, int* nrows, int* ncols, int64_t* nnz,
                     const int** rp, const int** ci, const double** v) {
  const mscg::host::Csr* a = nullptr;
  if (which == 0) a = &pb->pm.C;
  if (which == 5 && pb->have_schur) a = &pb->schur.s_hat;
  if (!a) return MSCG_ERR_INVALID_ARGUMENT;
  *nrows = a->nrows;
  *ncols = a->ncols;
  *nnz = a->nnz();
  *rp = a->rp.data();
  *ci = a->ci.data();
  *v = a->v.data();
  return MSCG_OK;
}

const int* mscg_problem_perm(const mscg_problem* pb) { return pb->pm.perm.data(); }
const int* mscg_problem_d_ranges(const mscg_problem* pb) { return pb->d_ranges_flat.data(); }
const double* mscg_problem_scaled_rhs(const mscg_problem* pb) {
  return pb->scaled_rhs.empty() ? nullptr : pb->scaled_rhs.data();
}

namespace {
std::vector<int> schur_sizes(const mscg_problem* pb, int mode, int sz, int nsizes,
                             const int* sizes) {
  const int ng = pb->pm.n_g();
  if (mode == 2) return std::vector<int>(sizes, sizes + nsizes);
  if (mode == 1) return mscg::host::anchored_sizes(pb->pm, sz);
  int s = sz <= 0 ? std::max(1, ng / 8) : sz;
  s = std::min(s, ng);
  return mscg::host::equal_sizes(ng, s);
}

// build_msc on the host (ctx == NULL) or the device; widths empty for the
// non-overlapped aggregate sets.
void build_schur_impl(mscg_ctx* ctx, mscg_problem* pb, const char* variant,
                      const std::vector<int>& sz_list, const std::vector<int>& widths,
                      int threads) {
  const mscg::host::Variant v = mscg::host::variant_from_name(variant ? variant : "");
  if (!ctx) {
    pb->schur = mscg::host::build_msc(pb->pm, sz_list, v, threads, widths);
  } else {
    mscg::host::SchurApprox out;
    mscg::host::aggregate_spans(pb->pm, sz_list, v, widths, out.ranges, out.spans);
    out.overlapped = mscg::host::variant_overlapped(v);
    const int kind = mscg::host::variant_lumped(v)   ? mscg::kMscLum
                     : mscg::host::variant_rowsum(v) ? mscg::kMscMscnr
                                                     : mscg::kMscMscn;
    std::lock_guard<std::mutex> lk(ctx->mu);
    const auto& c = pb->pm.C;
    const int ng = pb->pm.n_g();
    out.s_hat = mscg::host::Csr(ng, ng);
    mscg::build_msc_device(&ctx->ctx, c.nrows, pb->pm.p, c.rp.data(), c.ci.data(), c.v.data(),
                           out.ranges, out.spans, kind, out.s_hat.rp, out.s_hat.ci, out.s_hat.v);
    pb->schur = std::move(out);
  }
  pb->have_schur = true;
  flatten(pb->schur.ranges, pb->s_ranges_flat);
}
}  // namespace

int mscg_problem_build_schur(mscg_problem* pb, const char* variant, int mode, int sz, int nsizes,
                             const int* sizes, int threads, mscg_status* st) {
  return guard(st, [&] {
    build_schur_impl(nullptr, pb, variant, schur_sizes(pb, mode, sz, nsizes, sizes), {}, threads);
  });
}

int mscg_problem_build_schur_device(mscg_ctx* ctx, mscg_problem* pb, const char* variant,
                                    int mode, int sz, int nsizes, const int* sizes,
                                    mscg_status* st) {
  return guard(st, [&] {
    if (!ctx) throw std::invalid_argument("build_msc: null context");
    build_schur_impl(ctx, pb, variant, schur_sizes(pb, mode, sz, nsizes, sizes), {}, 0);
  });
}

int mscg_problem_build_schur_overlapped(mscg_ctx* ctx, mscg_problem* pb, const char* variant,
                                        int mode, int sz, int nsizes, const int* sizes,
                                        int overlap, int nwidths, const int* widths,
                                        int threads, mscg_status* st) {
  return guard(st, [&] {
    if (!pb) throw std::invalid_argument("build_msc: null problem");
    const std::vector<int> sz_list = schur_sizes(pb, mode, sz, nsizes, sizes);
    std::vector<int> w;
    if (widths) {
      if (nwidths < 0) throw std::invalid_argument("aggregate_overlapped: one width per aggregate");
      w.assign(widths, widths + nwidths);
      if (w.size() != sz_list.size())
        throw std::invalid_argument("aggregate_overlapped: one width per aggregate");
    } else {
      const int ng = pb->pm.n_g();
      int s = sz <= 0 ? std::max(1, ng / 8) : std::min(sz, ng);
      w = mscg::host::overlap_widths(ng, sz_list, s, overlap);
    }
    build_schur_impl(ctx, pb, variant, sz_list, w, threads);
  });
}

int mscg_problem_num_aggregates(const mscg_problem* pb) {
  return pb->have_schur ? static_cast<int>(pb->schur.ranges.size()) : -1;
}
const int* mscg_problem_schur_ranges(const mscg_problem* pb) {
  return pb->have_schur ? pb->s_ranges_flat.data() : nullptr;
}

// ---- device sparse matrices ---------------------------------------------

int mscg_csr_upload(mscg_ctx* ctx, int nrows, int ncols, const int* rp, const int* ci,
                    const double* v, mscg_csr** out, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx) throw std::invalid_argument("mscg_csr_upload: null context");
    if (nrows < 0 || ncols < 0) throw std::invalid_argument("SparseMatrix: negative dimension");
    auto h = std::make_unique<mscg_csr>();
    h->owned = mscg::upload_csr(&ctx->ctx, nrows, ncols, rp, ci, v);
    h->a = h->owned.get();
    h->ctx = ctx;
    *out = h.release();
  });
}

void mscg_csr_destroy(mscg_csr* a) { delete a; }

int mscg_spmv(mscg_csr* a, const double* x, double* y, int mem, mscg_status* st) {
  return guard(st, [&] {
    if (!a || !a->a) throw std::invalid_argument("matvec: null matrix (a shard has no full C)");
    if (mem == MSCG_MEM_HOST && a->owner && is_pinned(x) && is_pinned(y)) {
      // C of a preconditioner: block-chunked, copies overlapped with the rows
      mscg_ctx* c = a->ctx;
      std::lock_guard<std::mutex> lk(c->mu);
      const size_t n = a->a->nrows;
      const size_t need = sizeof(double) * 2 * std::max<size_t>(1, n);
      if (c->scratch.bytes < need) c->scratch = mscg::DevBuf(need);
      double* d_x = c->scratch.as<double>();
      double* d_y = d_x + std::max<size_t>(1, n);
      a->owner->spmv_host(x, y, d_x, d_y, c->ctx.stream);
      MSCG_CUDA(cudaStreamSynchronize(c->ctx.stream));
      return;
    }
    with_vectors(a->ctx, x, a->a->ncols, y, a->a->nrows, mem, [&](const double* dx, double* dy) {
      mscg::spmv(*a->a, dx, dy, nullptr, 0, a->ctx->ctx.stream);
    });
  });
}

// ---- preconditioner ------------------------------------------------------

int mscg_precond_build(mscg_ctx* ctx, int n, int p, const int* c_rp, const int* c_ci,
                       const double* c_v, int nblocks, const int* d_ranges, const int* s_rp,
                       const int* s_ci, const double* s_v, int nschur, const int* s_ranges,
                       double tol_a, int s_a, mscg_precond** out, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx) throw std::invalid_argument("build_preconditioner: null context");
    if (tol_a < 0.0) throw std::invalid_argument("factor_ilut: negative drop tolerance");
    auto h = std::make_unique<mscg_precond>();
    h->ctx = ctx;
    const bool single = nschur == MSCG_SCHUR_SINGLE;
    if (nschur < 0 && !single) throw std::invalid_argument("build_preconditioner: bad Schur range count");
    h->pc = mscg::build_precond(&ctx->ctx, n, p, c_rp, c_ci, c_v, pairs(nblocks, d_ranges), s_rp,
                                s_ci, s_v, single ? std::vector<std::pair<int, int>>{}
                                                  : pairs(nschur, s_ranges),
                                tol_a, s_a, 0, -1, single);
    h->matrix.a = h->pc->C.get();
    h->matrix.ctx = ctx;
    h->matrix.owner = h->pc.get();
    *out = h.release();
  });
}

int mscg_factor(mscg_ctx* ctx, int n, const int* rp, const int* ci, const double* v, int kind,
                double tol, mscg_factors** out, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx || !out) throw std::invalid_argument("factor: null context or output");
    if (kind != 0 && kind != 1) throw std::invalid_argument("factor: kind must be 0 or 1");
    if (kind == 0 && tol < 0.0) throw std::invalid_argument("factor_ilut: negative drop tolerance");
    if (n < 1) throw std::invalid_argument(kind ? "factor_exact: empty matrix"
                                                : "factor_ilut: empty matrix");
    cudaStream_t s = ctx->ctx.stream;
    const int64_t nnz = rp[n];
    mscg::DevBuf drp(sizeof(int) * (n + 1)), dci(sizeof(int) * std::max<int64_t>(1, nnz)),
        dv(sizeof(double) * std::max<int64_t>(1, nnz));
    MSCG_CUDA(cudaMemcpyAsync(drp.p, rp, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s));
    if (nnz) {
      MSCG_CUDA(cudaMemcpyAsync(dci.p, ci, sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
      MSCG_CUDA(cudaMemcpyAsync(dv.p, v, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    }
    auto h = std::make_unique<mscg_factors>();
    h->ctx = ctx;
    h->fs = mscg::factor_blocks(&ctx->ctx, drp.as<int>(), dci.as<int>(), dv.as<double>(),
                                {mscg::BlockSpec{0, n, 0}}, {static_cast<char>(kind)}, tol, "",
                                nullptr);
    MSCG_CUDA(cudaStreamSynchronize(s));
    *out = h.release();
  });
}

int mscg_factors_get(const mscg_factors* f, int* dim, int64_t* nnz_l, int64_t* nnz_u, int* lrp,
                     int* lci, double* lv, int* urp, int* uci, double* uv, int* perm,
                     mscg_status* st) {
  return guard(st, [&] {
    if (!f) throw std::invalid_argument("factors: null handle");
    const auto& fs = *f->fs;
    const int d = fs.h_dim[0];
    if (dim) *dim = d;
    if (nnz_l) *nnz_l = fs.h_nnz_l[0];
    if (nnz_u) *nnz_u = fs.h_nnz_u[0] + d;
    if (!lrp) return;
    std::vector<int> a, b2, c2, d2, e2;
    std::vector<double> f2, g2;
    mscg::download_factor(fs, 0, a, b2, f2, c2, d2, g2, e2);
    std::memcpy(lrp, a.data(), sizeof(int) * a.size());
    std::memcpy(lci, b2.data(), sizeof(int) * b2.size());
    std::memcpy(lv, f2.data(), sizeof(double) * f2.size());
    std::memcpy(urp, c2.data(), sizeof(int) * c2.size());
    std::memcpy(uci, d2.data(), sizeof(int) * d2.size());
    std::memcpy(uv, g2.data(), sizeof(double) * g2.size());
    if (perm) std::memcpy(perm, e2.data(), sizeof(int) * e2.size());
  });
}

int mscg_factors_solve(mscg_factors* f, const double* b, double* x, int mem, mscg_status* st) {
  return guard(st, [&] {
    if (!f) throw std::invalid_argument("solve: null factors");
    const size_t n = f->fs->h_dim[0];
    with_vectors(f->ctx, b, n, x, n, mem, [&](const double* db, double* dx) {
      mscg::block_trisolve(*f->fs, db, dx, nullptr, f->ctx->ctx.stream);
      f->ctx->ctx.launches++;
    });
  });
}

void mscg_factors_destroy(mscg_factors* f) { delete f; }

int mscg_precond_build_problem(mscg_ctx* ctx, const mscg_problem* pb, double tol_a, int s_a,
                               mscg_precond** out, mscg_status* st) {
  if (!pb || !pb->have_schur) {
    set_status(st, MSCG_ERR_INVALID_ARGUMENT,
               "build_preconditioner: Schur approximation does not match the split");
    return MSCG_ERR_INVALID_ARGUMENT;
  }
  const auto& c = pb->pm.C;
  const auto& s = pb->schur.s_hat;
  return mscg_precond_build(ctx, c.nrows, pb->pm.p, c.rp.data(), c.ci.data(), c.v.data(),
                            static_cast<int>(pb->pm.d_ranges.size()), pb->d_ranges_flat.data(),
                            s.rp.data(), s.ci.data(), s.v.data(),
                            pb->schur.overlapped ? MSCG_SCHUR_SINGLE
                                                 : static_cast<int>(pb->schur.ranges.size()),
                            pb->s_ranges_flat.data(), tol_a, s_a, out, st);
}

int mscg_precond_build_shard(mscg_ctx* ctx, int n, int p, const int* c_rp, const int* c_ci,
                             const double* c_v, int nblocks, const int* d_ranges,
                             const int* s_rp, const int* s_ci, const double* s_v, int nschur,
                             const int* s_ranges, double tol_a, int s_a, int block_begin,
                             int block_end, mscg_precond** out, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx) throw std::invalid_argument("build_preconditioner: null context");
    if (tol_a < 0.0) throw std::invalid_argument("factor_ilut: negative drop tolerance");
    if (block_begin < 0 || block_end <= block_begin || block_end > nblocks)
      throw std::invalid_argument("build_preconditioner: shard block range out of range");
    auto h = std::make_unique<mscg_precond>();
    h->ctx = ctx;
    const bool single = nschur == MSCG_SCHUR_SINGLE;
    if (nschur < 0 && !single) throw std::invalid_argument("build_preconditioner: bad Schur range count");
    h->pc = mscg::build_precond(&ctx->ctx, n, p, c_rp, c_ci, c_v, pairs(nblocks, d_ranges), s_rp,
                                s_ci, s_v, single ? std::vector<std::pair<int, int>>{}
                                                  : pairs(nschur, s_ranges),
                                tol_a, s_a, block_begin, block_end, single);
    h->matrix.a = h->pc->C.get();  // null for a true shard
    h->matrix.ctx = ctx;
    *out = h.release();
  });
}

int mscg_precond_build_problem_shard(mscg_ctx* ctx, const mscg_problem* pb, double tol_a,
                                     int s_a, int block_begin, int block_end,
                                     mscg_precond** out, mscg_status* st) {
  if (!pb || !pb->have_schur) {
    set_status(st, MSCG_ERR_INVALID_ARGUMENT,
               "build_preconditioner: Schur approximation does not match the split");
    return MSCG_ERR_INVALID_ARGUMENT;
  }
  const auto& c = pb->pm.C;
  const auto& s = pb->schur.s_hat;
  return mscg_precond_build_shard(
      ctx, c.nrows, pb->pm.p, c.rp.data(), c.ci.data(), c.v.data(),
      static_cast<int>(pb->pm.d_ranges.size()), pb->d_ranges_flat.data(), s.rp.data(),
      s.ci.data(), s.v.data(),
      pb->schur.overlapped ? MSCG_SCHUR_SINGLE : static_cast<int>(pb->schur.ranges.size()),
      pb->s_ranges_flat.data(), tol_a, s_a, block_begin, block_end, out, st);
}

int mscg_precond_shard_rows(const mscg_precond* pc, int* row_lo, int* row_hi) {
  if (!pc) return MSCG_ERR_INVALID_ARGUMENT;
  const auto& sh = pc->pc->shard;
  if (row_lo) *row_lo = sh.on ? sh.row_lo : 0;
  if (row_hi) *row_hi = sh.on ? sh.row_hi : pc->pc->p;
  return MSCG_OK;
}

int mscg_precond_apply_shard(mscg_precond* pc, int phase, const double* y, double* t, double* x,
                             mscg_status* st) {
  return guard(st, [&] {
    if (!pc || !pc->pc->shard.on)
      throw std::invalid_argument("mscg_precond_apply_shard: not a shard preconditioner");
    cudaStream_t s = pc->ctx->ctx.stream;
    if (phase == 0)
      pc->pc->apply_shard_begin(y, t, s);
    else if (phase == 1)
      pc->pc->apply_shard_end(y, t, x, s);
    else
      throw std::invalid_argument("mscg_precond_apply_shard: phase must be 0 or 1");
  });
}

int mscg_precond_spmv_shard(mscg_precond* pc, const double* x, double* y, double* y2part,
                            int with_interface_block, mscg_status* st) {
  return guard(st, [&] {
    if (!pc || !pc->pc->shard.on)
      throw std::invalid_argument("mscg_precond_spmv_shard: not a shard preconditioner");
    pc->pc->spmv_shard(x, y, y2part, with_interface_block != 0, pc->ctx->ctx.stream);
  });
}

void mscg_precond_destroy(mscg_precond* pc) { delete pc; }

int mscg_precond_apply(mscg_precond* pc, const double* y, double* x, int mem, mscg_status* st) {
  return guard(st, [&] {
    if (!pc) throw std::invalid_argument("MscPreconditioner::apply: null preconditioner");
    const size_t n = pc->pc->n;
    if (mem == MSCG_MEM_DEVICE) {
      // concurrent applies are safe: per-stream scratch (Precond::apply);
      // the stream is read under the context lock (mscg_ctx_set_stream)
      cudaStream_t s;
      {
        std::lock_guard<std::mutex> lk(pc->ctx->mu);
        s = pc->ctx->ctx.stream;
      }
      pc->pc->apply(y, x, s);
      return;
    }
    // Host vectors: chunked apply, copies of one block chunk overlap the
    // solves of the others (pageable buffers go through pinned staging).
    mscg_ctx* c = pc->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    const size_t need = sizeof(double) * 2 * std::max<size_t>(1, n);
    if (c->scratch.bytes < need) c->scratch = mscg::DevBuf(need);
    double* d_y = c->scratch.as<double>();
    double* d_x = d_y + std::max<size_t>(1, n);
    const bool pin_in = is_pinned(y), pin_out = is_pinned(x);
    double* stage = (pin_in && pin_out) ? nullptr : c->ctx.stage(2 * n);
    const double* src = y;
    double* dst = x;
    if (!pin_in) {
      std::memcpy(stage, y, sizeof(double) * n);
      src = stage;
    }
    if (!pin_out) dst = stage + n;
    cudaStream_t s = c->ctx.stream;
    pc->pc->apply_host(src, dst, d_y, d_x, s);
    MSCG_CUDA(cudaStreamSynchronize(s));
    if (!pin_out) std::memcpy(x, dst, sizeof(double) * n);
  });
}

int mscg_precond_apply_stream(mscg_precond* pc, const double* y_dev, double* x_dev, void* stream,
                              mscg_status* st) {
  return guard(st, [&] {
    if (!pc) throw std::invalid_argument("MscPreconditioner::apply: null preconditioner");
    pc->pc->apply(y_dev, x_dev, static_cast<cudaStream_t>(stream));
  });
}

int64_t mscg_precond_stored_nnz(const mscg_precond* pc) { return pc ? pc->pc->stored_nnz : -1; }

int mscg_precond_dims(const mscg_precond* pc, int* n, int* p, int* nblocks, int* nschur) {
  if (!pc) return MSCG_ERR_INVALID_ARGUMENT;
  if (n) *n = pc->pc->n;
  if (p) *p = pc->pc->p;
  if (nblocks) *nblocks = pc->pc->D ? pc->pc->D->nblocks : 0;
  if (nschur) *nschur = pc->pc->S ? pc->pc->S->nblocks : 0;
  return MSCG_OK;
}

int mscg_precond_factor(const mscg_precond* pc, int kind, int idx, int* dim, int64_t* nnz_l,
                        int64_t* nnz_u, int* lrp, int* lci, double* lv, int* urp, int* uci,
                        double* uv, int* perm, mscg_status* st) {
  return guard(st, [&] {
    const mscg::FactorSet* fs = kind == 0 ? pc->pc->D.get() : pc->pc->S.get();
    if (!fs || idx < 0 || idx >= fs->nblocks) throw std::invalid_argument("factor index out of range");
    const int d = fs->h_dim[idx];
    if (dim) *dim = d;
    if (nnz_l) *nnz_l = fs->h_nnz_l[idx];
    if (nnz_u) *nnz_u = fs->h_nnz_u[idx] + d;
    if (!lrp) return;
    std::vector<int> a, b2, c2, d2, e2;
    std::vector<double> f2, g2;
    mscg::download_factor(*fs, idx, a, b2, f2, c2, d2, g2, e2);
    std::memcpy(lrp, a.data(), sizeof(int) * a.size());
    std::memcpy(lci, b2.data(), sizeof(int) * b2.size());
    std::memcpy(lv, f2.data(), sizeof(double) * f2.size());
    std::memcpy(urp, c2.data(), sizeof(int) * c2.size());
    std::memcpy(uci, d2.data(), sizeof(int) * d2.size());
    std::memcpy(uv, g2.data(), sizeof(double) * g2.size());
    if (perm) std::memcpy(perm, e2.data(), sizeof(int) * e2.size());
  });
}

int mscg_precond_use_correction(mscg_precond* pc, int on) {
  if (!pc) return MSCG_ERR_INVALID_ARGUMENT;
  pc->pc->use_corr = on != 0;
  return MSCG_OK;
}

int mscg_precond_layout_bytes(const mscg_precond* pc, int64_t out[10]) {
  if (!pc) return MSCG_ERR_INVALID_ARGUMENT;
  for (int k = 0; k < 10; ++k) out[k] = 0;
  auto pass_bytes = [](const mscg::FactorSet& f) -> int64_t {
    // one solve pass reads: every near tile's copied prefix, the far
    // entries (fp64 + uint16 column), their row offsets, the work items
    // (int4), the U diagonal and reciprocal; rhs in + x out
    int64_t b = 0;
    for (int w : f.h_lwidth) b += 8 * static_cast<int64_t>(mscg::tile_elems(w));
    for (int w : f.h_uwidth) b += 8 * static_cast<int64_t>(mscg::tile_elems(w));
    b += 10 * (f.far_l() + f.far_u());
    b += 8 * static_cast<int64_t>(f.total_rows + f.nblocks);
    if (!f.h_lioff.empty()) b += 16 * (f.h_lioff.back() + f.h_uioff.back());
    b += 16 * static_cast<int64_t>(f.total_rows) * 2;
    return b;
  };
  const auto& p = *pc->pc;
  auto csr_bytes = [](const mscg::DevCsr* a) -> int64_t {
    return a ? 12 * a->padded + 8 * static_cast<int64_t>(a->nslices + 1) : 0;
  };
  if (p.D) out[0] = pass_bytes(*p.D);
  if (p.S) out[1] = pass_bytes(*p.S);
  if (p.corr) out[2] = 8 * p.corr->entries + 16 * static_cast<int64_t>(p.p);
  out[3] = csr_bytes(p.E.get()) + csr_bytes(p.F.get());
  out[4] = csr_bytes(p.C.get());
  out[5] = static_cast<int64_t>(p.n) * 8 * 4;  // y, x, z1 and interface vectors
  if (p.D) {  // breakdown of one interior solve pass
    const auto& f = *p.D;
    for (int w : f.h_lwidth) out[6] += 8 * static_cast<int64_t>(mscg::tile_elems(w));
    for (int w : f.h_uwidth) out[6] += 8 * static_cast<int64_t>(mscg::tile_elems(w));
    out[7] = 10 * (f.far_l() + f.far_u());
    if (!f.h_lioff.empty()) out[8] = 16 * (f.h_lioff.back() + f.h_uioff.back());
    int64_t dense = 0;
    for (int w : f.h_lwidth) dense += w == mscg::kDenseNbr;
    for (int w : f.h_uwidth) dense += w == mscg::kDenseNbr;
    out[9] = dense;  // near tiles kept dense (of 2 * tiles)
  }
  return MSCG_OK;
}

int mscg_precond_build_times(const mscg_precond* pc, double* ilut_s, double* schur_lu_s,
                             double* pack_s) {
  if (!pc) return MSCG_ERR_INVALID_ARGUMENT;
  if (ilut_s) *ilut_s = pc->pc->times.ilut_s;
  if (schur_lu_s) *schur_lu_s = pc->pc->times.lu_s;
  if (pack_s) *pack_s = pc->pc->times.pack_s;
  return MSCG_OK;
}

int mscg_precond_correction(const mscg_precond* pc, int* on, int64_t* entries, int* kmax,
                            double* build_s) {
  if (!pc) return MSCG_ERR_INVALID_ARGUMENT;
  const auto* c = pc->pc->corr.get();
  if (on) *on = c ? 1 : 0;
  if (entries) *entries = c ? c->entries : 0;
  if (kmax) *kmax = c ? c->kmax : 0;
  if (build_s) *build_s = c ? c->build_s : 0.0;
  return MSCG_OK;
}

mscg_csr* mscg_precond_matrix(mscg_precond* pc) { return pc ? &pc->matrix : nullptr; }

int mscg_precond_nnz(const mscg_precond* pc, int64_t counts[7]) {
  if (!pc) return MSCG_ERR_INVALID_ARGUMENT;
  const auto& p = *pc->pc;
  counts[0] = p.D ? p.D->nnz_l() : 0;
  counts[1] = p.D ? p.D->nnz_u() : 0;
  counts[2] = p.S ? p.S->nnz_l() : 0;
  counts[3] = p.S ? p.S->nnz_u() : 0;
  counts[4] = p.E ? p.E->nnz : 0;
  counts[5] = p.F ? p.F->nnz : 0;
  counts[6] = p.C ? p.C->nnz : (p.shard.Cr ? p.shard.Cr->nnz : 0);
  return MSCG_OK;
}

void mscg_random_vector(int n, unsigned seed, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int i = 0; i < n; ++i) out[i] = dist(rng);
}

int mscg_debug_trace_dsolve(mscg_precond* pc, const double* y, double* x, int64_t* out, int cap,
                            mscg_status* st) {
  int dim0 = -1;
  int rc = guard(st, [&] {
    const mscg::FactorSet& fs = *pc->pc->D;
    dim0 = fs.h_dim[0];
    if (cap < 32 * dim0) throw std::invalid_argument("trace buffer too small");
    mscg::DevBuf tr(sizeof(long long) * 32 * dim0);
    cudaStream_t s = pc->ctx->ctx.stream;
    MSCG_CUDA(cudaMemsetAsync(tr.p, 0, tr.bytes, s));
    mscg::block_trisolve(fs, y, x, nullptr, s, tr.as<long long>());
    MSCG_CUDA(cudaMemcpyAsync(out, tr.p, tr.bytes, cudaMemcpyDeviceToHost, s));
    MSCG_CUDA(cudaStreamSynchronize(s));
  });
  return rc == MSCG_OK ? dim0 : -rc;
}

int mscg_bench_apply(mscg_precond* pc, const double* y, double* x, double* w, int steps,
                     int with_spmv, double* total_ms, double* stage_ms, int64_t* launches,
                     mscg_status* st) {
  return guard(st, [&] {
    if (!pc || steps < 1) throw std::invalid_argument("mscg_bench_apply: bad arguments");
    cudaStream_t s = pc->ctx->ctx.stream;
    const int per = 7;
    std::vector<cudaEvent_t> ev(static_cast<size_t>(steps) * per);
    for (auto& e : ev) MSCG_CUDA(cudaEventCreate(&e));
    const int64_t l0 = pc->ctx->ctx.launches;
    for (int k = 0; k < steps; ++k) {
      cudaEvent_t* e = ev.data() + static_cast<size_t>(k) * per;
      pc->pc->apply(y, x, s, e);
      if (with_spmv) mscg::spmv(*pc->pc->C, x, w, nullptr, 0, s);
      MSCG_CUDA(cudaEventRecord(e[6], s));
    }
    MSCG_CUDA(cudaStreamSynchronize(s));
    if (launches) *launches = pc->ctx->ctx.launches - l0;
    float ms = 0;
    MSCG_CUDA(cudaEventElapsedTime(&ms, ev.front(), ev.back()));
    *total_ms = ms;
    for (int j = 0; j < 6; ++j) stage_ms[j] = 0;
    for (int k = 0; k < steps; ++k) {
      cudaEvent_t* e = ev.data() + static_cast<size_t>(k) * per;
      for (int j = 0; j < 6; ++j) {
        MSCG_CUDA(cudaEventElapsedTime(&ms, e[j], e[j + 1]));
        stage_ms[j] += ms;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

// ---- GMRES -----------------------------------------------------------------

int mscg_gmres(mscg_ctx* ctx, mscg_csr* a, mscg_precond* pc, const double* b, double* x, int mem,
               const mscg_gmres_config* cfg, mscg_gmres_report* rep, double* history,
               int hist_cap, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx || !a) throw std::invalid_argument("gmres: null context or matrix");
    mscg::GmresConfig c;
    if (cfg) {
      c.restart = cfg->restart;
      c.max_iters = cfg->max_iters;
      c.rel_tol = cfg->rel_tol;
      c.left = cfg->side == 1;
      c.orth = cfg->orth;
      if (c.orth < 0 || c.orth > 2) throw std::invalid_argument("gmres: orth must be 0 (MGS), 1 (CGS2) or 2 (DCGS2)");
    }
    if (!a || !a->a) throw std::invalid_argument("gmres: null matrix");
    const size_t n = a->a->nrows;
    if (a->a->ncols != static_cast<int>(n)) throw std::invalid_argument("gmres: dimension mismatch");
    mscg::GmresResult r;
    auto run = [&](const double* db, double* dx) {
      r = mscg::gmres(&ctx->ctx, *a->a, pc ? pc->pc.get() : nullptr, db, dx, c);
    };
    with_vectors(ctx, b, n, x, n, mem, run);
    if (rep) {
      rep->iterations = r.iterations;
      rep->converged = r.converged ? 1 : 0;
      rep->history_total = static_cast<int>(r.history.size());
      rep->history_len = std::min<int>(hist_cap, rep->history_total);
      rep->solve_seconds = r.seconds;
      rep->final_true_residual = r.final_true;
    }
    if (history)
      for (int i = 0; i < std::min<int>(hist_cap, static_cast<int>(r.history.size())); ++i)
        history[i] = r.history[i];
  });
}

int mscg_gmres_shard(mscg_ctx* ctx, mscg_precond* shard, int rank, int world, const double* b,
                     double* x, int mem, const mscg_gmres_config* cfg, double* comm_buf,
                     int comm_cap, mscg_allreduce_fn allreduce, void* user,
                     mscg_gmres_report* rep, double* history, int hist_cap, mscg_status* st) {
  return guard(st, [&] {
    if (!ctx || !shard || !shard->pc->shard.on)
      throw std::invalid_argument("gmres_shard: null context or not a shard preconditioner");
    if (world > 1 && (!allreduce || !comm_buf))
      throw std::invalid_argument("gmres_shard: an all-reduce callback and buffer are needed");
    if (rank < 0 || rank >= std::max(world, 1)) throw std::invalid_argument("gmres_shard: bad rank");
    mscg::GmresConfig c;
    if (cfg) {
      c.restart = cfg->restart;
      c.max_iters = cfg->max_iters;
      c.rel_tol = cfg->rel_tol;
      c.left = cfg->side == 1;
      c.orth = cfg->orth;
    }
    mscg::DistComm comm;
    comm.rank = rank;
    comm.size = std::max(world, 1);
    comm.buf = comm_buf;
    comm.cap = comm_cap;
    comm.allreduce = allreduce;
    comm.user = user;
    const size_t n = shard->pc->n;
    mscg::GmresResult r;
    with_vectors(ctx, b, n, x, n, mem, [&](const double* db, double* dx) {
      r = mscg::gmres_shard(&ctx->ctx, shard->pc.get(), db, dx, c, comm);
    });
    if (rep) {
      rep->iterations = r.iterations;
      rep->converged = r.converged ? 1 : 0;
      rep->history_total = static_cast<int>(r.history.size());
      rep->history_len = std::min<int>(hist_cap, rep->history_total);
      rep->solve_seconds = r.seconds;
      rep->final_true_residual = r.final_true;
    }
    if (history)
      for (int i = 0; i < std::min<int>(hist_cap, static_cast<int>(r.history.size())); ++i)
        history[i] = r.history[i];
  });
}

int mscg_true_residual(mscg_ctx* ctx, mscg_csr* a, const double* x, const double* b, int mem,
                       double* out, mscg_status* st) {
  return guard(st, [&] {
    if (!a || !a->a) throw std::invalid_argument("true_residual: null matrix");
    const size_t n = a->a->nrows;
    if (mem == MSCG_MEM_DEVICE) {
      *out = mscg::true_residual(&ctx->ctx, *a->a, x, b);
      return;
    }
    mscg::DevBuf dx(sizeof(double) * std::max<size_t>(1, a->a->ncols)),
        db(sizeof(double) * std::max<size_t>(1, n));
    // on the context stream (a non-blocking stream: a legacy-stream
    // cudaMemcpy from pageable memory may still be in flight when the
    // residual kernels start)
    cudaStream_t s = ctx->ctx.stream;
    MSCG_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * a->a->ncols, cudaMemcpyHostToDevice, s));
    MSCG_CUDA(cudaMemcpyAsync(db.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    *out = mscg::true_residual(&ctx->ctx, *a->a, dx.as<double>(), db.as<double>());
  });
}

// ---- Matrix Market I/O ------------------------------------------------------

int mscg_mm_read(const char* path, int* nrows, int* ncols, int64_t* nnz, int* rp, int* ci,
                 double* v, mscg_status* st) {
  return guard(st, [&] {
    if (!path || !nrows || !ncols || !nnz) throw std::invalid_argument("mm_read: null argument");
    const mscg::host::Csr a = mscg::host::load_matrix_market(path);
    *nrows = a.nrows;
    *ncols = a.ncols;
    *nnz = a.nnz();
    if (!rp) return;
    if (!ci || !v) throw std::invalid_argument("mm_read: null output array");
    std::memcpy(rp, a.rp.data(), sizeof(int) * a.rp.size());
    if (a.nnz()) {
      std::memcpy(ci, a.ci.data(), sizeof(int) * a.ci.size());
      std::memcpy(v, a.v.data(), sizeof(double) * a.v.size());
    }
  });
}

int mscg_mm_write(const char* path, int nrows, int ncols, const int* rp, const int* ci,
                  const double* v, mscg_status* st) {
  return guard(st, [&] {
    if (!path || nrows < 0 || ncols < 0 || !rp)
      throw std::invalid_argument("mm_write: bad matrix");
    mscg::host::Csr a(nrows, ncols);
    a.rp.assign(rp, rp + nrows + 1);
    a.ci.assign(ci, ci + rp[nrows]);
    a.v.assign(v, v + rp[nrows]);
    mscg::host::write_matrix_market(path, a);
  });
}

int mscg_mm_read_vector(const char* path, int* n, double* v, mscg_status* st) {
  return guard(st, [&] {
    if (!path || !n) throw std::invalid_argument("mm_read_vector: null argument");
    const std::vector<double> x = mscg::host::load_vector_market(path);
    *n = static_cast<int>(x.size());
    if (v && !x.empty()) std::memcpy(v, x.data(), sizeof(double) * x.size());
  });
}

int mscg_mm_write_vector(const char* path, int n, const double* v, mscg_status* st) {
  return guard(st, [&] {
    if (!path || n < 0 || (n && !v)) throw std::invalid_argument("mm_write_vector: bad vector");
    mscg::host::write_vector_market(path, v, n);
  });
}

}  // extern "C"
