// MSC preconditioner on the device: build (build_preconditioner,
// proj/src/preconditioner.cpp:26-83) and apply (MscPreconditioner::apply,
// proj/src/preconditioner.cpp:85-114, the paper's Alg. 2):
//
//   z1 = D^-1 y1                 block_trisolve over the interior blocks
//   t  = y2 - F z1               SELL SpMV with fused subtraction
//   z2 = S^-1 t  (-> x2)         block_trisolve over the Schur blocks (row_perm)
//   w  = E z2                    SELL SpMV
//   x1 = z1 - D^-1 w             block_trisolve with fused subtraction
//
// Five stream-ordered launches, no host synchronisation.  With the explicit
// correction (correct.cu, built when it saves bytes) the last two become
// one: x1 = z1 - W z2, W = D^-1 E precomputed per block.
#include <algorithm>
#include <chrono>

#include "common.cuh"
#include "internal.hpp"

namespace mscg {

namespace {

// Extract the rectangular block A[rb:re, cb:ce) of a host CSR (re-indexed).
void extract(const int* rp, const int* ci, const double* v, int rb, int re, int cb, int ce,
             std::vector<int>& orp, std::vector<int>& oci, std::vector<double>& ov) {
  orp.assign(re - rb + 1, 0);
  oci.clear();
  ov.clear();
  for (int i = rb; i < re; ++i) {
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] >= cb && ci[k] < ce) {
        oci.push_back(ci[k] - cb);
        ov.push_back(v[k]);
      }
    orp[i - rb + 1] = static_cast<int>(oci.size());
  }
}

struct DevArrays {
  DevBuf rp, ci, v;
  DevArrays(Ctx* ctx, int nrows, const int* hrp, const int* hci, const double* hv) {
    const int64_t nnz = hrp[nrows];
    rp = DevBuf(sizeof(int) * (nrows + 1));
    ci = DevBuf(sizeof(int) * std::max<int64_t>(1, nnz));
    v = DevBuf(sizeof(double) * std::max<int64_t>(1, nnz));
    MSCG_CUDA(cudaMemcpyAsync(rp.p, hrp, sizeof(int) * (nrows + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (nnz) {
      MSCG_CUDA(cudaMemcpyAsync(ci.p, hci, sizeof(int) * nnz, cudaMemcpyHostToDevice, ctx->stream));
      MSCG_CUDA(cudaMemcpyAsync(v.p, hv, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream));
    }
  }
};

}  // namespace

std::unique_ptr<Precond> build_precond(Ctx* ctx, int n, int p, const int* c_rp,
                                       const int* c_ci, const double* c_v,
                                       const std::vector<std::pair<int, int>>& d_ranges,
                                       const int* s_rp, const int* s_ci,
                                       const double* s_v,
                                       const std::vector<std::pair<int, int>>& s_ranges_in,
                                       double tol_a, int s_a, int block_begin,
                                       int block_end, bool schur_single) {
  if (p < 0 || p > n) throw Error(1, "build_preconditioner: split out of range");
  if (d_ranges.empty()) throw Error(1, "build_preconditioner: no interior D blocks");
  const int ng = n - p;
  const std::vector<std::pair<int, int>> s_ranges =
      schur_single ? std::vector<std::pair<int, int>>{{0, ng}} : s_ranges_in;
  if (schur_single && ng < 1)
    throw Error(1, "build_preconditioner: Schur approximation does not match the split");
  {
    int cov = 0;
    for (auto [b, e] : d_ranges) {
      if (b != cov || e <= b || e > p)
        throw Error(1, "build_preconditioner: interior block ranges must tile [0, p)");
      cov = e;
    }
    if (cov != p) throw Error(1, "build_preconditioner: interior block ranges must tile [0, p)");
    cov = 0;
    for (auto [b, e] : s_ranges) {
      if (b != cov || e <= b || e > ng)
        throw Error(1, "build_preconditioner: Schur ranges must tile [0, n_g)");
      cov = e;
    }
    if (cov != ng)
      throw Error(1, "build_preconditioner: Schur approximation does not match the split");
  }
  const int nb = static_cast<int>(d_ranges.size());
  const bool sharded = !(block_begin == 0 && (block_end < 0 || block_end == nb));
  if (block_end < 0) block_end = nb;
  if (block_begin < 0 || block_begin >= block_end || block_end > nb)
    throw Error(1, "build_preconditioner: shard block range out of range");
  auto pc = std::make_unique<Precond>();
  pc->ctx = ctx;
  pc->n = n;
  pc->p = p;
  const int lo = d_ranges[block_begin].first, hi = d_ranges[block_end - 1].second;
  std::vector<int> e_rp, e_ci;  // host E (rows of this set), kept for the correction
  std::vector<double> e_v;
  {
    std::vector<int> rp, ci;
    std::vector<double> v;
    if (!sharded) {
      // interior rows reading another interior block's columns (a coupled
      // user split): host-buffer matvecs must not overlap per chunk
      for (auto [b, e] : d_ranges) {
        for (int i = b; i < e && !pc->d_coupled; ++i)
          for (int k = c_rp[i]; k < c_rp[i + 1]; ++k)
            if (c_ci[k] < p && (c_ci[k] < b || c_ci[k] >= e)) {
              pc->d_coupled = true;
              break;
            }
        if (pc->d_coupled) break;
      }
      pc->C = upload_csr(ctx, n, n, c_rp, c_ci, c_v);
      extract(c_rp, c_ci, c_v, 0, p, p, n, e_rp, e_ci, e_v);  // E = C[0:p, p:n]
      pc->E = upload_csr(ctx, p, ng, e_rp.data(), e_ci.data(), e_v.data());
      extract(c_rp, c_ci, c_v, p, n, 0, p, rp, ci, v);  // F = C[p:n, 0:p]
      pc->F = upload_csr(ctx, ng, p, rp.data(), ci.data(), v.data());
    } else {
      pc->shard.on = true;
      pc->shard.b0 = block_begin;
      pc->shard.b1 = block_end;
      pc->shard.row_lo = lo;
      pc->shard.row_hi = hi;
      extract(c_rp, c_ci, c_v, lo, hi, 0, n, rp, ci, v);  // C[lo:hi, :]
      pc->shard.Cr = upload_csr(ctx, hi - lo, n, rp.data(), ci.data(), v.data());
      extract(c_rp, c_ci, c_v, p, n, p, n, rp, ci, v);  // G = C[p:n, p:n]
      pc->shard.G = upload_csr(ctx, ng, ng, rp.data(), ci.data(), v.data());
      extract(c_rp, c_ci, c_v, lo, hi, p, n, e_rp, e_ci, e_v);  // E_r = C[lo:hi, p:n]
      pc->E = upload_csr(ctx, hi - lo, ng, e_rp.data(), e_ci.data(), e_v.data());
      extract(c_rp, c_ci, c_v, p, n, lo, hi, rp, ci, v);  // F_r = C[p:n, lo:hi]
      pc->F = upload_csr(ctx, ng, hi - lo, rp.data(), ci.data(), v.data());
    }
  }
  // Interior blocks: ILUT(tolA) or exact LU when dim <= sA (:44-56).
  {
    DevArrays c(ctx, n, c_rp, c_ci, c_v);
    std::vector<BlockSpec> blocks;
    std::vector<char> exact;
    for (int k = block_begin; k < block_end; ++k) {
      const auto [b, e] = d_ranges[k];
      blocks.push_back({b, e - b, b});
      exact.push_back((e - b) <= s_a ? 1 : 0);
    }
    pc->D = factor_blocks(ctx, c.rp.as<int>(), c.ci.as<int>(), c.v.as<double>(), blocks, exact,
                          tol_a, "build_preconditioner: (1,1) block", &pc->times);
  }
  // Schur blocks: exact LU per owned range (:68-81).
  if (ng > 0) {
    DevArrays sm(ctx, ng, s_rp, s_ci, s_v);
    std::vector<BlockSpec> blocks;
    std::vector<char> exact;
    for (auto [b, e] : s_ranges) {
      blocks.push_back({b, e - b, b});
      exact.push_back(1);
    }
    if (!schur_single) {
      pc->S = factor_blocks(ctx, sm.rp.as<int>(), sm.ci.as<int>(), sm.v.as<double>(), blocks,
                            exact, 0.0, "build_preconditioner: Schur block", &pc->times);
    } else {
      // the overlapped band: one exact LU of the whole S^ (:58-67)
      try {
        pc->S = factor_blocks(ctx, sm.rp.as<int>(), sm.ci.as<int>(), sm.v.as<double>(), blocks,
                              exact, 0.0, "", &pc->times);
      } catch (const Error& e) {
        if (e.code != 2) throw;
        throw Error(2, std::string("build_preconditioner: overlapped Schur band: ") + e.what(),
                    -1, e.pivot);
      }
    }
  }
  pc->stored_nnz = pc->E->nnz + pc->F->nnz + pc->D->nnz_l() + pc->D->nnz_u() + (hi - lo);
  if (pc->S) pc->stored_nnz += pc->S->nnz_l() + pc->S->nnz_u() + ng;
  pc->z1 = DevBuf(sizeof(double) * std::max(1, p));
  pc->t = DevBuf(sizeof(double) * std::max(1, ng));
  pc->w = DevBuf(sizeof(double) * std::max(1, p));
  if (pc->S && ng > 0) {
    const int mode = ctx->correction >= 0 ? ctx->correction : correction_mode_default();
    pc->corr = build_correction(ctx, *pc->D, e_rp.data(), e_ci.data(), e_v.data(), mode,
                                pc->z1.as<double>(), pc->w.as<double>());
    if (pc->corr) pc->times.corr_s = pc->corr->build_s;
  }
  return pc;
}

namespace {
__global__ void sub_kernel(int n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __dsub_rn(a[i], b[i]);
}
}  // namespace

void Precond::apply_shard_begin(const double* y, double* tpart, cudaStream_t s) {
  if (!shard.on) throw Error(1, "apply_shard_begin: not a shard");
  // FactorSet rows are numbered from the set's first row: offset the vectors
  const int lo = shard.row_lo;
  double* z1 = this->z1.as<double>();
  block_trisolve(*D, y + lo, z1 + lo, nullptr, s);
  ctx->launches++;
  const int ng = n - p;
  if (ng > 0) spmv(*F, z1 + lo, tpart, nullptr, 0, s);
}

void Precond::apply_shard_end(const double* y, const double* tsum, double* x, cudaStream_t s) {
  if (!shard.on) throw Error(1, "apply_shard_end: not a shard");
  double* z1 = this->z1.as<double>();
  double* w = this->w.as<double>();
  const int ng = n - p;
  if (S && ng > 0) {
    double* t = this->t.as<double>();
    sub_kernel<<<(ng + 255) / 256, 256, 0, s>>>(ng, y + p, tsum, t);
    MSCG_CUDA(cudaGetLastError());
    ctx->launches++;
    block_trisolve(*S, t, x + p, nullptr, s);
    ctx->launches++;
    const int lo = shard.row_lo;
    if (corr) {
      apply_correction(*corr, x + p, z1 + lo, x + lo, -1, s);
    } else {
      spmv(*E, x + p, w + lo, nullptr, 0, s);
      block_trisolve(*D, w + lo, x + lo, z1 + lo, s);
    }
    ctx->launches++;
  } else {
    MSCG_CUDA(cudaMemcpyAsync(x + shard.row_lo, z1 + shard.row_lo,
                              sizeof(double) * (shard.row_hi - shard.row_lo),
                              cudaMemcpyDeviceToDevice, s));
  }
}

void Precond::spmv_shard(const double* x, double* y, double* y2part, bool with_g,
                         cudaStream_t s) {
  if (!shard.on) throw Error(1, "spmv_shard: not a shard");
  spmv(*shard.Cr, x, y + shard.row_lo, nullptr, 0, s);
  if (n - p > 0) {
    spmv(*F, x + shard.row_lo, y2part, nullptr, 0, s);
    if (with_g) spmv(*shard.G, x + p, y2part, y2part, 2, s);
  }
}

Precond::~Precond() {
  for (int c = 0; c < kSolveChunks; ++c) {
    if (side[c]) cudaStreamDestroy(side[c]);
    if (ev_in[c]) cudaEventDestroy(ev_in[c]);
    if (ev_out[c]) cudaEventDestroy(ev_out[c]);
  }
  if (ev_mid) cudaEventDestroy(ev_mid);
}

Precond::Scratch& Precond::scratch_for(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(scratch_mu);
  for (auto& e : scratch)
    if (e.first == s) return *e.second;
  auto sc = std::make_unique<Scratch>();
  sc->z1 = DevBuf(sizeof(double) * std::max(1, p));
  sc->t = DevBuf(sizeof(double) * std::max(1, n - p));
  sc->w = DevBuf(sizeof(double) * std::max(1, p));
  scratch.emplace_back(s, std::move(sc));
  return *scratch.back().second;
}

void Precond::ensure_side_streams() {
  if (side[0]) return;
  for (int c = 0; c < kSolveChunks; ++c) {
    MSCG_CUDA(cudaStreamCreateWithFlags(&side[c], cudaStreamNonBlocking));
    MSCG_CUDA(cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming));
    MSCG_CUDA(cudaEventCreateWithFlags(&ev_out[c], cudaEventDisableTiming));
  }
  MSCG_CUDA(cudaEventCreateWithFlags(&ev_mid, cudaEventDisableTiming));
}

// Interior rows [lo, hi) of block chunk c (the interface starts at p).
void Precond::chunk_rows(int c, int& lo, int& hi) const {
  const int b0 = D->h_chunk[c], b1 = D->h_chunk[c + 1];
  lo = b0 < D->nblocks ? D->h_row0[b0] : p;
  hi = b1 < D->nblocks ? D->h_row0[b1] : p;
}

void Precond::spmv_host(const double* x_h, double* y_h, double* d_x, double* d_y,
                        cudaStream_t s) {
  if (shard.on || !C) throw Error(1, "matvec: this preconditioner holds no full C");
  if (d_coupled) {
    MSCG_CUDA(cudaMemcpyAsync(d_x, x_h, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    spmv(*C, d_x, d_y, nullptr, 0, s);
    MSCG_CUDA(cudaMemcpyAsync(y_h, d_y, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    return;
  }
  ensure_side_streams();
  const int ng = n - p;
  cudaEvent_t ev_if = ev_mid;
  MSCG_CUDA(cudaEventRecord(ev_mid, s));  // after earlier work on s (scratch reuse)
  if (ng > 0)
    MSCG_CUDA(cudaMemcpyAsync(d_x + p, x_h + p, sizeof(double) * ng, cudaMemcpyHostToDevice, s));
  MSCG_CUDA(cudaEventRecord(ev_if, s));
  for (int c = 0; c < kSolveChunks; ++c) {
    int lo, hi;
    chunk_rows(c, lo, hi);
    MSCG_CUDA(cudaStreamWaitEvent(side[c], ev_if, 0));
    if (hi > lo)
      MSCG_CUDA(cudaMemcpyAsync(d_x + lo, x_h + lo, sizeof(double) * (hi - lo),
                                cudaMemcpyHostToDevice, side[c]));
    MSCG_CUDA(cudaEventRecord(ev_in[c], side[c]));
    spmv_rows(*C, d_x, d_y, nullptr, 0, lo, hi, side[c]);
    if (hi > lo)
      MSCG_CUDA(cudaMemcpyAsync(y_h + lo, d_y + lo, sizeof(double) * (hi - lo),
                                cudaMemcpyDeviceToHost, side[c]));
    MSCG_CUDA(cudaEventRecord(ev_out[c], side[c]));
  }
  // interface rows read every column: after all of x has arrived
  for (int c = 0; c < kSolveChunks; ++c) MSCG_CUDA(cudaStreamWaitEvent(s, ev_in[c], 0));
  spmv_rows(*C, d_x, d_y, nullptr, 0, p, n, s);
  if (ng > 0)
    MSCG_CUDA(cudaMemcpyAsync(y_h + p, d_y + p, sizeof(double) * ng, cudaMemcpyDeviceToHost, s));
  for (int c = 0; c < kSolveChunks; ++c) MSCG_CUDA(cudaStreamWaitEvent(s, ev_out[c], 0));
}

void Precond::apply_host(const double* y_h, double* x_h, double* d_y, double* d_x,
                         cudaStream_t s) {
  if (shard.on) throw Error(1, "MscPreconditioner::apply: this is a shard (use apply_shard_*)");
  ensure_side_streams();
  // keyed by this preconditioner's private side stream: host-buffer applies
  // are serialised by the context lock, and a device-buffer apply on s from
  // another thread must not share these vectors
  Scratch& sc = scratch_for(side[0]);
  double* z1 = sc.z1.as<double>();
  double* t = sc.t.as<double>();
  double* w = sc.w.as<double>();
  const int ng = n - p;
  const bool corr_on = corr && use_corr;
  auto rows = [&](int c, int& lo, int& hi) { chunk_rows(c, lo, hi); };
  // order the side streams after earlier work on s (scratch reuse)
  MSCG_CUDA(cudaEventRecord(ev_mid, s));
  // 1. per chunk: y rows in, z1 = D^-1 y1 on those blocks
  for (int c = 0; c < kSolveChunks; ++c) {
    int lo, hi;
    rows(c, lo, hi);
    MSCG_CUDA(cudaStreamWaitEvent(side[c], ev_mid, 0));
    if (hi > lo)
      MSCG_CUDA(cudaMemcpyAsync(d_y + lo, y_h + lo, sizeof(double) * (hi - lo),
                                cudaMemcpyHostToDevice, side[c]));
    block_trisolve(*D, d_y, z1, nullptr, side[c], nullptr, c);
    ctx->launches++;
    MSCG_CUDA(cudaEventRecord(ev_in[c], side[c]));
  }
  if (ng > 0)
    MSCG_CUDA(cudaMemcpyAsync(d_y + p, y_h + p, sizeof(double) * ng, cudaMemcpyHostToDevice, s));
  for (int c = 0; c < kSolveChunks; ++c) MSCG_CUDA(cudaStreamWaitEvent(s, ev_in[c], 0));
  // 2. interface (whole vector, on s)
  if (S) {
    spmv(*F, z1, t, d_y + p, 1, s);
    block_trisolve(*S, t, d_x + p, nullptr, s);
    ctx->launches++;
    MSCG_CUDA(cudaMemcpyAsync(x_h + p, d_x + p, sizeof(double) * ng, cudaMemcpyDeviceToHost, s));
    if (!corr_on) spmv(*E, d_x + p, w, nullptr, 0, s);
  }
  MSCG_CUDA(cudaEventRecord(ev_mid, s));
  // 3. per chunk: x1 = z1 - D^-1 w on those blocks, rows out
  for (int c = 0; c < kSolveChunks; ++c) {
    int lo, hi;
    rows(c, lo, hi);
    MSCG_CUDA(cudaStreamWaitEvent(side[c], ev_mid, 0));
    if (S) {
      if (corr_on)
        apply_correction(*corr, d_x + p, z1, d_x, c, side[c]);
      else
        block_trisolve(*D, w, d_x, z1, side[c], nullptr, c);
      ctx->launches++;
    } else if (hi > lo) {
      MSCG_CUDA(cudaMemcpyAsync(d_x + lo, z1 + lo, sizeof(double) * (hi - lo),
                                cudaMemcpyDeviceToDevice, side[c]));
    }
    if (hi > lo)
      MSCG_CUDA(cudaMemcpyAsync(x_h + lo, d_x + lo, sizeof(double) * (hi - lo),
                                cudaMemcpyDeviceToHost, side[c]));
    MSCG_CUDA(cudaEventRecord(ev_out[c], side[c]));
  }
  for (int c = 0; c < kSolveChunks; ++c) MSCG_CUDA(cudaStreamWaitEvent(s, ev_out[c], 0));
}

void Precond::apply(const double* y, double* x, cudaStream_t s, cudaEvent_t* ev) {
  if (shard.on) throw Error(1, "MscPreconditioner::apply: this is a shard (use apply_shard_*)");
  // ev (optional): 6 events bracketing the 5 stages (ev[0] before stage 0,
  // ev[k+1] after stage k) for the bench's per-kernel timing.
  Scratch& sc = scratch_for(s);
  double* z1 = sc.z1.as<double>();
  double* t = sc.t.as<double>();
  double* w = sc.w.as<double>();
  auto mark = [&](int k) {
    if (ev) MSCG_CUDA(cudaEventRecord(ev[k], s));
  };
  mark(0);
  block_trisolve(*D, y, z1, nullptr, s);
  ctx->launches++;
  mark(1);
  if (S) {
    spmv(*F, z1, t, y + p, 1, s);
    mark(2);
    block_trisolve(*S, t, x + p, nullptr, s);
    ctx->launches++;
    mark(3);
    if (corr && use_corr) {
      // x1 = z1 - (D^-1 E) z2 with the precomputed panels (correct.cu)
      mark(4);
      apply_correction(*corr, x + p, z1, x, -1, s);
    } else {
      spmv(*E, x + p, w, nullptr, 0, s);
      mark(4);
      block_trisolve(*D, w, x, z1, s);
    }
    ctx->launches++;
    mark(5);
  } else {
    MSCG_CUDA(cudaMemcpyAsync(x, z1, sizeof(double) * p, cudaMemcpyDeviceToDevice, s));
    for (int k = 2; k <= 5; ++k) mark(k);
  }
}

}  // namespace mscg
