"""GPU parity: the CUDA path (through the C ABI) against the oracle
restatement (oracle/restate.c, pinned to the compiled reference).

Bars (BASELINE.json north_star):
  * SpMV, ILUT factors, Schur LU factors: bit-identical (integer/byte work and
    order-preserving fp64 replay);
  * preconditioner apply: relative 2-norm error <= 1e-10 (fp64);
  * GMRES: iteration count within +-1 of the oracle, both true residuals
    below the requested tolerance.
"""
import json
import os

import numpy as np
import pytest

from helpers import csr_tuple, oracle_msc, rel_err, same_bits, split_blocks

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-10
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def cfg1(msc):
    pb = msc.oseen_problem(32, 0.1, 8)
    pb.build_msc("lum")
    return pb


@pytest.fixture(scope="module")
def cfg1_pc(msc, ctx, cfg1):
    return msc.build_preconditioner(cfg1, tolA=1e-4, sA=0, ctx=ctx)


@pytest.fixture(scope="module")
def cfg1_oracle(rs, cfg1):
    return oracle_msc(rs, cfg1, 1e-4, 0)


def test_spmv_bit_identical(msc, ctx, rs, cfg1, ref):
    C = cfg1.C
    A = msc.DeviceMatrix(ctx, C)
    for seed in (0, 1, 2):
        x = ref.random_vector(C.ncols, seed)
        y = msc.matvec(A, x)
        assert same_bits(y, rs.matvec(*csr_tuple(C), x))


def test_spmv_rectangular_and_empty_rows(msc, ctx, rs):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((70, 45)) * (rng.random((70, 45)) < 0.1)
    a[3, :] = 0.0
    a[40:, :] = 0.0  # trailing empty rows, ragged slices
    A = msc.SparseMatrix.from_dense(a)
    x = rng.standard_normal(45)
    y = msc.matvec(msc.DeviceMatrix(ctx, A), x)
    assert same_bits(y, rs.matvec(*csr_tuple(A), x))


def test_ilut_factors_bit_identical(cfg1_pc, cfg1_oracle, cfg1):
    assert cfg1_pc.nblocks == cfg1.nblocks
    for b in range(cfg1.nblocks):
        f = cfg1_pc.d_factors(b)
        o = cfg1_oracle.dfac[b]
        assert np.array_equal(f.lower.row_offsets, o.lrp)
        assert np.array_equal(f.lower.col_indices, o.lci)
        assert same_bits(f.lower.values, o.lv)
        assert np.array_equal(f.upper.row_offsets, o.urp)
        assert np.array_equal(f.upper.col_indices, o.uci)
        assert same_bits(f.upper.values, o.uv)


def test_schur_factors_bit_identical(cfg1_pc, cfg1_oracle):
    assert cfg1_pc.nschur == len(cfg1_oracle.sfac)
    for b in range(cfg1_pc.nschur):
        f = cfg1_pc.schur_factors(b)
        o = cfg1_oracle.sfac[b]
        assert np.array_equal(f.row_perm, o.perm)
        assert np.array_equal(f.lower.row_offsets, o.lrp)
        assert np.array_equal(f.lower.col_indices, o.lci)
        assert same_bits(f.lower.values, o.lv)
        assert np.array_equal(f.upper.col_indices, o.uci)
        assert same_bits(f.upper.values, o.uv)


def test_stored_nnz_matches_oracle(cfg1_pc, cfg1_oracle, msc, cfg1):
    assert cfg1_pc.stored_nnz() == cfg1_oracle.stored_nnz
    assert msc.fill_factor(cfg1_pc, cfg1.C) == cfg1_oracle.stored_nnz / cfg1.C.nnz


def test_apply_matches_oracle(cfg1_pc, cfg1_oracle, ref, cfg1):
    for seed in (0, 1, 7):
        y = ref.random_vector(cfg1.n, seed)
        got = cfg1_pc.apply(y)
        want = cfg1_oracle.apply(y)
        assert rel_err(got, want) <= APPLY_TOL


def test_apply_zero_and_linearity(cfg1_pc, ref, cfg1):
    z = np.zeros(cfg1.n)
    assert np.array_equal(cfg1_pc.apply(z), z)
    y1 = ref.random_vector(cfg1.n, 11)
    y2 = ref.random_vector(cfg1.n, 12)
    a, b = 0.75, -1.25
    lhs = cfg1_pc.apply(a * y1 + b * y2)
    rhs = a * cfg1_pc.apply(y1) + b * cfg1_pc.apply(y2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(1.0, np.max(np.abs(lhs)))


def test_apply_device_tensor(cfg1_pc, cfg1_oracle, ref, cfg1):
    import torch
    y = ref.random_vector(cfg1.n, 3)
    x = cfg1_pc.apply(torch.from_numpy(y).cuda())
    assert x.is_cuda
    assert rel_err(x.cpu().numpy(), cfg1_oracle.apply(y)) <= APPLY_TOL


@pytest.mark.parametrize("orth", ["dcgs2", "cgs2", "mgs"])
def test_gmres_cfg1_iterations(msc, cfg1_pc, cfg1_oracle, cfg1, ref, rs, orth):
    b = ref.random_vector(cfg1.n, 0)
    want = rs.gmres(csr_tuple(cfg1.C), b, 30, 3000, 1e-8, msc=cfg1_oracle)
    cfg = msc.SolverConfig(restart=30, max_iters=3000, rel_tol=1e-8, orth=orth)
    x, rep = msc.gmres(cfg1_pc.matrix, cfg1_pc, b, cfg)
    assert want["iterations"] == 88  # SURVEY §8(d) target (LUM, seed 0)
    assert abs(rep.iterations - want["iterations"]) <= 1
    assert rep.converged and want["converged"]
    tr = msc.true_residual(cfg1_pc.matrix, x, b)
    assert tr <= 1e-8
    assert rep.residual_history[-1] <= 1e-8
    # the recurrence history tracks the oracle's closely
    h1 = np.asarray(rep.residual_history[:-1])
    h2 = np.asarray(want["history"][:-1])
    k = min(len(h1), len(h2)) - 2
    assert np.allclose(h1[:k], h2[:k], rtol=1e-6, atol=0)


@pytest.mark.parametrize("n,restart", [(4099, 70), (3000, 33), (257, 5)])
def test_gmres_cgs2_fused_matches_four_sweeps(msc, ctx, n, restart, monkeypatch):
    """The fused axpy+dot CGS2 step (three sweeps over the basis) against the
    four-sweep CGS2 (MSCG_CGS2_FUSED=0): odd and even lengths, more than one
    group of 32 basis vectors. Same operator, reductions regrouped: the
    residual histories agree to 1e-9 relative and the iteration counts match."""
    rng = np.random.default_rng(n)
    a = np.zeros((n, n))
    idx = np.arange(n)
    a[idx, idx] = 1.2 + rng.uniform(0, 1, n)  # ~43 iterations (scipy)
    a[idx, (idx + 1) % n] = -0.9
    a[idx, (idx + 7) % n] = rng.uniform(-0.5, 0.5, n)
    A = msc.DeviceMatrix(ctx, msc.SparseMatrix.from_dense(a))
    b = rng.uniform(-1, 1, n)
    cfg = msc.SolverConfig(restart=restart, max_iters=400, rel_tol=1e-10, orth="cgs2")
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("MSCG_CGS2_FUSED", mode)
        out[mode] = msc.gmres(A, None, b, cfg)
    (x0, r0), (x1, r1) = out["0"], out["1"]
    assert r1.converged and r0.converged
    assert r1.iterations == r0.iterations and r1.iterations > 33  # two groups of 32
    h0, h1 = np.asarray(r0.residual_history), np.asarray(r1.residual_history)
    assert np.allclose(h1, h0, rtol=1e-9, atol=1e-15)
    assert rel_err(x1, x0) < 1e-9
    assert np.linalg.norm(b - a @ x1) / np.linalg.norm(b) <= 1e-10


def _banded_system(msc, ctx, n, seed):
    """Sparse nonsymmetric test operator (CSR built directly, any n)."""
    rng = np.random.default_rng(seed)
    idx = np.arange(n)
    rows = np.concatenate([idx, idx, idx])
    cols = np.concatenate([idx, (idx + 1) % n, (idx + 7) % n])
    vals = np.concatenate([1.2 + rng.uniform(0, 1, n), np.full(n, -0.9), rng.uniform(-0.5, 0.5, n)])
    o = np.lexsort((cols, rows))
    rows, cols, vals = rows[o], cols[o], vals[o]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    S = msc.SparseMatrix(n, n, np.cumsum(rp).astype(np.int32), cols.astype(np.int32), vals)
    return S, msc.DeviceMatrix(ctx, S), rng.uniform(-1, 1, n)


@pytest.mark.parametrize("n,restart", [(4099, 70), (3000, 33), (257, 5), (160001, 40)])
def test_gmres_dcgs2_matches_cgs2(msc, ctx, n, restart, monkeypatch):
    """DCGS2 (two basis sweeps, delayed reorthogonalisation) against CGS2
    (three sweeps): same projections, regrouped arithmetic, so the residual
    histories agree to 1e-9 relative and the iteration counts match; odd and
    even lengths, restarts, several groups of basis vectors, and a long
    vector (n = 160001) where the 16-vector dot groups are chosen."""
    S, A, b = _banded_system(msc, ctx, n, n)
    out = {}
    for orth in ("cgs2", "dcgs2"):
        cfg = msc.SolverConfig(restart=restart, max_iters=400, rel_tol=1e-10, orth=orth)
        out[orth] = msc.gmres(A, None, b, cfg)
    (x0, r0), (x1, r1) = out["cgs2"], out["dcgs2"]
    assert r0.converged and r1.converged
    assert r1.iterations == r0.iterations and r1.iterations > restart // 2
    h0, h1 = np.asarray(r0.residual_history), np.asarray(r1.residual_history)
    assert np.allclose(h1, h0, rtol=1e-9, atol=1e-15)
    assert rel_err(x1, x0) < 1e-9
    ax = np.zeros(n)
    rows = np.repeat(np.arange(n), np.diff(S.row_offsets))
    np.add.at(ax, rows, S.values * x1[S.col_indices])
    assert np.linalg.norm(b - ax) / np.linalg.norm(b) <= 1e-10


@pytest.mark.parametrize("n,restart", [(3001, 30), (48896, 50)])
def test_gmres_dcgs2_cooperative_step_matches(msc, ctx, n, restart, monkeypatch):
    """Short vectors run each DCGS2 step as one cooperative kernel
    (MSCG_DCGS2_COOP): the same arithmetic per row, the reductions over a
    different CTA grid — iterations equal, histories to 1e-10."""
    S, A, b = _banded_system(msc, ctx, n, 11)
    cfg = msc.SolverConfig(restart=restart, max_iters=300, rel_tol=1e-10, orth="dcgs2")
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("MSCG_DCGS2_COOP", mode)
        out[mode] = msc.gmres(A, None, b, cfg)
    (x0, r0), (x1, r1) = out["0"], out["1"]
    assert r0.converged and r1.converged and r0.iterations == r1.iterations
    assert np.allclose(r1.residual_history, r0.residual_history, rtol=1e-10, atol=1e-15)
    assert rel_err(x1, x0) < 1e-10


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
def test_gmres_dot_groups_bit_identical(msc, ctx, orth, monkeypatch):
    """Basis dots in groups of 8 or 16 vectors (MSCG_DOT16) keep every
    per-vector summation order: identical residual histories, bit for bit."""
    S, A, b = _banded_system(msc, ctx, 160001, 7)
    cfg = msc.SolverConfig(restart=40, max_iters=120, rel_tol=1e-10, orth=orth)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("MSCG_DOT16", mode)
        out[mode] = msc.gmres(A, None, b, cfg)
    (x0, r0), (x1, r1) = out["0"], out["1"]
    assert r0.iterations == r1.iterations
    assert same_bits(np.asarray(r0.residual_history), np.asarray(r1.residual_history))
    assert same_bits(x0, x1)


def test_gmres_unpreconditioned_identity(msc, ctx, ref):
    n = 12
    I = msc.SparseMatrix.from_dense(np.eye(n))
    A = msc.DeviceMatrix(ctx, I)
    b = ref.random_vector(n, 3)
    x, rep = msc.gmres(A, None, b, msc.SolverConfig(rel_tol=1e-9))
    assert rep.converged and rep.iterations == 1
    assert rel_err(x, b) < 1e-12


def test_gmres_zero_rhs(msc, cfg1_pc, cfg1):
    x, rep = msc.gmres(cfg1_pc.matrix, cfg1_pc, np.zeros(cfg1.n), msc.SolverConfig())
    assert rep.converged and np.all(x == 0) and rep.residual_history == [0.0]


def test_gmres_iteration_cap(msc, ctx, ref):
    # test_krylov.cpp:101-116: cap => NC with exactly 4 iterations.
    n = 60
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = 1.0 + 0.01 * i
        a[i, (i + 1) % n] = -0.99
    A = msc.DeviceMatrix(ctx, msc.SparseMatrix.from_dense(a))
    b = np.random.default_rng(19).uniform(-1, 1, n)
    x, rep = msc.gmres(A, None, b, msc.SolverConfig(restart=2, max_iters=4, rel_tol=1e-9))
    assert not rep.converged and rep.iterations == 4


@pytest.mark.parametrize("seed,variant", [(37, "mscn"), (23, "lum"), (47, "mscnr")])
def test_random_saddle_exact_blocks(msc, ctx, ref, rs, seed, variant):
    """Random saddles (tests/oracles.hpp:122-142) with sA = inf: exact LU of
    D, Schur blocks from build_msc; apply vs the oracle."""
    R = ref.Problem.random_saddle(20, 8, seed, 0.3)
    Cr = R.csr(0)
    C = msc.SparseMatrix(Cr.nrows, Cr.ncols, Cr.rp, Cr.ci, Cr.v)
    pb = msc.partitioned_problem(C, R.p)
    pb.build_msc(variant, mode="explicit", sizes=[4, 4])
    pc = msc.build_preconditioner(pb, tolA=0.0, sA=1 << 30, ctx=ctx)
    M = oracle_msc(rs, pb, 0.0, 1 << 30)
    for s in range(3):
        y = ref.random_vector(R.n, 100 + s)
        assert rel_err(pc.apply(y), M.apply(y)) <= APPLY_TOL
    # reference preconditioner on the same system agrees too
    R.build_schur(variant, 0, 2, sizes=[4, 4])
    R.build_precond(0.0, 1 << 30)
    y = ref.random_vector(R.n, 9)
    assert rel_err(pc.apply(y), R.apply(y)) <= APPLY_TOL


def test_ilut_policy_switch(msc, ctx, rs, ref):
    """sA decides exact vs ILUT per interior block (preconditioner.cpp:44-56)."""
    pb = msc.oseen_problem(16, 0.1, 4)
    pb.build_msc("lum")
    dims = np.diff(pb.d_ranges(), axis=1).ravel()
    sA = int(np.sort(dims)[1])  # some blocks exact, some ILUT
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=sA, ctx=ctx)
    M = oracle_msc(rs, pb, 1e-4, sA)
    for b, d in enumerate(dims):
        f = pc.d_factors(b)
        assert f.kind == ("exact" if d <= sA else "incomplete")
        o = M.dfac[b]
        assert same_bits(f.upper.values, o.uv) and np.array_equal(f.row_perm, o.perm)
    y = ref.random_vector(pb.n, 4)
    assert rel_err(pc.apply(y), M.apply(y)) <= APPLY_TOL


def test_cfg3_zero_pivot_error(msc, ctx):
    """BASELINE cfg3 as written (stretch 1.1): the reference's ILUT raises
    SingularMatrixError in interior block 0 (tests/golden/cfg3_error.json,
    produced by the compiled reference); the GPU ILUT must raise the
    identical error (same block, same local pivot row, same message)."""
    want = json.load(open(os.path.join(GOLDEN, "cfg3_error.json")))
    pb = msc.oseen_problem(256, 0.002, 64, stretched=True, stretch=1.1)
    pb.build_msc("lum", sz=795)
    with pytest.raises(msc.SingularMatrixError) as e:
        msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    assert e.value.pivot_index == want["pivot_index"]
    assert e.value.block == 0
    assert str(e.value) == want["error"]


def test_cfg2_ilut_and_apply(msc, ctx, rs, ref):
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    M = oracle_msc(rs, pb, 1e-4, 0)
    for b in range(pb.nblocks):
        f = pc.d_factors(b)
        o = M.dfac[b]
        assert np.array_equal(f.lower.row_offsets, o.lrp)
        assert np.array_equal(f.upper.col_indices, o.uci)
        assert same_bits(f.lower.values, o.lv) and same_bits(f.upper.values, o.uv)
    # SURVEY §6 (measured on the reference): nnz(L+U) of D at cfg2
    assert sum(pc.d_factors(b).nnz() for b in range(pb.nblocks)) == 21083149
    y = ref.random_vector(pb.n, 0)
    assert rel_err(pc.apply(y), M.apply(y)) <= APPLY_TOL


@pytest.mark.parametrize("env", [
    {"MSCG_PACK_SLACK_U": "0"},                                # items by readiness alone
    {"MSCG_PACK_SLACK_U": "3", "MSCG_PACK_SLACK_L": "5"},      # deadline-aware, both passes
    {"MSCG_PACK_PIECES_L": "4", "MSCG_PACK_PIECES_U": "4"},    # long rows cut by readiness
    {"MSCG_PACK_PIECES_L": "3", "MSCG_PACK_SLACK_U": "16"},
])
def test_work_item_policies_same_operator(msc, ctx, rs, ref, env, monkeypatch):
    """The pack's work-item policy (how long far rows are cut, in which order
    the workers take the items: factor.cu pack_tiled_kernel) only schedules
    the interior solve: the stored factors stay the reference's bit for bit
    and the apply stays within the bar (sums regrouped, nothing else)."""
    pb = msc.oseen_problem(128, 0.01, 16)  # cfg2: ~3000-row blocks, long pressure rows
    pb.build_msc("lum")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    M = oracle_msc(rs, pb, 1e-4, 0)
    for b in (0, pb.nblocks - 1):
        f, o = pc.d_factors(b), M.dfac[b]
        assert np.array_equal(f.lower.row_offsets, o.lrp)
        assert np.array_equal(f.lower.col_indices, o.lci)
        assert same_bits(f.lower.values, o.lv) and same_bits(f.upper.values, o.uv)
    for seed in (0, 1):
        y = ref.random_vector(pb.n, seed)
        assert rel_err(pc.apply(y), M.apply(y)) <= APPLY_TOL
    # deterministic: the same launch twice gives the same bits
    y = ref.random_vector(pb.n, 2)
    assert same_bits(pc.apply(y), pc.apply(y))


@pytest.mark.parametrize("nshards", [2, 3])
def test_sharded_apply_and_spmv_match_full(msc, ctx, ref, nshards):
    """the interior blocks split over ranks, one n_g all-reduce
    per apply.  Ranks are simulated in one process (one GPU); the all-reduce
    is the sum of the per-shard partials.  The sharded apply must equal the
    single-GPU apply to the apply bar, the sharded SpMV to rounding of the
    split interface sums."""
    import torch
    from paper_1104_3349_b200 import dist
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    full = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    dr = pb.d_ranges()
    ranges = dist.shard_blocks(dr[:, 1] - dr[:, 0], nshards)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    try:
        shards = [msc.build_preconditioner_shard(pb, b0, b1, tolA=1e-4, sA=0, ctx=ctx)
                  for b0, b1 in ranges]
        assert sum(s.rows[1] - s.rows[0] for s in shards) == pb.p
        n, p = pb.n, pb.p
        y_h = ref.random_vector(n, 3)
        want = full.apply(y_h)
        y = torch.from_numpy(y_h).cuda()
        ts = [torch.empty(n - p, dtype=torch.float64, device="cuda") for _ in shards]
        xs = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda") for _ in shards]
        for s, t in zip(shards, ts):
            s.apply_begin(y, t)
        tsum = torch.stack(ts).sum(0)  # the all-reduce
        for s, x in zip(shards, xs):
            s.apply_end(y, tsum, x)
        got = np.empty(n)
        for s, x in zip(shards, xs):
            lo, hi = s.rows
            got[lo:hi] = x[lo:hi].cpu().numpy()
            assert np.array_equal(x[p:].cpu().numpy(), xs[0][p:].cpu().numpy())
        got[p:] = xs[0][p:].cpu().numpy()
        assert rel_err(got, want) <= 1e-12
        # sharded SpMV of C against the full one
        A = msc.DeviceMatrix(ctx, pb.C)
        wy = msc.matvec(A, want)
        yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        parts = [torch.empty(n - p, dtype=torch.float64, device="cuda") for _ in shards]
        xd = torch.from_numpy(want).cuda()
        for k, (s, y2) in enumerate(zip(shards, parts)):
            s.spmv(xd, yd, y2, with_interface_block=(k == 0))
        yd[p:] = torch.stack(parts).sum(0)
        assert rel_err(yd.cpu().numpy(), wy) <= 1e-14
        assert np.array_equal(yd[:p].cpu().numpy(), wy[:p])  # interior rows: same row sums
    finally:
        ctx.set_stream(None)


def test_shard_rejects_full_apply(msc, ctx):
    pb = msc.oseen_problem(32, 0.1, 8)
    pb.build_msc("lum")
    s = msc.build_preconditioner_shard(pb, 0, 4, tolA=1e-4, sA=0, ctx=ctx)
    assert s.rows == (0, int(pb.d_ranges()[3, 1]))
    from paper_1104_3349_b200 import _capi
    import ctypes as C
    st = _capi.Status()
    rc = _capi.lib().mscg_precond_apply(s.h, None, None, _capi.MEM_DEVICE, C.byref(st))
    assert rc != 0 and b"shard" in st.message


def test_host_buffer_apply_chunked_matches_device(msc, ctx, ref):
    """Host-buffer applies run chunk by chunk on side streams (copies overlap
    solves); the result must be bit-identical to the device-buffer apply, for
    page-locked and pageable buffers alike."""
    import ctypes as C
    import torch
    from paper_1104_3349_b200 import _capi
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    y = ref.random_vector(pb.n, 11)
    want = pc.apply(torch.from_numpy(y).cuda()).cpu().numpy()
    got_pageable = pc.apply(y)
    assert same_bits(got_pageable, want)
    yp = torch.from_numpy(y).pin_memory()
    xp = torch.full((pb.n,), float("nan"), dtype=torch.float64).pin_memory()
    st = _capi.Status()
    for _ in range(3):  # repeated calls reuse streams and scratch
        rc = _capi.lib().mscg_precond_apply(pc.h, C.c_void_p(yp.data_ptr()),
                                            C.c_void_p(xp.data_ptr()), _capi.MEM_HOST,
                                            C.byref(st))
        assert rc == 0, st.message
        assert same_bits(xp.numpy(), want)


@pytest.mark.gpu
def test_host_buffer_spmv_chunked_matches_device(msc, ctx, ref, rs):
    """matvec(C, x) of a preconditioner's own C with page-locked host
    buffers runs block chunk by block chunk (copies overlapped with the
    rows); it must equal the device-buffer SpMV and the reference bit for
    bit."""
    import ctypes as C
    import torch
    from paper_1104_3349_b200 import _capi
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    x = ref.random_vector(pb.n, 5)
    want = rs.matvec(*pb.C.arrays(), x)
    mat = _capi.lib().mscg_precond_matrix(pc.h)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.full((pb.n,), float("nan"), dtype=torch.float64).pin_memory()
    st = _capi.Status()
    for _ in range(3):
        rc = _capi.lib().mscg_spmv(mat, C.c_void_p(xp.data_ptr()), C.c_void_p(yp.data_ptr()),
                                   _capi.MEM_HOST, C.byref(st))
        assert rc == 0, st.message
        assert same_bits(yp.numpy(), want)
    dev = torch.empty(pb.n, dtype=torch.float64, device="cuda")
    xd = xp.cuda()
    torch.cuda.synchronize()
    rc = _capi.lib().mscg_spmv(mat, C.c_void_p(xd.data_ptr()), C.c_void_p(dev.data_ptr()),
                               _capi.MEM_DEVICE, C.byref(st))
    assert rc == 0, st.message
    ctx.synchronize()
    assert same_bits(dev.cpu().numpy(), want)


@pytest.mark.parametrize("grid,nu,n_a,anchored,sz", [
    (32, 0.1, 8, False, 0),      # cfg1
    (128, 0.01, 16, False, 0),   # cfg2 (aggregates of 158)
    (64, 0.01, 16, False, 0),    # MSCN / MSCNR singular at aggregate 7
    (64, 0.01, 16, True, 40),    # anchored aggregates
])
def test_device_build_msc_matches_reference(msc, ctx, ref, grid, nu, n_a, anchored, sz):
    """build_msc on the device gives the reference's S^
    bit for bit, and the reference's SingularMatrixError for a singular D
    block."""
    R = ref.Problem.oseen(grid, nu, n_a, anchored=anchored)
    P = msc.oseen_problem(grid, nu, n_a, anchored=anchored)
    mode_r, mode_p = (1, "anchored") if anchored else (0, "equal")
    for variant in ("lum", "mscn", "mscnr"):
        err_r = err_p = None
        try:
            R.build_schur(variant, sz, mode_r)
        except ref.RefError as e:
            err_r = str(e)
        try:
            P.build_msc(variant, sz=sz, mode=mode_p, ctx=ctx)
        except (msc.SingularMatrixError, ValueError) as e:
            err_p = str(e)
        assert err_r == err_p, variant
        if err_r:
            continue
        Rs, Ps = R.csr(5), P.s_hat
        assert np.array_equal(Rs.rp, Ps.row_offsets) and np.array_equal(Rs.ci, Ps.col_indices)
        assert same_bits(Rs.v, Ps.values), variant
        assert np.array_equal(R.schur_ranges(), P.schur_ranges())


@pytest.mark.parametrize("grid,nu,n_a,stretched,stretch,anchored", [
    (32, 0.1, 8, False, 1.056, False),     # cfg1
    (128, 0.01, 16, False, 1.056, False),  # cfg2
    (64, 0.002, 16, True, 1.1, False),     # stretched grid
    (96, 0.001, 32, False, 1.056, True),   # anchored interface
])
def test_device_oseen_assembly_matches_reference(msc, ctx, ref, grid, nu, n_a, stretched,
                                                  stretch, anchored):
    """generate_oseen + scale_rows on the device: the
    reference's matrix, permutation and scaled rhs bit for bit."""
    R = ref.Problem.oseen(grid, nu, n_a, stretched=stretched, stretch=stretch, anchored=anchored)
    P = msc.oseen_problem(grid, nu, n_a, stretched=stretched, stretch=stretch,
                          anchored=anchored, ctx=ctx)
    Rc, Pc = R.csr(0), P.C
    assert np.array_equal(Rc.rp, Pc.row_offsets) and np.array_equal(Rc.ci, Pc.col_indices)
    assert same_bits(Rc.v, Pc.values)
    assert np.array_equal(R.perm(), P.perm())
    assert np.array_equal(R.d_ranges(), P.d_ranges())
    assert same_bits(R.scaled_rhs(), P.scaled_rhs())


def test_device_oseen_assembly_cfg5_digest(msc, ctx):
    """At cfg5 size the device-assembled problem equals the host one (whose
    digests are pinned to the reference in tests/golden/cfg5.json)."""
    import json
    js = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg5.json")))
    P = msc.oseen_problem(2048, 0.01, 4096, anchored=True, ctx=ctx)
    from test_host_setup import csr_digest, digest
    assert csr_digest(P.C) == js["c_sha"]
    assert digest(P.perm().astype("<i4")) == js["perm_sha"]


def _interface_columns(pb):
    """k_b: distinct interface columns of E in each interior block's rows."""
    rp, ci, _ = csr_tuple(pb.C)
    p = pb.p
    out = []
    for b, e in pb.d_ranges():
        c = ci[rp[b]:rp[e]]
        out.append((e - b, len(np.unique(c[c >= p]))))
    return out


@pytest.mark.parametrize("grid,nu,n_a,anchored", [(32, 0.1, 8, False), (128, 0.01, 16, False),
                                                  (64, 0.01, 16, True), (256, 0.01, 64, True)])
def test_correction_on_and_off_match_oracle(msc, rs, ref, grid, nu, n_a, anchored):
    """Explicit interior correction (csrc/device/correct.cu): x1 = z1 - W z2
    with W = D^-1 E precomputed per block.  Same operator as the reference's
    w = E z2, x1 = z1 - D^-1 w (preconditioner.cpp:105-111); both modes must
    meet the apply bar against the oracle and agree with each other."""
    import torch
    pb = msc.oseen_problem(grid, nu, n_a, anchored=anchored)
    if anchored:
        pb.build_msc("lum", sz=40, mode="anchored")
    else:
        pb.build_msc("lum")
    M = oracle_msc(rs, pb, 1e-4, 0)
    out = {}
    for mode in ("off", "on"):
        c = msc.Context(0)
        c.set_correction(mode)
        pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=c)
        info = pc.correction()
        assert info["on"] == (mode == "on")
        if info["on"]:
            kb = _interface_columns(pb)
            assert info["entries"] == sum(d * k for d, k in kb)
            assert info["kmax"] == max(k for _, k in kb)
        # the reference's stored_nnz does not count the panels
        assert pc.stored_nnz() == M.stored_nnz
        ys = [ref.random_vector(pb.n, s) for s in (0, 5)]
        xs = [pc.apply(y) for y in ys]
        for y, x in zip(ys, xs):
            assert rel_err(x, M.apply(y)) <= APPLY_TOL
        # host-buffer (chunked) path bit-identical to the device path
        xd = pc.apply(torch.from_numpy(ys[0]).cuda()).cpu().numpy()
        assert same_bits(xs[0], xd)
        # deterministic
        assert same_bits(pc.apply(ys[0]), xs[0])
        out[mode] = xs[0]
        del pc
    assert rel_err(out["on"], out["off"]) <= 1e-12


def test_correction_sharded_matches_full(msc, ref):
    """Shards build their own panels from their rows of E."""
    import torch
    from paper_1104_3349_b200 import dist
    c = msc.Context(0)
    c.set_correction("on")
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    full = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=c)
    assert full.correction()["on"]
    dr = pb.d_ranges()
    ranges = dist.shard_blocks(dr[:, 1] - dr[:, 0], 2)
    c.set_stream(torch.cuda.current_stream().cuda_stream)
    try:
        shards = [msc.build_preconditioner_shard(pb, b0, b1, tolA=1e-4, sA=0, ctx=c)
                  for b0, b1 in ranges]
        n, p = pb.n, pb.p
        y_h = ref.random_vector(n, 4)
        want = full.apply(y_h)
        y = torch.from_numpy(y_h).cuda()
        ts = [torch.empty(n - p, dtype=torch.float64, device="cuda") for _ in shards]
        xs = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda") for _ in shards]
        for s, t in zip(shards, ts):
            s.apply_begin(y, t)
        tsum = torch.stack(ts).sum(0)
        for s, x in zip(shards, xs):
            s.apply_end(y, tsum, x)
        got = np.empty(n)
        for s, x in zip(shards, xs):
            lo, hi = s.rows
            got[lo:hi] = x[lo:hi].cpu().numpy()
        got[p:] = xs[0][p:].cpu().numpy()
        assert rel_err(got, want) <= 1e-12
    finally:
        c.set_stream(None)


@pytest.mark.parametrize("mode", ["off", "on"])
def test_gmres_cfg1_iterations_both_corrections(msc, cfg1, cfg1_oracle, ref, rs, mode):
    c = msc.Context(0)
    c.set_correction(mode)
    pc = msc.build_preconditioner(cfg1, tolA=1e-4, sA=0, ctx=c)
    assert pc.correction()["on"] == (mode == "on")
    b = ref.random_vector(cfg1.n, 0)
    x, rep = msc.gmres(pc.matrix, pc, b, msc.SolverConfig(restart=30, max_iters=3000,
                                                          rel_tol=1e-8))
    assert abs(rep.iterations - 88) <= 1
    assert rep.converged and msc.true_residual(pc.matrix, x, b) <= 1e-8


def test_set_correction_rejects_bad_mode(msc):
    c = msc.Context(0)
    with pytest.raises(KeyError):
        c.set_correction("sometimes")
    import ctypes as C
    from paper_1104_3349_b200 import _capi
    st = _capi.Status()
    assert _capi.lib().mscg_ctx_set_correction(c.h, 7, C.byref(st)) != 0


@pytest.mark.parametrize("grid,nu,n_a,sample", [
    (1024, 0.001, 1024, (0, 511, 1023)),   # BASELINE cfg4
    (2048, 0.01, 4096, (0, 2047, 4095)),   # BASELINE cfg5
])
def test_full_scale_apply_parity(msc, ctx, ref, grid, nu, n_a, sample):
    """BASELINE cfg4 / cfg5 at full size (anchored LUM sz 256).
    The CPU reference cannot build the whole preconditioner in test time
    (cfg4: ~580 s of ILUT), so parity is checked block by block on a sample:
      * the reference's own factor_ilut on the sampled block gives the same
        factors (pattern + bits) as the GPU;
      * x1_b = solve(y1_b) - solve(E_b x2) with the reference's solve, given
        the GPU's interface part x2, equals the GPU's x1_b to the apply bar
        (with and without the explicit correction);
      * both correction modes agree over the whole vector to 1e-12."""
    import torch
    pb = msc.oseen_problem(grid, nu, n_a, anchored=True, ctx=ctx)
    pb.build_msc("lum", sz=256, mode="anchored", ctx=ctx)
    n, p = pb.n, pb.p
    rp, ci, v = csr_tuple(pb.C)
    dr = pb.d_ranges()
    y = ref.random_vector(n, 0)
    xs = {}
    for mode in ("on", "off"):
        c = msc.Context(0)
        c.set_correction(mode)
        pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=c)
        assert pc.correction()["on"] == (mode == "on")
        xs[mode] = pc.apply(torch.from_numpy(y).cuda()).cpu().numpy()
        if mode == "on":
            facs = {int(b): pc.d_factors(int(b)) for b in sample}
        del pc
        torch.cuda.empty_cache()
    assert rel_err(xs["on"], xs["off"]) <= 1e-12
    x2 = xs["on"][p:]
    for b, f in facs.items():
        r0, r1 = dr[b]
        # the block D_b and its interface rows E_b from C
        brp = [0]
        bci, bv, erp, eci, ev = [], [], [0], [], []
        for i in range(r0, r1):
            for k in range(rp[i], rp[i + 1]):
                if r0 <= ci[k] < r1:
                    bci.append(ci[k] - r0)
                    bv.append(v[k])
                elif ci[k] >= p:
                    eci.append(ci[k] - p)
                    ev.append(v[k])
            brp.append(len(bci))
            erp.append(len(eci))
        d = r1 - r0
        Db = ref.Csr(d, d, np.asarray(brp, np.int32), np.asarray(bci, np.int32), np.asarray(bv))
        R = ref.factor_ilut(Db, 1e-4)
        assert np.array_equal(R.L.rp, f.lower.row_offsets) and np.array_equal(R.L.ci, f.lower.col_indices)
        assert np.array_equal(R.U.rp, f.upper.row_offsets) and np.array_equal(R.U.ci, f.upper.col_indices)
        assert same_bits(R.L.v, f.lower.values) and same_bits(R.U.v, f.upper.values)
        erp, eci, ev = np.asarray(erp), np.asarray(eci, np.int64), np.asarray(ev)
        w = np.array([np.dot(ev[erp[i]:erp[i + 1]], x2[eci[erp[i]:erp[i + 1]]]) for i in range(d)])
        want = R.solve(y[r0:r1]) - R.solve(w)
        for mode in ("on", "off"):
            assert rel_err(xs[mode][r0:r1], want) <= APPLY_TOL, (b, mode)


def test_host_buffer_spmv_coupled_split(msc, ctx, rs):
    """PartitionedMatrix::from_split accepts interior ranges that are still
    coupled (entries of C[0:p, 0:p] between blocks); the preconditioner keeps
    only the diagonal blocks, but matvec(C, x) with page-locked host buffers
    must still be the full product: bit-identical to the reference matvec,
    also right after a call with a different x (no stale rows)."""
    import ctypes as C
    import torch
    from paper_1104_3349_b200 import _capi
    rng = np.random.default_rng(31)
    n, p = 600, 480
    a = np.zeros((n, n))
    a[:p, :p] = (rng.uniform(size=(p, p)) < 0.02) * rng.uniform(-1, 1, (p, p))
    a[np.arange(p), np.arange(p)] = 8.0 + rng.uniform(0, 1, p)
    a[:p, p:] = (rng.uniform(size=(p, n - p)) < 0.03) * rng.uniform(-1, 1, (p, n - p))
    a[p:, :p] = (rng.uniform(size=(n - p, p)) < 0.03) * rng.uniform(-1, 1, (n - p, p))
    a[np.arange(p, n), np.arange(p, n)] = 1.0
    Cm = msc.SparseMatrix.from_dense(a)
    ranges = [(0, 120), (120, 240), (240, 360), (360, 480)]
    S = msc.SparseMatrix.from_dense(np.eye(n - p) * 2.0)
    pc = msc.build_preconditioner_arrays(ctx, Cm, p, ranges, S, [(0, n - p)], tolA=1e-4, sA=1000)
    mat = _capi.lib().mscg_precond_matrix(pc.h)
    st = _capi.Status()
    for seed in (1, 2, 3):
        x = rng.uniform(-1, 1, n) * seed
        want = rs.matvec(*Cm.arrays(), x)
        xp = torch.from_numpy(x).pin_memory()
        yp = torch.full((n,), float("nan"), dtype=torch.float64).pin_memory()
        rc = _capi.lib().mscg_spmv(mat, C.c_void_p(xp.data_ptr()), C.c_void_p(yp.data_ptr()),
                                   _capi.MEM_HOST, C.byref(st))
        assert rc == 0, st.message
        assert same_bits(yp.numpy(), want)


@pytest.mark.parametrize("variant,grid,nu,n_a,sz,overlap", [
    ("omscn", 32, 0.1, 8, 0, -1),     # cfg1, overlap = sz (clipped)
    ("omscnr", 32, 0.1, 8, 0, 5),
    ("olum", 64, 0.01, 16, 40, 12),
    ("olum", 128, 0.01, 16, 0, 40),   # cfg2 grid: band of n_g = 1264
])
def test_overlapped_schur_band_matches_reference(msc, ctx, ref, variant, grid, nu, n_a, sz,
                                                 overlap):
    """Overlapped variants end to end on the device: build_msc over
    overlapped aggregates (device local blocks, reference merge) gives the
    reference's banded S^ bit for bit; the preconditioner factors the band
    whole by one exact LU (schur_single_, preconditioner.cpp:58-67,100-102):
    its factor is the reference's, the apply matches the reference's
    MscPreconditioner::apply to 1e-10, and right-preconditioned GMRES takes
    the reference's iteration count."""
    R = ref.Problem.oseen(grid, nu, n_a)
    P = msc.oseen_problem(grid, nu, n_a)
    R.build_schur(variant, sz, 0, overlap=overlap)
    P.build_msc(variant, sz=sz, overlap=overlap, ctx=ctx)
    Rs, Ps = R.csr(5), P.s_hat
    assert np.array_equal(Rs.rp, Ps.row_offsets) and np.array_equal(Rs.ci, Ps.col_indices)
    assert same_bits(Rs.v, Ps.values)
    R.build_precond(1e-4, 0)
    pc = msc.build_preconditioner(P, tolA=1e-4, sA=0, ctx=ctx)
    assert pc.kind() == variant
    f = pc.schur_factors(0)
    assert f.dim() == P.n - P.p
    L, U, perm = R.factors(1, 0)
    assert same_bits(f.lower.values, L.v) and same_bits(f.upper.values, U.v)
    assert np.array_equal(f.row_perm, perm)
    with pytest.raises(IndexError):
        R.factors(1, 1)  # one factor for the whole band
    assert pc.stored_nnz() == R.stored_nnz()
    for seed in (1, 2):
        y = ref.random_vector(P.n, seed)
        assert rel_err(pc.apply(y), R.apply(y)) <= APPLY_TOL
    if grid == 32:
        b = ref.random_vector(P.n, 0)
        want = R.gmres(b, 30, 3000, 1e-8)
        x, rep = msc.gmres(pc.matrix, pc, b, msc.SolverConfig(restart=30, rel_tol=1e-8))
        assert abs(rep.iterations - want["iterations"]) <= 1
        assert rep.converged and msc.true_residual(pc.matrix, x, b) <= 1e-8


def test_overlapped_band_singular_error(msc, ctx, ref):
    """A singular overlapped band raises the reference's error text
    ("build_preconditioner: overlapped Schur band: dense_lu: zero pivot at
    index i", preconditioner.cpp:58-67)."""
    n, p = 40, 30
    rng = np.random.default_rng(4)
    a = np.zeros((n, n))
    a[:p, :p] = np.diag(4.0 + rng.uniform(0, 1, p))
    a[:p, p:] = rng.uniform(-1, 1, (p, n - p)) * (rng.uniform(size=(p, n - p)) < 0.3)
    a[p:, :p] = a[:p, p:].T
    Cm = msc.SparseMatrix.from_dense(a)
    band = np.eye(n - p)
    band[3, 3] = 0.0  # zero column 3 of the band
    band[3, 4] = 1.0
    S = msc.SparseMatrix.from_dense(band)
    with pytest.raises(msc.SingularMatrixError) as e:
        msc.build_preconditioner_arrays(ctx, Cm, p, [(0, 15), (15, 30)], S, None, sA=1000,
                                        kind="omscn")
    assert str(e.value) == ("build_preconditioner: overlapped Schur band: dense_lu: zero pivot "
                            "at index 3")
    assert e.value.pivot_index == 3


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_nested_dissection_device_matches_reference(msc, ctx, ref, seed):
    """Nested dissection on the device (csrc/device/dissect.cu, SURVEY 8(f)
    row 2): random patterns with disconnected pieces, isolated nodes and
    nonsymmetric rows, plus grid graphs — the reference's permutation and
    block ranges exactly."""
    from test_host_setup import _random_pattern
    rng = np.random.default_rng(100 + seed)
    cases = []
    for _ in range(12):
        n = int(rng.integers(3, 2000))
        cases.append((_random_pattern(msc, rng, n, int(rng.integers(1, 4)),
                                      int(rng.integers(1, 6)), bool(rng.integers(0, 2))),
                      int(rng.integers(1, min(n, 256) + 1))))
    m = 40 + seed
    g = np.zeros((m * m, m * m))
    for i in range(m):
        for j in range(m):
            u = i * m + j
            if i + 1 < m:
                g[u, u + m] = g[u + m, u] = 1
            if j + 1 < m:
                g[u, u + 1] = g[u + 1, u] = 1
    cases.append((msc.SparseMatrix.from_dense(g), 64))
    for A, target in cases:
        p_ref, r_ref = ref.nested_dissection(A.row_offsets, A.col_indices, target)
        p, r = msc.nested_dissection(A, target, ctx=ctx)
        assert np.array_equal(p, p_ref) and np.array_equal(r, r_ref), (A.nrows, target)


def test_nested_dissection_device_many_pieces(msc, ctx, ref):
    """More than 8191 pieces at the last levels: the device dissection falls
    back from the cooperative search to the per-round kernels (global piece
    prefix); still the reference's permutation and ranges."""
    import scipy.sparse as sp
    m = 300
    e = np.ones(m)
    T = sp.diags([e[:-1], e[:-1]], [-1, 1], shape=(m, m))
    G = (sp.kron(sp.eye(m), T) + sp.kron(T, sp.eye(m)) + sp.eye(m * m)).tocsr()
    G.sort_indices()
    A = msc.SparseMatrix(m * m, m * m, G.indptr.astype(np.int32), G.indices.astype(np.int32),
                         G.data.astype(np.float64))
    target = 16384
    p_ref, r_ref = ref.nested_dissection(A.row_offsets, A.col_indices, target)
    p, r = msc.nested_dissection(A, target, ctx=ctx)
    assert len(r_ref) > 8192
    assert np.array_equal(p, p_ref) and np.array_equal(r, r_ref)


def test_device_partition_cfg4_digest(msc, ctx):
    """cfg4 (1024^2, 1024 blocks, anchored) through the device problem path
    (device assembly + device nested dissection): C and the permutation
    equal the reference's digests (tests/golden/cfg4.json)."""
    js = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg4.json")))
    P = msc.oseen_problem(1024, 0.001, 1024, anchored=True, ctx=ctx)
    from test_host_setup import csr_digest, digest
    assert csr_digest(P.C) == js["c_sha"]
    assert digest(P.perm().astype("<i4")) == js["perm_sha"]
