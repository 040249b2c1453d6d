"""GPU parity at every BASELINE config, against the UNMODIFIED reference.

Fixtures (tests/golden/, produced by tests/golden/make_golden.py running the
compiled reference in the build container):
  cfg2   GMRES(50) history to rtol 1e-8 (1844 iterations, converged)
  cfg3'  (stretch 1.0313) full apply(y) vector + the capped GMRES(50) history
  cfg4   apply(y) fingerprint + the first GMRES(100) cycle (100 iterations)
  cfg5   apply(y) fingerprint
At cfg4 / cfg5 the whole apply vector, interface part included, is also
checked live against the reference's own MscPreconditioner::apply
(preconditioner.cpp:85-114), run on the GPU's interior factors (shown
bit-identical to the reference ILUT on sampled blocks, and through the
fingerprint on every block) with the reference's own Schur factors, E, F and
matvec.  The ILUT contract cases of test_sparse_core.cpp:161-190 and
acceptance criterion #9 run on the device ILUT kernel.

Bars (BASELINE.json north_star): apply <= 1e-10 relative (fp64); GMRES
iteration counts within +-1 and both residuals < tol where the reference
converges; capped runs end NC at the same cap with matching histories.
"""
import json
import os
import threading

import numpy as np
import pytest

from helpers import rel_err, same_bits

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-10
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return json.load(open(os.path.join(GOLDEN, name)))


def ref_csr(ref, a):
    return ref.Csr(a.nrows, a.ncols, np.ascontiguousarray(a.row_offsets, np.int32),
                   np.ascontiguousarray(a.col_indices, np.int32),
                   np.ascontiguousarray(a.values, np.float64))


def history_dev(got, want, k):
    """max relative deviation of the first k residual-history entries."""
    g = np.asarray(got[:k])
    w = np.asarray(want[:k])
    return float(np.max(np.abs(g - w) / np.abs(w)))


# ---- ILUT / exact LU contracts on the device kernels -----------------------

def _dense(f):
    return f.lower.to_dense(), f.upper.to_dense()


def _spd_tridiag(msc, n):
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = 4.0
        if i + 1 < n:
            a[i, i + 1] = a[i + 1, i] = -1.0
    return msc.SparseMatrix.from_dense(a)


def _same_factors(f, r):
    assert np.array_equal(f.lower.row_offsets, r.L.rp)
    assert np.array_equal(f.lower.col_indices, r.L.ci)
    assert same_bits(f.lower.values, r.L.v)
    assert np.array_equal(f.upper.row_offsets, r.U.rp)
    assert np.array_equal(f.upper.col_indices, r.U.ci)
    assert same_bits(f.upper.values, r.U.v)


def test_ilut_tol0_reconstructs(msc, ctx, ref):
    """test_sparse_core.cpp:161-165: ILUT(0) of spd_tridiag(10) rebuilds A."""
    a = _spd_tridiag(msc, 10)
    f = msc.factor_ilut(a, 0.0, ctx=ctx)
    lo, up = _dense(f)
    lu = (lo + np.eye(10)) @ up
    A = a.to_dense()
    assert np.linalg.norm(lu - A) / np.linalg.norm(A) < 1e-12
    _same_factors(f, ref.factor_ilut(ref_csr(ref, a), 0.0))


def test_ilut_huge_tol_keeps_diagonal(msc, ctx, ref):
    """test_sparse_core.cpp:167-174: tol 1e30 keeps only the diagonal."""
    r = ref.random_dd_sparse(12, 0.4, 3)
    a = msc.SparseMatrix(r.nrows, r.ncols, r.rp, r.ci, r.v)
    f = msc.factor_ilut(a, 1e30, ctx=ctx)
    assert f.lower.nnz == 0 and f.upper.nnz == 12
    A = a.to_dense()
    assert np.array_equal(np.diag(f.upper.to_dense()), np.diag(A))
    _same_factors(f, ref.factor_ilut(r, 1e30))


def test_ilut_nnz_monotone_in_tol(msc, ctx, ref):
    """test_sparse_core.cpp:176-185 (random_dd_sparse(60, 0.15), seed 5)."""
    r = ref.random_dd_sparse(60, 0.15, 5)
    a = msc.SparseMatrix(r.nrows, r.ncols, r.rp, r.ci, r.v)
    prev = None
    for tol in (0.0, 1e-6, 1e-3, 1e-1, 1e30):
        f = msc.factor_ilut(a, tol, ctx=ctx)
        assert prev is None or f.nnz() <= prev
        prev = f.nnz()
        _same_factors(f, ref.factor_ilut(r, tol))


def test_ilut_zero_pivot_throws(msc, ctx, ref):
    """test_sparse_core.cpp:187-190: [[0, 1], [1, 0]] raises SingularMatrixError
    with the reference's message and pivot."""
    a = msc.SparseMatrix.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(msc.SingularMatrixError) as e:
        msc.factor_ilut(a, 0.0, ctx=ctx)
    with pytest.raises(ref.RefError) as r:
        ref.factor_ilut(ref_csr(ref, a), 0.0)
    assert str(e.value) == str(r.value)
    assert e.value.pivot_index == r.value.pivot_index == 0
    with pytest.raises(ValueError, match="negative drop tolerance"):
        msc.factor_ilut(a, -1.0, ctx=ctx)


def test_factor_exact_singular_pivot(msc, ctx, ref):
    """test_sparse_core.cpp:150-158: [[1, 2], [2, 4]] -> pivot 1."""
    a = msc.SparseMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 4.0]]))
    with pytest.raises(msc.SingularMatrixError) as e:
        msc.factor_exact(a, ctx=ctx)
    assert e.value.pivot_index == 1
    with pytest.raises(ref.RefError) as r:
        ref.factor_exact(ref_csr(ref, a))
    assert str(e.value) == str(r.value)


def test_factor_exact_and_solve_match_reference(msc, ctx, ref):
    r = ref.random_dd_sparse(40, 0.2, 11)
    a = msc.SparseMatrix(r.nrows, r.ncols, r.rp, r.ci, r.v)
    f = msc.factor_exact(a, ctx=ctx)
    rf = ref.factor_exact(r)
    assert np.array_equal(f.row_perm, rf.perm)
    _same_factors(f, rf)
    b = ref.random_vector(40, 2)
    assert rel_err(f.solve(b), rf.solve(b)) <= 1e-13


def test_ilut_oseen_block_acceptance9(msc, ctx, ref):
    """acceptance.cpp:513-537: ILUT(0) of the Oseen (1,1) block (grid 16,
    nu 0.01) rebuilds D to 1e-12, nnz non-increasing over the tol ladder;
    every factor bit-identical to the reference's, solve to 1e-13."""
    r = ref.oseen_raw_d(16, 0.01)
    a = msc.SparseMatrix(r.nrows, r.ncols, r.rp, r.ci, r.v)
    A = a.to_dense()
    prev = None
    b = ref.random_vector(a.nrows, 4)
    for tol in (0.0, 1e-6, 1e-4, 1e-2, 1.0):
        f = msc.factor_ilut(a, tol, ctx=ctx)
        rf = ref.factor_ilut(r, tol)
        _same_factors(f, rf)
        assert rel_err(f.solve(b), rf.solve(b)) <= 1e-13
        if tol == 0.0:
            lo, up = _dense(f)
            lu = (lo + np.eye(a.nrows)) @ up
            assert np.linalg.norm(lu - A) / np.linalg.norm(A) <= 1e-12
        assert prev is None or f.nnz() <= prev
        prev = f.nnz()


# ---- concurrency (preconditioner.hpp:17-18) ---------------------------------

def test_concurrent_applies_on_two_streams(msc, ctx, ref):
    """Two threads apply the same preconditioner on two streams at once
    (per-stream scratch): every result equals the serial apply bit for bit."""
    import torch
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    ys = [torch.from_numpy(ref.random_vector(pb.n, 40 + k)).cuda() for k in range(4)]
    want = [pc.apply(y).cpu().numpy() for y in ys]
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [[torch.full((pb.n,), float("nan"), dtype=torch.float64, device="cuda")
             for _ in range(4)] for _ in range(2)]
    torch.cuda.synchronize()
    errors = []

    def worker(t):
        try:
            for rep in range(6):
                for k in range(4):
                    kk = (k + t + rep) % 4
                    pc.apply_on_stream(ys[kk], outs[t][kk], streams[t].cuda_stream)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errors
    for t in range(2):
        for k in range(4):
            assert same_bits(outs[t][k].cpu().numpy(), want[k])


def test_correction_toggle_same_operator(msc, ref):
    """use_correction(False) runs the reference's E SpMV + second interior
    solve on a preconditioner built with panels: same operator to 1e-12."""
    c = msc.Context(0)
    c.set_correction("on")
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=c)
    assert pc.correction()["on"]
    y = ref.random_vector(pb.n, 9)
    on = pc.apply(y)
    pc.use_correction(False)
    off = pc.apply(y)
    pc.use_correction(True)
    assert rel_err(on, off) <= 1e-12 and not same_bits(on, off)
    assert same_bits(pc.apply(y), on)


# ---- cfg2: GMRES(50) converges in 1844 iterations ---------------------------

def test_cfg2_gmres_matches_reference(msc, ctx, ref):
    g = golden("cfg2.json")["gmres"]
    assert g["iterations"] == 1844 and g["converged"]
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    b = ref.random_vector(pb.n, 0)
    x, rep = msc.gmres(pc.matrix, pc, b, msc.SolverConfig(restart=50, max_iters=3000,
                                                          rel_tol=1e-8))
    assert abs(rep.iterations - g["iterations"]) <= 1
    assert rep.converged
    tr = msc.true_residual(pc.matrix, x, b)
    assert tr < 1e-8 and g["history"][-1] < 1e-8
    # the recurrence residuals track the reference's: first cycle tightly,
    # the whole run within 1e-3 relative (CGS2 vs the reference's MGS)
    h = rep.residual_history
    assert history_dev(h, g["history"], 51) <= 1e-7
    k = min(len(h), len(g["history"])) - 2
    assert history_dev(h, g["history"], k) <= 1e-3


# ---- cfg3' (stretch 1.0313): apply vector + capped GMRES(50) ---------------

def test_cfg3p_apply_and_capped_gmres(msc, ctx, ref):
    g = golden("cfg3p.json")
    want = np.load(os.path.join(GOLDEN, "cfg3p_apply.npz"))["apply_y"]
    pb = msc.oseen_problem(256, 0.002, 64, stretched=True, stretch=1.0313, ctx=ctx)
    pb.build_msc("lum", sz=795, ctx=ctx)
    from test_host_setup import csr_digest, digest
    assert csr_digest(pb.C) == g["c_sha"]
    assert digest(pb.perm().astype("<i4")) == g["perm_sha"]
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    assert pc.stored_nnz() == g["stored_nnz"]
    y = ref.random_vector(pb.n, 0)
    x = pc.apply(y)
    assert rel_err(x, want) <= APPLY_TOL
    assert rel_err(x[pb.p:], want[pb.p:]) <= APPLY_TOL
    gm = g["gmres"]
    assert gm["iterations"] == 3000 and not gm["converged"]
    x, rep = msc.gmres(pc.matrix, pc, y, msc.SolverConfig(restart=50, max_iters=3000,
                                                          rel_tol=1e-8))
    assert rep.iterations == gm["iterations"] and not rep.converged
    h = rep.residual_history
    assert len(h) == len(gm["history"])
    assert history_dev(h, gm["history"], 51) <= 1e-7
    assert history_dev(h, gm["history"], len(h)) <= 5e-2
    tr = msc.true_residual(pc.matrix, x, y)
    assert abs(tr - gm["history"][-1]) <= 5e-2 * gm["history"][-1]


# ---- cfg4 / cfg5: fingerprints, first GMRES cycle, live full vector --------

def _fingerprint_check(x, fp, d_ranges, s_ranges, p, tol=APPLY_TOL):
    bn = np.array([np.linalg.norm(x[a:b]) for a, b in d_ranges])
    an = np.array([np.linalg.norm(x[p + a:p + b]) for a, b in s_ranges])
    assert np.max(np.abs(bn - fp["block_norm"]) / fp["block_norm"]) <= tol
    assert np.max(np.abs(an - fp["agg_norm"]) / fp["agg_norm"]) <= tol
    bs = np.array([np.sum(x[a:b]) for a, b in d_ranges])
    assert np.max(np.abs(bs - fp["block_sum"])) <= tol * np.max(fp["block_norm"]) * 100
    smp = x[::int(fp["stride"][0])]
    assert rel_err(smp, fp["sample"]) <= tol
    assert abs(np.linalg.norm(x) - fp["norm"][0]) <= tol * fp["norm"][0]


def _reference_apply_on_gpu_factors(ref, pb, pc, y):
    """The reference's own apply, on the product's (reference-identical)
    problem arrays and the GPU's interior factors; the Schur blocks are
    factored by the reference's factor_exact."""
    R = ref.Problem.from_arrays(ref_csr(ref, pb.C), pb.p, pb.d_ranges())
    R.set_schur("lum", ref_csr(ref, pb.s_hat), pb.schur_ranges())

    def block(b):
        f = pc.d_factors(b)
        return f.lower.nrows, ref_csr(ref, f.lower), ref_csr(ref, f.upper)

    R.precond_from_factors(block)
    return R, R.apply_threads(y)


@pytest.mark.parametrize("name,grid,nu,n_a", [("cfg4", 1024, 0.001, 1024),
                                              ("cfg5", 2048, 0.01, 4096)])
def test_full_scale_full_vector_apply(msc, ref, name, grid, nu, n_a):
    """BASELINE cfg4 / cfg5 (anchored LUM sz 256): the WHOLE apply vector,
    interface part included, against the reference's apply, in both
    correction modes; the fingerprint of the independent reference run (its
    own ILUT of every block) on every block and aggregate; at cfg4 the first
    GMRES(100) cycle's history."""
    import torch
    g = golden(f"{name}.json")
    fp = np.load(os.path.join(GOLDEN, f"{name}_apply_fp.npz"))
    ctx = msc.Context(0)
    ctx.set_correction("on")
    pb = msc.oseen_problem(grid, nu, n_a, anchored=True, ctx=ctx)
    pb.build_msc("lum", sz=256, mode="anchored", ctx=ctx)
    from test_host_setup import csr_digest
    assert csr_digest(pb.C) == g["c_sha"] and csr_digest(pb.s_hat) == g["s_hat_sha"]
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    assert pc.correction()["on"]
    assert pc.stored_nnz() == g["stored_nnz"]
    y = ref.random_vector(pb.n, 0)
    yd = torch.from_numpy(y).cuda()
    x_on = pc.apply(yd).cpu().numpy()
    pc.use_correction(False)
    x_off = pc.apply(yd).cpu().numpy()
    pc.use_correction(True)
    dr, sr, p = pb.d_ranges(), pb.schur_ranges(), pb.p
    R, want = _reference_apply_on_gpu_factors(ref, pb, pc, y)
    # the reference apply on the GPU factors reproduces the independent
    # reference run (its own ILUT of every block) to rounding of the norms
    _fingerprint_check(want, fp, dr, sr, p, tol=1e-13)
    for x in (x_on, x_off):
        assert rel_err(x, want) <= APPLY_TOL
        assert rel_err(x[p:], want[p:]) <= APPLY_TOL
        _fingerprint_check(x, fp, dr, sr, p)
    del R
    if name == "cfg4":
        gm = g["gmres_first_cycle"]
        x, rep = msc.gmres(pc.matrix, pc, y, msc.SolverConfig(restart=100, max_iters=100,
                                                              rel_tol=1e-8))
        assert rep.iterations == gm["iterations"] == 100 and not rep.converged
        h = rep.residual_history
        assert len(h) == len(gm["history"])
        assert history_dev(h, gm["history"], len(h)) <= 1e-6
