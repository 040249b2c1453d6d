"""CPU: pin the oracle restatement (oracle/restate.c) to the reference.

1. against the committed golden fixtures (produced by the compiled reference,
   tests/golden/make_golden.py) — runs anywhere, including the GPU box;
2. against the live compiled reference (oracle/_ref) on fresh random inputs
   where that library is available.
Bit-identical results are required: the restatement keeps the reference's
operation order and is compiled without FMA contraction.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from helpers import csr_tuple, same_bits

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def g1():
    return (json.load(open(os.path.join(GOLDEN, "cfg1.json"))),
            np.load(os.path.join(GOLDEN, "cfg1.npz")))


def _sub(rp, ci, v, b, e):
    import restatepy
    return restatepy._sub_csr(rp, ci, v, b, e)


def cfg1_oracle(rs, g1):
    js, z = g1
    n, p = js["n"], js["p"]
    rp, ci, v = z["c_rp"], z["c_ci"], z["c_v"]
    from helpers import split_blocks
    import paper_1104_3349_b200 as msc  # only for the SparseMatrix container
    C = msc.SparseMatrix(n, n, rp, ci, v)
    D, E, F = split_blocks(C, p)
    S = (z["s_rp"], z["s_ci"], z["s_v"])
    return rs.Msc(n, p, D, E, F, S, js["d_ranges"], js["schur_ranges"], 1e-4, 0)


def test_cfg1_factors_match_golden(rs, g1):
    js, z = g1
    M = cfg1_oracle(rs, g1)
    for b, want in enumerate(js["d_factors"]):
        f = M.dfac[b]
        assert int(f.lrp[-1]) == want["nnz_l"] and int(f.urp[-1]) == want["nnz_u"]
        assert digest(f.lrp.astype("<i4"), f.lci.astype("<i4"), f.lv.astype("<f8"),
                      f.urp.astype("<i4"), f.uci.astype("<i4"), f.uv.astype("<f8")) == want["sha"]
    assert M.stored_nnz == js["stored_nnz"]


def test_cfg1_apply_and_matvec_match_golden(rs, g1):
    js, z = g1
    M = cfg1_oracle(rs, g1)
    assert same_bits(M.apply(z["y"]), z["apply_y"])
    assert same_bits(rs.matvec(z["c_rp"], z["c_ci"], z["c_v"], z["y"]), z["matvec_y"])


def test_cfg1_gmres_matches_golden(rs, g1):
    js, z = g1
    M = cfg1_oracle(rs, g1)
    r = rs.gmres((z["c_rp"], z["c_ci"], z["c_v"]), z["y"], 30, 3000, 1e-8, msc=M)
    assert r["iterations"] == js["gmres"]["iterations"] == 88
    assert r["converged"]
    assert np.array_equal(r["history"], np.asarray(js["gmres"]["history"]))
    assert same_bits(r["x"], z["gmres_x"])


def test_random_saddles_match_golden(rs):
    import paper_1104_3349_b200 as msc
    from helpers import split_blocks
    cases = json.load(open(os.path.join(GOLDEN, "random_saddles.json")))
    z = np.load(os.path.join(GOLDEN, "random_saddles.npz"))
    for k, c in enumerate(cases):
        n = c["p"] + c["ng"]
        C = msc.SparseMatrix(n, n, z[f"c{k}_rp"], z[f"c{k}_ci"], z[f"c{k}_v"])
        D, E, F = split_blocks(C, c["p"])
        pb = msc.partitioned_problem(C, c["p"])
        pb.build_msc(c["variant"], mode="explicit", sizes=c["sizes"])
        S = csr_tuple(pb.s_hat)
        M = rs.Msc(n, c["p"], D, E, F, S, [(0, c["p"])], pb.schur_ranges(), c["tolA"], c["sA"])
        assert same_bits(M.apply(z[f"y{k}"]), z[f"x{k}"]), k
        assert same_bits(M.dfac[0].lv, z[f"l{k}_v"]) and same_bits(M.dfac[0].uv, z[f"u{k}_v"])
        assert M.stored_nnz == c["stored_nnz"]


def test_ilut_contracts(rs):
    """test_sparse_core.cpp:161-190: tol 0 reproduces the matrix, tol 1e30
    keeps only the diagonal in U and nothing in L, nnz is monotone in tol."""
    z = np.load(os.path.join(GOLDEN, "ilut_contracts.npz"))
    a = z["a"]
    import paper_1104_3349_b200 as msc
    A = msc.SparseMatrix.from_dense(a)
    nnz = []
    for tol in (0.0, 1e-3, 1e-1, 1e30):
        f = rs.factor_ilut(A.nrows, *A.arrays(), tol)
        key = str(tol).replace(".", "p").replace("-", "m").replace("+", "")
        L = msc.SparseMatrix(A.nrows, A.nrows, f.lrp, f.lci, f.lv).to_dense()
        U = msc.SparseMatrix(A.nrows, A.nrows, f.urp, f.uci, f.uv).to_dense()
        assert np.array_equal(L, z[f"L_{key}"]) and np.array_equal(U, z[f"U_{key}"])
        nnz.append(f.nnz)
        if tol == 0.0:
            lu = (L + np.eye(A.nrows)) @ U
            assert np.linalg.norm(lu - a) <= 1e-12 * np.linalg.norm(a)
        if tol == 1e30:
            assert int(f.lrp[-1]) == 0 and int(f.urp[-1]) == A.nrows
    assert nnz == sorted(nnz, reverse=True)


def test_ilut_zero_pivot_throws(rs):
    import paper_1104_3349_b200 as msc
    a = np.array([[1.0, 2.0], [2.0, 4.0]])
    A = msc.SparseMatrix.from_dense(a)
    with pytest.raises(rs.SingularMatrixError) as e:
        rs.factor_ilut(2, *A.arrays(), 0.0)
    assert e.value.pivot_index == 1


def test_restatement_vs_live_reference(rs, ref):
    """Fresh random blocks: factors, solves and SpMV bit-identical."""
    rng = np.random.default_rng(123)
    for trial in range(6):
        n = int(rng.integers(5, 60))
        a = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.25)
        a += np.diag(np.abs(a).sum(1) + rng.random(n))
        rows, cols = np.nonzero(a)
        rp = np.zeros(n + 1, np.int32)
        np.add.at(rp, rows + 1, 1)
        rp = np.cumsum(rp).astype(np.int32)
        ci, v = cols.astype(np.int32), a[rows, cols].copy()
        A = ref.Csr(n, n, rp, ci, v)
        for tol in (0.0, 1e-3, 0.2):
            fr = ref.factor_ilut(A, tol)
            fo = rs.factor_ilut(n, rp, ci, v, tol)
            assert np.array_equal(fr.L.rp, fo.lrp) and same_bits(fr.L.v, fo.lv)
            assert np.array_equal(fr.U.ci, fo.uci) and same_bits(fr.U.v, fo.uv)
            b = rng.uniform(-1, 1, n)
            assert same_bits(fr.solve(b), fo.solve(b))
        fe = ref.factor_exact(A)
        fo = rs.factor_exact(n, rp, ci, v)
        assert np.array_equal(fe.perm, fo.perm) and same_bits(fe.U.v, fo.uv)
        x = rng.uniform(-1, 1, n)
        P = ref.Problem.from_csr(A, n)
        assert same_bits(rs.matvec(rp, ci, v, x), P.matvec(x, 0))


def test_restatement_apply_vs_live_reference(rs, ref):
    import paper_1104_3349_b200 as msc
    from helpers import split_blocks
    R = ref.Problem.oseen(16, 0.1, 4)
    R.build_schur("lum", 0, 0)
    R.build_precond(1e-4, 0)
    Cr = R.csr(0)
    C = msc.SparseMatrix(R.n, R.n, Cr.rp, Cr.ci, Cr.v)
    D, E, F = split_blocks(C, R.p)
    S = R.csr(5)
    M = rs.Msc(R.n, R.p, D, E, F, (S.rp, S.ci, S.v), R.d_ranges(), R.schur_ranges(), 1e-4, 0)
    for seed in range(3):
        y = ref.random_vector(R.n, seed)
        assert same_bits(M.apply(y), R.apply(y))
    y = ref.random_vector(R.n, 5)
    a = R.gmres(y, 20, 500, 1e-9)
    b = rs.gmres((Cr.rp, Cr.ci, Cr.v), y, 20, 500, 1e-9, msc=M)
    assert a["iterations"] == b["iterations"] and np.array_equal(a["history"], b["history"])
    for side in ("left",):
        a = R.gmres(y, 20, 500, 1e-9, left=True)
        b = rs.gmres((Cr.rp, Cr.ci, Cr.v), y, 20, 500, 1e-9, msc=M, side=side)
        assert a["iterations"] == b["iterations"] and np.array_equal(a["history"], b["history"])
