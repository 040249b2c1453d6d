"""CPU: the product's host problem layer (generate_oseen -> scale_rows ->
partition_saddle -> anchoring -> aggregates -> build_msc) reproduces the
reference's matrices bit for bit."""
import hashlib
import json
import os

import numpy as np
import pytest

from helpers import same_bits

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_digest(a):
    return digest(a.row_offsets.astype("<i4"), a.col_indices.astype("<i4"),
                  a.values.astype("<f8"))


def test_cfg1_matches_golden(msc):
    js = json.load(open(os.path.join(GOLDEN, "cfg1.json")))
    z = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    pb = msc.oseen_problem(32, 0.1, 8)
    pb.build_msc("lum")
    C = pb.C
    assert (pb.n, pb.p, pb.nblocks, C.nnz) == (js["n"], js["p"], js["nblocks"], js["nnz_c"])
    assert np.array_equal(C.row_offsets, z["c_rp"]) and np.array_equal(C.col_indices, z["c_ci"])
    assert same_bits(C.values, z["c_v"])
    assert np.array_equal(pb.perm(), z["perm"])
    assert pb.d_ranges().tolist() == js["d_ranges"]
    assert pb.schur_ranges().tolist() == js["schur_ranges"]
    assert csr_digest(pb.s_hat) == js["s_hat_sha"]


def test_cfg2_matches_golden(msc):
    js = json.load(open(os.path.join(GOLDEN, "cfg2.json")))
    pb = msc.oseen_problem(128, 0.01, 16)
    pb.build_msc("lum")
    assert csr_digest(pb.C) == js["c_sha"]
    assert digest(pb.perm().astype("<i4")) == js["perm_sha"]
    assert pb.d_ranges().tolist() == js["d_ranges"]
    assert csr_digest(pb.s_hat) == js["s_hat_sha"]


def test_cfg3_stretched_matches_golden(msc):
    js = json.load(open(os.path.join(GOLDEN, "cfg3_error.json")))
    pb = msc.oseen_problem(256, 0.002, 64, stretched=True, stretch=1.1)
    assert csr_digest(pb.C) == js["c_sha"]


@pytest.mark.parametrize("name,grid,nu,n_a", [("cfg4", 1024, 0.001, 1024)])
def test_large_config_digest(msc, name, grid, nu, n_a):
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip("large-config digest not generated (make_golden.py --large)")
    js = json.load(open(path))
    pb = msc.oseen_problem(grid, nu, n_a, anchored=True)
    pb.build_msc("lum", sz=256, mode="anchored")
    assert (pb.n, pb.p, pb.nblocks) == (js["n"], js["p"], js["nblocks"])
    assert csr_digest(pb.C) == js["c_sha"]
    assert digest(pb.perm().astype("<i4")) == js["perm_sha"]
    assert pb.schur_ranges().tolist() == js["schur_ranges"]
    assert csr_digest(pb.s_hat) == js["s_hat_sha"]


CASES = [
    (16, 0.1, 4, False, 1.056, False),
    (32, 0.002, 4, False, 1.056, False),
    (24, 0.05, 8, True, 1.08, False),
    (40, 0.01, 16, False, 1.056, True),
    (64, 0.01, 32, False, 1.056, True),
    (17, 0.1, 3, True, 1.2, False),     # odd grid, non power-of-two target
]


@pytest.mark.parametrize("grid,nu,n_a,stretched,stretch,anchored", CASES)
def test_matches_live_reference(msc, ref, grid, nu, n_a, stretched, stretch, anchored):
    R = ref.Problem.oseen(grid, nu, n_a, stretched=stretched, stretch=stretch, anchored=anchored)
    P = msc.oseen_problem(grid, nu, n_a, stretched=stretched, stretch=stretch, anchored=anchored)
    Rc, Pc = R.csr(0), P.C
    assert np.array_equal(Rc.rp, Pc.row_offsets) and np.array_equal(Rc.ci, Pc.col_indices)
    assert same_bits(Rc.v, Pc.values)
    assert np.array_equal(R.perm(), P.perm())
    assert np.array_equal(R.d_ranges(), P.d_ranges())
    assert same_bits(R.scaled_rhs(), P.scaled_rhs())
    mode_r, mode_p, sz = (1, "anchored", 12) if anchored else (0, "equal", 0)
    for variant in ("lum", "mscn", "mscnr"):
        err_r = err_p = None
        try:
            R.build_schur(variant, sz, mode_r)
        except ref.RefError as e:
            err_r = str(e)
        try:
            P.build_msc(variant, sz=sz, mode=mode_p)
        except (msc.SingularMatrixError, ValueError) as e:
            err_p = str(e)
        assert err_r == err_p
        if err_r:
            continue
        Rs, Ps = R.csr(5), P.s_hat
        assert np.array_equal(Rs.rp, Ps.row_offsets) and np.array_equal(Rs.ci, Ps.col_indices)
        assert same_bits(Rs.v, Ps.values)
        assert np.array_equal(R.schur_ranges(), P.schur_ranges())


def test_thread_count_does_not_change_partition(msc):
    a = msc.oseen_problem(48, 0.01, 16, threads=1)
    b = msc.oseen_problem(48, 0.01, 16, threads=7)
    assert csr_digest(a.C) == csr_digest(b.C)
    assert np.array_equal(a.perm(), b.perm())


def test_setup_errors(msc):
    with pytest.raises(ValueError, match="grid_n must be >= 8"):
        msc.oseen_problem(4, 0.1, 2)
    with pytest.raises(ValueError, match="viscosity must be positive"):
        msc.oseen_problem(16, 0.0, 2)
    pb = msc.oseen_problem(16, 0.1, 4)
    with pytest.raises(ValueError, match="sizes sum to"):
        pb.build_msc("lum", mode="explicit", sizes=[1, 2])
    with pytest.raises(ValueError, match="unknown or unsupported MSC variant"):
        pb.build_msc("nope")


@pytest.mark.parametrize("variant", ["omscn", "omscnr", "olum"])
@pytest.mark.parametrize("grid,nu,n_a,sz,overlap", [
    (32, 0.1, 8, 0, -1),    # overlap = sz, clipped to size - 1
    (32, 0.1, 8, 0, 5),
    (64, 0.01, 16, 40, 12),  # OMSCN / OMSCNR: singular D block of aggregate 13
])
def test_overlapped_build_msc_matches_reference(msc, ref, variant, grid, nu, n_a, sz, overlap):
    """Overlapped numbering aggregates (aggregate_overlapped,
    aggregates.cpp:50-85, widths as make_aggregates makes them) and the
    banded S^ of build_msc (schur_approx.cpp:88-161): bit-identical to the
    live reference, identical errors."""
    R = ref.Problem.oseen(grid, nu, n_a)
    P = msc.oseen_problem(grid, nu, n_a)
    err_r = err_p = None
    try:
        R.build_schur(variant, sz, 0, overlap=overlap)
    except ref.RefError as e:
        err_r = str(e)
    try:
        P.build_msc(variant, sz=sz, overlap=overlap)
    except (msc.SingularMatrixError, ValueError) as e:
        err_p = str(e)
    assert err_r == err_p
    if err_r:
        return
    Rs, Ps = R.csr(5), P.s_hat
    assert np.array_equal(Rs.rp, Ps.row_offsets) and np.array_equal(Rs.ci, Ps.col_indices)
    assert same_bits(Rs.v, Ps.values)
    assert np.array_equal(R.schur_ranges(), P.schur_ranges())
    # banded: some owned column is written outside its own aggregate's rows
    ranges = P.schur_ranges()
    own = np.repeat(np.arange(len(ranges)), np.diff(ranges, axis=1).ravel())
    rows = np.repeat(np.arange(Ps.nrows), np.diff(Ps.row_offsets))
    assert np.any(own[rows] != own[Ps.col_indices])


def test_overlapped_aggregate_errors(msc):
    """aggregate_overlapped / check_agg_compatible argument errors
    (aggregates.cpp:57-74, schur_approx.cpp:65-72): same text."""
    P = msc.oseen_problem(32, 0.1, 8)
    ng = P.n - P.p
    k = len(np.asarray(msc.oseen_problem(32, 0.1, 8).build_msc("lum").schur_ranges()))
    with pytest.raises(ValueError, match="variant mscn needs a non-overlapped aggregate set"):
        P.build_msc("mscn", widths=[1] * (k - 1) + [0])
    with pytest.raises(ValueError, match="widths must be >= 0 and end with 0"):
        P.build_msc("omscn", widths=[1] * k)
    with pytest.raises(ValueError, match="violates w < size"):
        P.build_msc("omscn", widths=[ng] + [0] * (k - 1))
    with pytest.raises(ValueError, match="one width per aggregate"):
        P.build_msc("omscn", widths=[0])


def _random_pattern(msc, rng, n, deg, comps, symmetric):
    """Random sparse pattern with `comps` groups (disconnected pieces) and
    isolated nodes; nonsymmetric unless asked."""
    a = np.zeros((n, n))
    lab = rng.integers(0, comps, n)
    for i in range(n):
        for _ in range(deg):
            j = rng.integers(0, n)
            if lab[j] == lab[i]:
                a[i, j] = 1.0
    if symmetric:
        a = a + a.T
    return msc.SparseMatrix.from_dense(a + np.eye(n))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_nested_dissection_host_matches_reference(msc, ref, seed):
    """nested_dissection(build_graph(A), target) (graph.cpp:8-30,178-230) on
    random patterns — disconnected pieces, isolated nodes, nonsymmetric rows
    (the reference's build_graph keeps only later rows' in-edges) —
    identical permutation and block ranges."""
    rng = np.random.default_rng(seed)
    for _ in range(25):
        n = int(rng.integers(3, 400))
        A = _random_pattern(msc, rng, n, int(rng.integers(1, 4)), int(rng.integers(1, 5)),
                            bool(rng.integers(0, 2)))
        target = int(rng.integers(1, min(n, 128) + 1))
        p_ref, r_ref = ref.nested_dissection(A.row_offsets, A.col_indices, target)
        p, r = msc.nested_dissection(A, target)
        assert np.array_equal(p, p_ref) and np.array_equal(r, r_ref), (n, target)
