"""Shared test helpers: build the oracle (plain-C restatement) preconditioner
for a problem produced by the product's host layer, and comparison utils."""
import numpy as np


def csr_tuple(a):
    return (np.ascontiguousarray(a.row_offsets, np.int32),
            np.ascontiguousarray(a.col_indices, np.int32),
            np.ascontiguousarray(a.values, np.float64))


def split_blocks(C, p):
    """D, E, F CSR tuples of C split at p (PartitionedMatrix::from_split)."""
    rp, ci, v = csr_tuple(C)
    n = C.nrows

    def extract(rb, re, cb, ce):
        orp = [0]
        oci, ov = [], []
        for i in range(rb, re):
            s, e = rp[i], rp[i + 1]
            cols = ci[s:e]
            m = (cols >= cb) & (cols < ce)
            oci.append(cols[m] - cb)
            ov.append(v[s:e][m])
            orp.append(orp[-1] + int(m.sum()))
        return (np.asarray(orp, np.int32),
                np.concatenate(oci).astype(np.int32) if oci else np.zeros(0, np.int32),
                np.concatenate(ov).astype(np.float64) if ov else np.zeros(0))

    return extract(0, p, 0, p), extract(0, p, p, n), extract(p, n, 0, p)


def oracle_msc(rs, problem, tolA=1e-4, sA=0):
    C = problem.C
    D, E, F = split_blocks(C, problem.p)
    S = csr_tuple(problem.s_hat)
    return rs.Msc(problem.n, problem.p, D, E, F, S, problem.d_ranges(),
                  problem.schur_ranges(), tolA=tolA, sA=sA)


def rel_err(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (den if den else 1.0)


def same_bits(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))
