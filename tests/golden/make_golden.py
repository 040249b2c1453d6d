"""Generate the committed golden fixtures from the UNMODIFIED reference.

Runs the compiled reference (oracle/_ref/libmscref.so, built in place from
/root/reference/proj/src by oracle/Makefile) in this container and writes
small fixtures next to this script.  The GPU box never reads
/root/reference; tests there compare against these files and against the
oracle restatement.

    python tests/golden/make_golden.py [--cfg2]     (--cfg2 adds the 3-minute
                                                     GMRES(50) reference solve)
    python tests/golden/make_golden.py --only cfg3p|cfg4|cfg5
        cfg3p: BASELINE cfg3 at stretch 1.0313: full apply(y) + the capped
               GMRES(50) history (3000 its, ~15 min);
        cfg4:  apply(y) fingerprint + the first GMRES(100) cycle (100 its,
               ~10 min after a ~2 min threaded ILUT);
        cfg5:  apply(y) fingerprint (~55 GB host RAM).
    The large configs factor their interior blocks with the reference's
    factor_ilut on all host threads (ref_build_precond_parallel: the same
    MscPreconditioner build_preconditioner returns, only the block loop is
    concurrent); apply and gmres are the reference's own, single-threaded.
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import refpy  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_digest(a) -> str:
    return digest(a.rp.astype("<i4"), a.ci.astype("<i4"), a.v.astype("<f8"))


def problem_summary(P, with_factors=True):
    C = P.csr(0)
    out = dict(n=P.n, p=P.p, nblocks=P.nblocks, nnz_c=C.nnz,
               c_sha=csr_digest(C), perm_sha=digest(P.perm().astype("<i4")),
               d_ranges=P.d_ranges().tolist())
    try:
        out["schur_ranges"] = P.schur_ranges().tolist()
        out["s_hat_sha"] = csr_digest(P.csr(5))
    except Exception:
        pass
    if with_factors:
        fl = []
        for b in range(P.nblocks):
            L, U, perm = P.factors(0, b)
            fl.append(dict(nnz_l=L.nnz, nnz_u=U.nnz, sha=digest(
                L.rp.astype("<i4"), L.ci.astype("<i4"), L.v.astype("<f8"),
                U.rp.astype("<i4"), U.ci.astype("<i4"), U.v.astype("<f8"))))
        out["d_factors"] = fl
        out["stored_nnz"] = P.stored_nnz()
    return out


def cfg1():
    P = refpy.Problem.oseen(32, 0.1, 8)
    P.build_schur("lum", 0, 0)
    P.build_precond(1e-4, 0)
    y = refpy.random_vector(P.n, 0)
    x = P.apply(y)
    r = P.gmres(y, 30, 3000, 1e-8)
    s = problem_summary(P)
    s["gmres"] = dict(restart=30, rel_tol=1e-8, iterations=r["iterations"],
                      converged=r["converged"], history=r["history"].tolist())
    C = P.csr(0)
    S = P.csr(5)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), c_rp=C.rp, c_ci=C.ci, c_v=C.v,
                        perm=P.perm(), y=y, apply_y=x, matvec_y=P.matvec(y), gmres_x=r["x"],
                        s_rp=S.rp, s_ci=S.ci, s_v=S.v)
    with open(os.path.join(HERE, "cfg1.json"), "w") as f:
        json.dump(s, f, indent=1)


def random_saddles():
    cases = []
    arrays = {}
    for k, (p, ng, seed, dens, variant, sizes, sA, tol) in enumerate([
            (20, 8, 37, 0.3, "mscn", [4, 4], 1 << 30, 0.0),
            (20, 8, 23, 0.3, "lum", [4, 4], 1 << 30, 0.0),
            (18, 8, 47, 0.3, "mscnr", [4, 4], 1 << 30, 0.0),
            (60, 20, 5, 0.2, "mscn", [5, 5, 5, 5], 1 << 30, 0.0),
            (40, 10, 9, 0.2, "lum", [10], 0, 1e-2),      # ILUT on one block
            (40, 10, 11, 0.2, "lum", [10], 0, 0.0)]):    # ILUT tol 0 == exact pattern
        P = refpy.Problem.random_saddle(p, ng, seed, dens)
        P.build_schur(variant, 0, 2, sizes=sizes)
        P.build_precond(tol, sA)
        C = P.csr(0)
        y = refpy.random_vector(P.n, 1000 + k)
        arrays[f"c{k}_rp"], arrays[f"c{k}_ci"], arrays[f"c{k}_v"] = C.rp, C.ci, C.v
        arrays[f"y{k}"] = y
        arrays[f"x{k}"] = P.apply(y)
        L, U, perm = P.factors(0, 0)
        arrays[f"l{k}_v"], arrays[f"u{k}_v"], arrays[f"u{k}_ci"] = L.v, U.v, U.ci
        cases.append(dict(p=p, ng=ng, seed=seed, density=dens, variant=variant, sizes=sizes,
                          sA=sA, tolA=tol, stored_nnz=P.stored_nnz()))
    np.savez_compressed(os.path.join(HERE, "random_saddles.npz"), **arrays)
    with open(os.path.join(HERE, "random_saddles.json"), "w") as f:
        json.dump(cases, f, indent=1)


def ilut_contracts():
    """test_sparse_core.cpp:161-190 analogues on a grid Laplacian-like matrix."""
    rng = np.random.default_rng(3)
    n = 40
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = 4.0 + rng.random()
        for j in (i - 1, i + 1, i - 7, i + 7):
            if 0 <= j < n:
                a[i, j] = -1.0 + 0.1 * rng.random()
    rows, cols = np.nonzero(a)
    rp = np.zeros(n + 1, np.int32)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    A = refpy.Csr(n, n, rp, cols.astype(np.int32), a[rows, cols].copy())
    out = {"a": a}
    for tol in (0.0, 1e-3, 1e-1, 1e30):
        f = refpy.factor_ilut(A, tol)
        key = str(tol).replace(".", "p").replace("-", "m").replace("+", "")
        out[f"L_{key}"] = f.L.to_dense()
        out[f"U_{key}"] = f.U.to_dense()
    np.savez_compressed(os.path.join(HERE, "ilut_contracts.npz"), **out)


def cfg3_error():
    P = refpy.Problem.oseen(256, 0.002, 64, stretched=True, stretch=1.1)
    P.build_schur("lum", 795, 0)
    try:
        P.build_precond(1e-4, 0)
        res = dict(error=None)
    except refpy.RefError as e:
        res = dict(error=str(e), pivot_index=e.pivot_index)
    res["c_sha"] = csr_digest(P.csr(0))
    with open(os.path.join(HERE, "cfg3_error.json"), "w") as f:
        json.dump(res, f, indent=1)


def cfg2(run_gmres: bool):
    P = refpy.Problem.oseen(128, 0.01, 16)
    P.build_schur("lum", 0, 0)
    t = time.time()
    P.build_precond(1e-4, 0)
    setup = time.time() - t
    s = problem_summary(P)
    s["setup_seconds_ref"] = setup
    y = refpy.random_vector(P.n, 0)
    t = time.time()
    x = P.apply(y)
    s["apply_seconds_ref"] = time.time() - t
    s["apply_y_sha"] = digest(x.astype("<f8"))
    s["apply_y_norm"] = float(np.linalg.norm(x))
    np.savez_compressed(os.path.join(HERE, "cfg2_apply.npz"), apply_y=x)
    if run_gmres:
        r = P.gmres(y, 50, 3000, 1e-8)
        s["gmres"] = dict(restart=50, rel_tol=1e-8, iterations=r["iterations"],
                          converged=r["converged"], seconds=r["seconds"],
                          history=r["history"].tolist())
    else:
        old = os.path.join(HERE, "cfg2.json")
        if os.path.exists(old):
            s["gmres"] = json.load(open(old)).get("gmres")
    with open(os.path.join(HERE, "cfg2.json"), "w") as f:
        json.dump(s, f, indent=1)


def apply_fingerprint(x, d_ranges, schur_ranges, p, nsample=50000):
    """Size-independent summary of an apply output that still touches every
    unknown: per interior block and per Schur aggregate the 2-norm and the
    plain sum, the global norm, and an evenly strided sample."""
    x = np.asarray(x, np.float64)
    stride = max(1, len(x) // nsample)
    blk = [x[a:b] for a, b in d_ranges]
    agg = [x[p + a:p + b] for a, b in schur_ranges]
    return dict(block_norm=np.array([np.linalg.norm(v) for v in blk]),
                block_sum=np.array([np.sum(v) for v in blk]),
                agg_norm=np.array([np.linalg.norm(v) for v in agg]),
                agg_sum=np.array([np.sum(v) for v in agg]),
                norm=np.array([np.linalg.norm(x)]), stride=np.array([stride]),
                sample=x[::stride].copy())


def _large_precond(grid_n, nu, n_a, variant, sz, mode, stretched=False, stretch=1.056,
                   anchored=False):
    t = time.time()
    P = refpy.Problem.oseen(grid_n, nu, n_a, stretched=stretched, stretch=stretch,
                            anchored=anchored)
    P.build_schur(variant, sz, mode, workers=0)
    t_setup = time.time() - t
    t = time.time()
    P.build_precond_parallel(1e-4, 0, workers=0)
    t_ilut = time.time() - t
    s = problem_summary(P, with_factors=False)
    s.pop("d_ranges")
    s["stored_nnz"] = P.stored_nnz()
    s["generate_partition_msc_seconds_ref"] = t_setup
    s["ilut_seconds_ref_threads"] = t_ilut
    s["threads"] = refpy.hardware_threads()
    return P, s


def cfg3p():
    """BASELINE cfg3 with stretch 1.0313 (max aspect 50.1)."""
    P, s = _large_precond(256, 0.002, 64, "lum", 795, 0, stretched=True, stretch=1.0313)
    y = refpy.random_vector(P.n, 0)
    t = time.time()
    x = P.apply(y)
    s["apply_seconds_ref"] = time.time() - t
    s["apply_y_norm"] = float(np.linalg.norm(x))
    np.savez_compressed(os.path.join(HERE, "cfg3p_apply.npz"), apply_y=x)
    r = P.gmres(y, 50, 3000, 1e-8)
    s["gmres"] = dict(restart=50, max_iters=3000, rel_tol=1e-8, iterations=r["iterations"],
                      converged=r["converged"], seconds=r["seconds"],
                      history=r["history"].tolist())
    with open(os.path.join(HERE, "cfg3p.json"), "w") as f:
        json.dump(s, f, indent=1)


def cfg4_cycle():
    """BASELINE cfg4: apply fingerprint + the first GMRES(100) cycle."""
    P, s = _large_precond(1024, 0.001, 1024, "lum", 256, 1, anchored=True)
    y = refpy.random_vector(P.n, 0)
    t = time.time()
    x = P.apply(y)
    s["apply_seconds_ref"] = time.time() - t
    fp = apply_fingerprint(x, P.d_ranges(), P.schur_ranges(), P.p)
    np.savez_compressed(os.path.join(HERE, "cfg4_apply_fp.npz"), **fp)
    r = P.gmres(y, 100, 100, 1e-8)
    s["gmres_first_cycle"] = dict(restart=100, max_iters=100, rel_tol=1e-8,
                                  iterations=r["iterations"], converged=r["converged"],
                                  seconds=r["seconds"], history=r["history"].tolist())
    old = os.path.join(HERE, "cfg4.json")
    base = json.load(open(old)) if os.path.exists(old) else {}
    base.update({k: v for k, v in s.items() if k not in base or k in (
        "stored_nnz", "gmres_first_cycle", "apply_seconds_ref", "ilut_seconds_ref_threads",
        "threads", "generate_partition_msc_seconds_ref")})
    with open(old, "w") as f:
        json.dump(base, f, indent=1)


def cfg5_apply():
    """BASELINE cfg5: apply fingerprint."""
    P, s = _large_precond(2048, 0.01, 4096, "lum", 256, 1, anchored=True)
    y = refpy.random_vector(P.n, 0)
    t = time.time()
    x = P.apply(y)
    s["apply_seconds_ref"] = time.time() - t
    fp = apply_fingerprint(x, P.d_ranges(), P.schur_ranges(), P.p)
    np.savez_compressed(os.path.join(HERE, "cfg5_apply_fp.npz"), **fp)
    old = os.path.join(HERE, "cfg5.json")
    base = json.load(open(old)) if os.path.exists(old) else {}
    for k in ("stored_nnz", "apply_seconds_ref", "ilut_seconds_ref_threads", "threads",
              "generate_partition_msc_seconds_ref"):
        base[k] = s[k]
    with open(old, "w") as f:
        json.dump(base, f, indent=1)


def cfg_large(grid_n, nu, n_a, name):
    """Setup-only digests at cfg4/cfg5 (anchored LUM, sz 256)."""
    t = time.time()
    P = refpy.Problem.oseen(grid_n, nu, n_a, anchored=True)
    P.build_schur("lum", 256, 1)
    s = problem_summary(P, with_factors=False)
    s["setup_seconds_ref"] = time.time() - t
    s.pop("d_ranges")
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(s, f, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg2", action="store_true", help="also run the cfg2 GMRES (~3 min)")
    ap.add_argument("--large", action="store_true", help="cfg4/cfg5 setup digests (~5 min)")
    ap.add_argument("--only", choices=["cfg2gmres", "cfg3p", "cfg4", "cfg5"])
    a = ap.parse_args()
    refpy.build()
    if a.only:
        {"cfg2gmres": lambda: cfg2(True), "cfg3p": cfg3p, "cfg4": cfg4_cycle,
         "cfg5": cfg5_apply}[a.only]()
        print("written", a.only)
        sys.exit(0)
    cfg1()
    random_saddles()
    ilut_contracts()
    cfg3_error()
    cfg2(a.cfg2)
    if a.large:
        cfg_large(1024, 0.001, 1024, "cfg4")
        cfg_large(2048, 0.01, 4096, "cfg5")
    print("golden fixtures written to", HERE)
