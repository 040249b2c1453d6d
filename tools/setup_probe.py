"""Build the preconditioner of one bench config and print the setup times
(for ncu captures of the factorisation kernels).

    python tools/setup_probe.py --config cfg4
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    a = ap.parse_args()
    import bench
    import paper_1104_3349_b200 as msc
    cfg = bench.CONFIGS[a.config]
    ctx = msc.Context(0)
    pb, t = bench.build_problem(cfg, ctx=ctx)
    t0 = time.perf_counter()
    pc = msc.build_preconditioner(pb, tolA=bench.TOL_A, sA=bench.S_A, ctx=ctx)
    t["build_preconditioner_s"] = time.perf_counter() - t0
    t.update(pc.build_times())
    print(a.config, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in t.items()})


if __name__ == "__main__":
    main()
