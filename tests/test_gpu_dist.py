"""GPU: the sharded preconditioner and the distributed GMRES driven across
two processes (torchrun, gloo on CUDA tensors, both ranks on the one GPU this
sandbox has — functional, never a timing).  Each rank calls
mscg_precond_apply_shard / mscg_precond_spmv_shard / mscg_gmres_shard on its
own shard; the results are checked against the single-GPU preconditioner."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("grid,nu,n_a", [(32, 0.1, 8), (64, 0.01, 16)])
def test_two_rank_shard_apply_spmv_gmres(grid, nu, n_a):
    env = dict(os.environ, DW_GRID=str(grid), DW_NU=str(nu), DW_NA=str(n_a))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = next(ln for ln in r.stdout.splitlines() if ln.startswith("DIST_RESULT "))
    outs = json.loads(line[len("DIST_RESULT "):])
    assert [o["rank"] for o in outs] == [0, 1]
    # the two shards tile the interior blocks
    assert outs[0]["blocks"][0] == 0 and outs[0]["blocks"][1] == outs[1]["blocks"][0]
    for o in outs:
        assert o["err_apply"] <= 1e-12, o
        assert o["err_spmv"] <= 1e-14, o
        # same iteration count as the single-GPU DCGS2 solve (+-1), both converged
        assert abs(o["its"] - o["its_single"]) <= 1, o
        assert o["converged"] and o["true_residual"] <= 1e-8, o
        assert o["hist_dev"] <= 1e-6, o
        assert o["x_rel"] <= 1e-6, o
    assert outs[0]["its"] == outs[1]["its"]
