# cluster trisolve: parity subset + cfg2 / cfg3 timings with and without clusters
set -u
T=${TAG:-cc}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cfg2 or cfg3p or overlapped or factor_exact_and_solve or apply_matches or gmres_cfg1 or ilut_contract or correction" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
for cl in ${CLS:--1 0}; do
  for c in cfg2 cfg3; do
    MSCG_TRI_CLUSTER=$cl timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/${T}_bench_${c}_cl$cl.json 2> gpurun_out/${T}_bench_${c}_cl$cl.err
    python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench_${c}_cl$cl.json').read().strip().splitlines()[-1]); print('$c cl=$cl apply_ms', round(d['apply_ms'],4), 'dsolve_ms', round(d['stage_ms']['d_solve'],4), 'value', round(d['value'],1))" || tail -3 gpurun_out/${T}_bench_${c}_cl$cl.err
  done
  MSCG_TRI_CLUSTER=$cl timeout 600 python bench.py --config cfg2 --mode gmres > gpurun_out/${T}_gmres_cfg2_cl$cl.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_gmres_cfg2_cl$cl.json').read().strip().splitlines()[-1]); print('gmres cfg2 cl=$cl its', d['iterations'], 'solve_s %.3f'%d['solve_s'], 'true %.2e'%d['final_true_residual'])"
done
