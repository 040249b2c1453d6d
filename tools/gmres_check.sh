# GMRES parity + time-to-solution check on one GPU (DCGS2 vs CGS2).
# usage: TAG=r02_v2 bash tools/gmres_check.sh
set -u
T=${TAG:-gc}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gmres or cfg2 or cfg3p or smoke" > gpurun_out/${T}_pytest_gmres.log 2>&1; tail -3 gpurun_out/${T}_pytest_gmres.log
for o in ${ORTHS:-dcgs2 cgs2}; do
  for c in ${CONFIGS:-cfg2 cfg4}; do
    timeout 900 python bench.py --config $c --mode gmres --orth $o > gpurun_out/${T}_gmres_${c}_${o}.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/${T}_gmres_${c}_${o}.json').read().strip().splitlines()[-1]); print('$c $o its', d['iterations'], 'conv', d['converged'], 'true', '%.3e'%d['final_true_residual'], 'solve_s %.3f'%d['solve_s'], 'ms/it %.3f'%d['ms_per_iteration'], 'clk', d['clocks'])"
  done
done
