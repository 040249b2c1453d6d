# one vs two solver warps per block (MSCG_TRI_SOLVERS)
set -u
mkdir -p gpurun_out
MSCG_TRI_SOLVERS=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
for c in ${CONFIGS:-cfg2 cfg3 cfg5 cfg4}; do
  for sv in 1 2; do
    MSCG_TRI_SOLVERS=$sv timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-gmres > gpurun_out/sv_${c}_$sv.json 2> gpurun_out/sv_${c}_$sv.err
    python -c "
import json; d=json.loads(open('gpurun_out/sv_${c}_$sv.json').read().strip().splitlines()[-1]); print('$c solvers $sv', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['reasons'])" || tail -3 gpurun_out/sv_${c}_$sv.err
  done
done
done
for sv in 1 2; do MSCG_TRI_SOLVERS=$sv timeout 600 python bench.py --config cfg2 --mode gmres 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gmres cfg2 solvers $sv', d['iterations'], round(d['solve_s'],4))"; done
