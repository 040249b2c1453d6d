# helper-warp cluster solve: parity subset, then D-solve / GMRES with and without it
timeout 400 python -m pytest tests -m gpu -x -q -k "cfg2 or overlapped or cfg3p or factor_exact_and_solve or gmres_cfg1 or dist" > gpurun_out/hc_pytest.log 2>&1; tail -3 gpurun_out/hc_pytest.log
for h in 1 0; do
  for c in cfg2 cfg3; do
    MSCG_TRI_HELPER=$h timeout 200 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/hc_$c.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/hc_$c.json').read().strip().splitlines()[-1]); print('helper=$h $c dsolve_ms', round(d['stage_ms']['d_solve'],4), 'apply', round(d['apply_ms'],4))" 2>/dev/null || echo "helper=$h $c failed"
  done
  MSCG_TRI_HELPER=$h timeout 200 python bench.py --config cfg2 --mode gmres > gpurun_out/hc_gmres.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/hc_gmres.json').read().strip().splitlines()[-1]); print('helper=$h gmres cfg2 its', d['iterations'], 'solve_s %.3f'%d['solve_s'])" 2>/dev/null || echo "gmres failed"
done
