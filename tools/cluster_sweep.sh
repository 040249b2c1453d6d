# cluster sizes at cfg2/cfg3 (D-solve ms) + GMRES cfg2 at the default size
for cl in ${CLS:-8 6 4 -1}; do
  for c in cfg2 cfg3; do
    MSCG_TRI_CLUSTER=$cl timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/cs_$c.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/cs_$c.json').read().strip().splitlines()[-1]); print('cl=$cl $c dsolve_ms', round(d['stage_ms']['d_solve'],4), 'apply', round(d['apply_ms'],4))" 2>/dev/null || echo "cl=$cl $c failed"
  done
done
timeout 300 python bench.py --config cfg2 --mode gmres > gpurun_out/cs_gmres.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/cs_gmres.json').read().strip().splitlines()[-1]); print('gmres cfg2 its', d['iterations'], 'solve_s %.3f'%d['solve_s'])"
