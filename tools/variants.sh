# D-solve time per trisolve kernel variant (MSCG_TRI_VARIANT) at the given configs
for c in ${CONFIGS:-cfg5}; do
  for v in ${VARIANTS:-0 1 2}; do
    MSCG_TRI_VARIANT=$v timeout 400 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/var_${c}_$v.json 2> gpurun_out/var_${c}_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/var_${c}_$v.json').read().strip().splitlines()[-1]); print('$c variant $v', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/var_${c}_$v.err
  done
done
