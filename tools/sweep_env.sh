# usage: VAR=NAME VALUES="a b c" CONFIGS="cfg2 cfg4" bash tools/sweep_env.sh
for V in $VALUES; do
  for c in ${CONFIGS:-cfg2 cfg4}; do
    env $VAR=$V timeout 300 python bench.py --config $c --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline > gpurun_out/sw_${c}_$V.json 2>gpurun_out/sw_${c}_$V.err
    python -c "
import json; d=json.loads(open('gpurun_out/sw_${c}_$V.json').read().strip().splitlines()[-1]); print('$c $VAR=$V', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'GB/s', round(d['roofline']['achieved'],1))" || tail -3 gpurun_out/sw_${c}_$V.err
  done
done
