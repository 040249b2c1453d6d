# env sweeps of the interior solve on the default build (cfg5)
set -u
mkdir -p gpurun_out
i=0
while read -r line; do
  [ -z "$line" ] && continue
  i=$((i+1))
  env $line timeout 600 python bench.py --config ${CONFIG:-cfg5} --steps 20 --warmup 5 --no-cpu-baseline --no-gmres > gpurun_out/env_$i.json 2> gpurun_out/env_$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/env_$i.json').read().strip().splitlines()[-1]); print('$line', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/env_$i.err
done <<LIST
${SWEEP}
LIST
