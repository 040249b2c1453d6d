# quick GPU regression: parity tests + apply bench at cfg2/cfg4 (no cpu baseline)
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in ${CONFIGS:-cfg2 cfg4}; do
  timeout 400 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/chk_$c.json 2> gpurun_out/chk_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/chk_$c.json').read().strip().splitlines()[-1]); print('$c', 'apply_ms', round(d['apply_ms'],3), 'stage', {k:round(v,3) for k,v in d['stage_ms'].items()}, 'dsolve GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3), 'setup', {k:(round(v,2) if isinstance(v,float) else v) for k,v in d['setup'].items()})" || tail -5 gpurun_out/chk_$c.err
done
