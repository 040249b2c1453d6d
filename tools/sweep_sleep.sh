for S in 0 16 64 256; do
  for c in cfg2 cfg4; do
    MSCG_TRI_SLEEP_NS=$S timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/sl_${c}_$S.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/sl_${c}_$S.json').read().strip().splitlines()[-1]); print('$c sleep=$S', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'GB/s', round(d['roofline']['achieved'],1))"
  done
done
