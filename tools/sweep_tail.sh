for T in 1 2 4 8 16; do
  for c in cfg2 cfg4; do
    MSCG_TRI_TAIL=$T timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_${c}_T$T.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/sweep_${c}_T$T.json').read().strip().splitlines()[-1]); print('$c T=$T', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'GB/s', round(d['roofline']['achieved'],1))"
  done
done
