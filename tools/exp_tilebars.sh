# A/B of the U-pass readiness signalling (MSCG_TRI_TILEBARS) + solver trace at cfg5
set -u
mkdir -p gpurun_out
for tb in 0 1 0 1; do
  for c in ${CONFIGS:-cfg5 cfg4}; do
    MSCG_TRI_TILEBARS=$tb timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-gmres > gpurun_out/tb${tb}_$c.json 2> gpurun_out/tb${tb}_$c.err
    python -c "
import json; d=json.loads(open('gpurun_out/tb${tb}_$c.json').read().strip().splitlines()[-1]); print('$c tilebars $tb', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3), d['clocks'])" || tail -3 gpurun_out/tb${tb}_$c.err
  done
done
for tb in 0 1; do
  MSCG_TRI_TILEBARS=$tb timeout 600 python tools/trace_dsolve.py --config cfg5 --out gpurun_out/trace_cfg5_tb$tb.npz > gpurun_out/trace_tb$tb.log 2>&1
  python tools/trace_tiles.py gpurun_out/trace_cfg5_tb$tb.npz
  python tools/trace_workers.py gpurun_out/trace_cfg5_tb$tb.npz
done
MSCG_TRI_TILEBARS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
