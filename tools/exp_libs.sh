# A/B/C... of in-tree builds: LIBS="a b c" -> paper_1104_3349_b200/libmscg_<x>.so
set -u
mkdir -p gpurun_out
run() {
  c=$1; which=$2; rep=$3
  lib=$PWD/paper_1104_3349_b200/libmscg_$which.so
  MSCG_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-gmres > gpurun_out/ab_${c}_${which}$rep.json 2> gpurun_out/ab_${c}_${which}$rep.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_${c}_${which}$rep.json').read().strip().splitlines()[-1]); print('$c $which', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3), 'corr_off_dsolve', round(d['apply_correction_off']['d_solve_ms'],3), d['clocks']['reasons'])" || tail -3 gpurun_out/ab_${c}_${which}$rep.err
}
for rep in 1 2; do
  for c in ${CONFIGS:-cfg5 cfg4 cfg2}; do
    for l in ${LIBS:-a b}; do run $c $l $rep; done
  done
done
for l in ${TESTLIBS:-}; do
  MSCG_LIB=$PWD/paper_1104_3349_b200/libmscg_$l.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
done
