# A/B of two in-tree builds (MSCG_LIB): A = paper_1104_3349_b200/libmscg_a.so, B = ${LIBB:-libmscg_b.so}
set -u
mkdir -p gpurun_out
run() {
  c=$1; which=$2; rep=$3
  lib=$PWD/paper_1104_3349_b200/${LIBB:-libmscg_b.so}
  [ $which = A ] && lib=$PWD/paper_1104_3349_b200/libmscg_a.so
  MSCG_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-gmres > gpurun_out/ab_${c}_${which}$rep.json 2> gpurun_out/ab_${c}_${which}$rep.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_${c}_${which}$rep.json').read().strip().splitlines()[-1]); print('$c $which', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3), 'corr_off_dsolve', round(d['apply_correction_off']['d_solve_ms'],3), d['clocks']['reasons'])" || tail -3 gpurun_out/ab_${c}_${which}$rep.err
}
for rep in 1 2; do
  for c in ${CONFIGS:-cfg5 cfg4 cfg2}; do
    run $c A $rep; run $c B $rep
  done
done
if [ -n "${TRACE:-}" ]; then
  MSCG_LIB=$PWD/paper_1104_3349_b200/${LIBB:-libmscg_b.so} timeout 600 python tools/trace_dsolve.py --config cfg5 --out gpurun_out/trace_cfg5_B.npz > gpurun_out/trace_B.log 2>&1
  python tools/trace_tiles.py gpurun_out/trace_cfg5_B.npz
fi
[ -n "${NOTEST:-}" ] || MSCG_LIB=$PWD/paper_1104_3349_b200/${LIBB:-libmscg_b.so} timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
