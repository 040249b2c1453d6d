# pack policy sweep: pieces per long row (L,U) and ordering slack (L,U)
set -u
mkdir -p gpurun_out
run() {
  c=$1; pl=$2; pu=$3; sl=$4; su=$5
  tag=${c}_${pl}${pu}_${sl}_${su}
  MSCG_PACK_PIECES_L=$pl MSCG_PACK_PIECES_U=$pu MSCG_PACK_SLACK_L=$sl MSCG_PACK_SLACK_U=$su timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-gmres > gpurun_out/pk_$tag.json 2> gpurun_out/pk_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/pk_$tag.json').read().strip().splitlines()[-1]); print('$c pieces $pl $pu slack $sl $su', 'apply_ms', round(d['apply_ms'],3), 'dsolve', round(d['stage_ms']['d_solve'],3), 'frac', round(d['roofline']['frac'],3), 'corr_off_dsolve', round(d['apply_correction_off']['d_solve_ms'],3), d['clocks']['reasons'])" || tail -3 gpurun_out/pk_$tag.err
}
for v in "1 1 0 0" "1 1 0 4" "1 1 0 8" "1 1 0 16" "3 1 0 0" "3 1 0 8" "4 1 0 8" "2 1 0 8" "3 1 8 8" "4 4 0 8" "1 1 0 0"; do
  run cfg5 $v
done
for v in "1 1 0 0" "1 1 0 8" "3 1 0 8" "4 4 0 8"; do
  run cfg4 $v
done
MSCG_PACK_PIECES_L=3 MSCG_PACK_SLACK_U=8 timeout 600 python tools/trace_dsolve.py --config cfg5 --out gpurun_out/trace_cfg5_pk.npz > gpurun_out/trace_pk.log 2>&1
python tools/trace_tiles.py gpurun_out/trace_cfg5_pk.npz
MSCG_PACK_PIECES_L=4 MSCG_PACK_PIECES_U=4 MSCG_PACK_SLACK_U=8 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
