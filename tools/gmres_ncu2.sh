# ncu launch lists of GMRES at cfg4 (150 iterations) for each orthogonalisation
set -u
T=${TAG:-gn}
mkdir -p gpurun_out
for o in ${ORTHS:-dcgs2 cgs2}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/${T}_launches_cfg4_$o.csv python bench.py --config cfg4 --mode gmres --max-iters 150 --orth $o > gpurun_out/${T}_ncu_$o.log 2>&1
  echo "$o rc=$?"
done
