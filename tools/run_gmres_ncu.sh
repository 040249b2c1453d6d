mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
  --log-file gpurun_out/gm_launches_cfg4.csv python bench.py --config cfg4 --mode gmres --max-iters 150 > gpurun_out/gm_ncu.log 2>&1
echo rc=$?
