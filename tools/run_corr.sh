set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in cfg2 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1_$c.json 2> gpurun_out/c1_$c.err; tail -2 gpurun_out/c1_$c.err
done
MSCG_CORRECTION=off timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1_cfg5_off.json 2> gpurun_out/c1_cfg5_off.err
timeout 600 python bench.py --config cfg2 --mode gmres > gpurun_out/c1_gmres_cfg2.json 2>gpurun_out/c1_gmres_cfg2.err
timeout 900 python bench.py --config cfg4 --mode gmres > gpurun_out/c1_gmres_cfg4.json 2>gpurun_out/c1_gmres_cfg4.err
