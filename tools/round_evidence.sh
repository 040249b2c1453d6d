# Round-end evidence on one GPU: parity tests, default bench line (cfg5 with
# cpu_baseline), cfg4 bench line, GMRES time-to-solution at cfg1/cfg2/cfg4.
# usage: TAG=v17 bash tools/round_evidence.sh   (outputs in gpurun_out/)
set -u
T=${TAG:-ev}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg5.json 2> gpurun_out/${T}_bench_cfg5.err; tail -c 400 gpurun_out/${T}_bench_cfg5.json
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_cfg4.json 2>/dev/null
for c in cfg1 cfg2 cfg4; do
  timeout 900 python bench.py --config $c --mode gmres > gpurun_out/${T}_gmres_$c.json 2>/dev/null
done
echo done
