# Round-end evidence at HEAD: full GPU suite, smoke, the driver's bench
# command, GMRES time-to-solution lines, ncu launch lists of GMRES (cfg2
# clusters, cfg4 DCGS2) and one full capture of the cluster trisolve at cfg2
set -u
T=${TAG:-fe}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_cfg5.json 2> gpurun_out/${T}_bench_cfg5.err; echo "bench rc=$?"
for c in cfg1 cfg2 cfg4; do
  timeout 600 python bench.py --config $c --mode gmres > gpurun_out/${T}_gmres_$c.json 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/${T}_launches_gmres_cfg4.csv python bench.py --config cfg4 --mode gmres --max-iters 150 > gpurun_out/${T}_ncu_g4.log 2>&1; echo "ncu g4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches_gmres_cfg2.csv python bench.py --config cfg2 --mode gmres --max-iters 100 > gpurun_out/${T}_ncu_g2.log 2>&1; echo "ncu g2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:trisolve_kernel -s 40 -c 1 -f -o gpurun_out/${T}_trisolve_cluster_cfg2 python bench.py --config cfg2 --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/${T}_ncu_full_cfg2.log 2>&1; echo "ncu full cfg2 rc=$?"
