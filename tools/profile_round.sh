# Round profile for the bench workload (default cfg5):
#   1. plain bench line (must exit 0 before any ncu pass)
#   2. ncu launch list (gpu__time_duration per launch, serialised, cold cache)
#   3. ncu --set full of one interior-block trisolve launch
# usage: TAG=r01_v8 CONFIG=cfg5 bash tools/profile_round.sh
set -u
C=${CONFIG:-cfg5}; T=${TAG:-prof}
mkdir -p gpurun_out
python bench.py --config $C --steps ${STEPS:-20} --warmup 3 > gpurun_out/${T}_bench_$C.json 2> gpurun_out/${T}_bench_$C.err || { tail -5 gpurun_out/${T}_bench_$C.err; exit 1; }
tail -1 gpurun_out/${T}_bench_$C.json
python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches_$C.csv python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_list.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:trisolve -s 2 -c 1 -f \
  -o gpurun_out/${T}_trisolve_$C python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1
echo "full rc=$?"
