# Round profile for the bench workload (default cfg5):
#   1. plain bench line (must exit 0 before any ncu pass)
#   2. ncu launch list (gpu__time_duration per launch, serialised, cold cache)
#   3. ncu --set full of one interior-block trisolve launch of an apply (the
#      correction build's column solves come first: TRI_SKIP)
#   4. ncu --set full of one correct_kernel launch
# usage: TAG=r01_v8 CONFIG=cfg5 bash tools/profile_round.sh
set -u
C=${CONFIG:-cfg5}; T=${TAG:-prof}
mkdir -p gpurun_out
if [ -z "${ONLY_FULL:-}" ]; then
python bench.py --config $C --steps ${STEPS:-20} --warmup 3 > gpurun_out/${T}_bench_$C.json 2> gpurun_out/${T}_bench_$C.err || { tail -5 gpurun_out/${T}_bench_$C.err; exit 1; }
tail -1 gpurun_out/${T}_bench_$C.json
python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-3000} --csv \
  --log-file gpurun_out/${T}_launches_$C.csv python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_list.log 2>&1
echo "launch list rc=$?"
fi
# trisolve launches before the first apply's correction = setup (the
# correction build's column solves) + that apply's D and S solves: skip those
# and the next apply's two, so the capture is a warm-up apply's D-solve
if [ -z "${TRI_SKIP:-}" ]; then
  TRI_SKIP=$(python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/${T}_launches_$C.csv')) if len(r)>10]
i=rows[0].index('Kernel Name'); names=[r[i] for r in rows[1:]]
f=next((j for j,n in enumerate(names) if 'correct_kernel' in n), None)
print(2 if f is None else sum('trisolve' in n for n in names[:f]) + 2)")
fi
echo "TRI_SKIP=$TRI_SKIP"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:trisolve -s $TRI_SKIP -c 1 -f \
  -o gpurun_out/${T}_trisolve_$C python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1
echo "full rc=$?"
[ -n "${ONLY_FULL:-}" ] || timeout 900 ncu --set full --import-source on --clock-control none -k regex:correct_kernel -s 3 -c 1 -f \
  -o gpurun_out/${T}_correct_$C python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_correct.log 2>&1
echo "correct rc=$?"
