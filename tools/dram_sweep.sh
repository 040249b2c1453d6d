# DRAM bytes of one trisolve launch under ncu for each value of an env knob.
# usage: VAR=MSCG_TRI_PF VALUES="0 1 2" CONFIG=cfg4 bash tools/dram_sweep.sh
C=${CONFIG:-cfg4}
python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ds_plain.json 2>&1 || { tail -3 gpurun_out/ds_plain.json; exit 1; }
for V in $VALUES; do
  env $VAR=$V timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:trisolve -s 2 -c 1 --csv python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E '"(dram|gpu__time|lts)' | awk -F'","' -v v=$V '{print "'$VAR'=" v, $(NF-2), $(NF-1), $NF}'
done
