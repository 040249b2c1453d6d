# Default bench line + reference arm on one GPU box (round evidence).
# usage: TAG=r02_v1 bash tools/box_bench.sh
set -u
T=${TAG:-bb}
mkdir -p gpurun_out
{ nproc; free -g; lscpu | grep -E "Model name|Socket|Thread|Core"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/${T}_host.txt 2>&1
cat gpurun_out/${T}_host.txt
if [ "${SKIP_OURS:-0}" = 0 ]; then s0=$(date +%s)
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$? wall=$(( $(date +%s) - s0 )) s"; tail -c 300 gpurun_out/${T}_bench.err; fi
avail=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
if [ "${SKIP_REF:-0}" = 0 ] && [ "$avail" -gt 100 ]; then
  s0=$(date +%s)
  timeout 2400 python bench.py --impl reference > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
  echo "reference rc=$? wall=$(( $(date +%s) - s0 )) s"; tail -c 600 gpurun_out/${T}_reference.json
else
  echo "reference arm skipped (MemAvailable ${avail} GB)"
fi
