#!/bin/bash
# Round profile on one B200, one ncu per gpurun call:
#   scripts/profile_round.sh TAG launches  -> bench line (no profiler) + per-launch gpu__time_duration list
#   scripts/profile_round.sh TAG full      -> one --set full capture of each pipeline kernel (chunk 8, as bench.py)
# Each ncu pass runs only after the same command exited 0 without ncu.  Outputs under gpurun_out/.
set -e
TAG=${1:-r01}
MODE=${2:-launches}
cd "$(dirname "$0")/.."
if [ "$MODE" = launches ]; then
  python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
  cat gpurun_out/bench_${TAG}.json
  CMD="python bench.py --steps 2 --warmup 1 --slices 128 --no-cpu-baseline --e2e-slices 16 --e2e-steps 1"
  $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD \
    > gpurun_out/ncu_launches_${TAG}.log 2>&1
  tail -2 gpurun_out/ncu_launches_${TAG}.log
else
  CMD2="python scripts/time_stages.py --n 2048 --batch 8 --reps 1"
  $CMD2 > gpurun_out/plain2_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_ramp|k_row_rdft|k_rho_conv|k_irdft_readout" \
    -s 4 -c 4 -o gpurun_out/full_${TAG} $CMD2 > gpurun_out/ncu_full_${TAG}.log 2>&1
  tail -2 gpurun_out/ncu_full_${TAG}.log
fi
