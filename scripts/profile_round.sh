#!/bin/bash
# Round profile on one B200: plain bench line, launch list (gpu__time_duration per launch)
# of a short bench run, and one --set full capture of each pipeline kernel at the bench's
# chunk size.  Outputs under gpurun_out/.  Usage: scripts/profile_round.sh TAG
set -e
TAG=${1:-r01}
cd "$(dirname "$0")/.."
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
cat gpurun_out/bench_${TAG}.json
CMD="python bench.py --steps 2 --warmup 1 --slices 128 --no-cpu-baseline --e2e-slices 16 --e2e-steps 1"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
CMD2="python scripts/time_stages.py --n 2048 --batch 32 --reps 1"
$CMD2 > gpurun_out/plain2_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_ramp|k_row_rdft|k_rho_conv|k_irdft_readout" -s 4 -c 4 -o gpurun_out/full_${TAG} $CMD2 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
