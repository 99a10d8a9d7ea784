#!/bin/bash
# One-call round profile on one B200 (each ncu pass only after the same command exited 0 without ncu):
#   bench line (no profiler), launch list (gpu__time_duration), --set full of each pipeline kernel,
#   the config-4 direct backprojector line and its --set full capture.  Outputs under gpurun_out/.
TAG=${1:-r02}
cd "$(dirname "$0")/.."
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
CMD="python bench.py --steps 2 --warmup 3 --slices 128 --no-cpu-baseline --e2e-slices 16 --e2e-steps 1"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD \
    > gpurun_out/ncu_launches_${TAG}.log 2>&1
CMD2="python scripts/time_stages.py --n 2048 --batch 128 --reps 1"  # 128-slice launches: the bench chunk
$CMD2 > gpurun_out/plain2_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_ramp|k_row_rdft|k_rho_conv|k_irdft_readout" \
    -s 4 -c 4 -o gpurun_out/full_${TAG} $CMD2 > gpurun_out/ncu_full_${TAG}.log 2>&1
python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_direct_${TAG}.json 2> gpurun_out/bench_direct_${TAG}.err
CMD3="python scripts/time_naive.py 4"
$CMD3 > gpurun_out/plain3_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_direct -c 2 -o gpurun_out/full_direct_${TAG} $CMD3 \
    > gpurun_out/ncu_direct_${TAG}.log 2>&1
tail -1 gpurun_out/bench_${TAG}.json | cut -c1-400
tail -1 gpurun_out/ncu_full_${TAG}.log; tail -1 gpurun_out/ncu_direct_${TAG}.log
