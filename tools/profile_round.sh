#!/bin/bash
# One gpurun call's worth of evidence for profiles/ (run on the GPU box from the repo root):
#   bench lines (C3 default with CPU baseline, C2, C1, C4, C5 under a 120 GB pool, the C3
#   "whole device 12 GB" variant), the reference arm, the ncu launch list of one WARM bench
#   step, `ncu --set full` captures of K3 (isolated waves per config shape) and of the fused
#   K1/K2 grouping kernel, and the C5 request-rate sweep.
#   Summarise here with: python tools/summarize_profiles.py <tag>
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c3.log 2>&1
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.log 2>&1
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/${TAG}_bench_c1.log 2>&1
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.log 2>&1
timeout 1500 python bench.py --config c5 --alloc-count 201 --steps 3 > gpurun_out/${TAG}_bench_c5.log 2>&1
# experts + activations within 12 GB: 17 experts (3.4 GB) + the 3,633-slot ring (7.6 GB) + H at 8,192-row waves
COE_MAX_WAVE_ROWS=8192 timeout 900 python bench.py --alloc-count 17 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3_dev12gb.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
# launch list of ONE warm step (3 untimed warm-ups outside the profiled range)
COE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks \
  > gpurun_out/${TAG}_ncu_launches.log 2>&1
# K3: the bench's isolated wave for each config's expert shape (groups x max batch), C3 / C2 / C1
for w in "16 6 4096 12288 256" "11 22 2048 8192 128" "11 44 1024 4096 64"; do
  set -- $w
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -c 2 -f \
    -o gpurun_out/k3_full_$1_$2_$3x$4x$5 python tools/k3_profile.py $1 $2 1 $3 $4 $5 \
    > gpurun_out/${TAG}_ncu_k3_$3.log 2>&1
done
COE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"group_compact|radix|onesweep|compact_batches|batch_block|scan_block" -c 4 -f \
  -o gpurun_out/k12_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks \
  > gpurun_out/${TAG}_ncu_k12.log 2>&1
ALLOC_COUNT=201 timeout 1800 python tools/rate_sweep.py c5 10000 gpurun_out/${TAG}_rate_sweep_c5_10000.json > gpurun_out/${TAG}_rate_sweep_c5.log 2>&1
tail -c 400 gpurun_out/${TAG}_bench_c3.log
