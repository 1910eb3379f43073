#!/bin/bash
# One gpurun call's worth of evidence for profiles/ (run on the GPU box from the repo root):
#   bench lines (C3 default with CPU baseline, C2, C1), the ncu launch list of one bench
#   step, one `ncu --set full` capture of K3 (C3 shape, the bench's isolated wave) and of the
#   K1/K2 grouping kernels.  Summarise here with: python tools/summarize_profiles.py <tag>
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c3.log 2>&1
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.log 2>&1
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/${TAG}_bench_c1.log 2>&1
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
COE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"group|radix|onesweep|compact|batch" -c 4 -f \
  -o gpurun_out/k12_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks \
  > gpurun_out/${TAG}_ncu_k12.log 2>&1
tail -c 400 gpurun_out/${TAG}_bench_c3.log
