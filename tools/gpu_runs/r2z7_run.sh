# Final code: ncu launch list of ONE warm bench step (C3) and the K1/K2 --set full capture
set -u
mkdir -p gpurun_out
COE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks \
  > gpurun_out/r2z7_ncu_launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/r2z7_rc.txt
COE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"group_compact|radix|onesweep|compact_batches|batch_block|scan_block|compact_gather" -c 6 -f \
  -o gpurun_out/k12_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/r2z7_ncu_k12.log 2>&1; echo "ncu k12 rc=$?" >> gpurun_out/r2z7_rc.txt
cat gpurun_out/r2z7_rc.txt
