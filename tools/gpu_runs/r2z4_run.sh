# Final code after the K1 counting-read change: GPU suite, smoke, default bench (C3), C1 bench,
# warm-step K1/K2 ncu
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2z4_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2z4_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2z4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2z4_rc.txt
timeout 900 python bench.py > gpurun_out/r2z4_bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/r2z4_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2z4_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2z4_rc.txt
COE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"group_compact|radix|onesweep|compact_batches|batch_block|scan_block" -c 4 -f \
  -o gpurun_out/k12_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/r2z4_ncu_k12.log 2>&1; echo "ncu k12 rc=$?" >> gpurun_out/r2z4_rc.txt
cat gpurun_out/r2z4_rc.txt; tail -2 gpurun_out/r2z4_gputest.log
