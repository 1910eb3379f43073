set -u
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_parity_full.py::test_c5_pooled_budget_swaps_across_shapes -m gpu -q -x > gpurun_out/r2m2_c5pool_$i.log 2>&1; echo "c5 pooled rep $i rc=$?" >> gpurun_out/r2m2_rc.txt; done
timeout 1800 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2m2_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2m2_rc.txt
timeout 1500 python bench.py --config c5 --alloc-count 201 --steps 3 --no-cpu-baseline > gpurun_out/r2m2_bench_c5.log 2>&1; echo "bench c5 rc=$?" >> gpurun_out/r2m2_rc.txt
cat gpurun_out/r2m2_rc.txt
