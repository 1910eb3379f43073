set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2y_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2y_rc.txt
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_parity_full.py::test_c5_pooled_budget_swaps_across_shapes -m gpu -q -x > gpurun_out/r2y_c5pool_$i.log 2>&1; echo "c5 pooled rep $i rc=$?" >> gpurun_out/r2y_rc.txt; done
cat gpurun_out/r2y_rc.txt
