# K2 batch kernels with 4 batches per thread: K1/K2 tests, a serving test, k12_scale, ncu per kernel
set -u
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "group_sort or run_compact" --timeout 200 > gpurun_out/r2n10_k12_tests.log 2>&1; echo "k1k2 tests rc=$?" >> gpurun_out/r2n10_rc.txt
timeout 400 python -m pytest tests/test_gpu_serving.py tests/test_gpu_parity_full.py -m gpu -q -x -k "c2_three or c3_budgeted or c3_full_plan" --timeout 300 > gpurun_out/r2n10_serving.log 2>&1; echo "serving rc=$?" >> gpurun_out/r2n10_rc.txt
for rep in 1 2; do timeout 150 python tools/k12_scale.py gpurun_out/r2n10_k12_serving_$rep.json serving > /dev/null 2>&1; echo "k12 rc=$?" >> gpurun_out/r2n10_rc.txt; done
timeout 150 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2n10_k2_after.csv python tools/k2_once.py 16777216 > /dev/null 2>&1; echo "ncu rc=$?" >> gpurun_out/r2n10_rc.txt
cat gpurun_out/r2n10_rc.txt; tail -1 gpurun_out/r2n10_k12_tests.log; tail -1 gpurun_out/r2n10_serving.log
