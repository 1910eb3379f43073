# K1 counting read with per-thread run aggregation: K1 tests, k12_scale (serving / random), ncu per kernel
set -u
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "group_sort or run_compact" --timeout 300 > gpurun_out/r2n8_k1_tests.log 2>&1; echo "k1 tests rc=$?" >> gpurun_out/r2n8_rc.txt
for rep in 1 2; do for d in serving random; do
  timeout 150 python tools/k12_scale.py gpurun_out/r2n8_k12_${d}_$rep.json $d > /dev/null 2>&1; echo "k12 $d rc=$?" >> gpurun_out/r2n8_rc.txt
done; done
for d in serving random; do
  timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2n8_k1_$d.csv python tools/k1_once.py 16777216 $d > /dev/null 2>&1; echo "ncu $d rc=$?" >> gpurun_out/r2n8_rc.txt
done
timeout 400 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "c2_three or c3_budgeted" --timeout 300 > gpurun_out/r2n8_serving.log 2>&1; echo "serving rc=$?" >> gpurun_out/r2n8_rc.txt
cat gpurun_out/r2n8_rc.txt; tail -2 gpurun_out/r2n8_k1_tests.log
