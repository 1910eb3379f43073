# K1 wide digits: kernel tests, then k12_scale A/B (8-bit vs wide) on serving-like and random keys
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "group_sort or run_compact" --timeout 300 > gpurun_out/r2n4_k1_tests.log 2>&1; echo "k1 tests rc=$?" >> gpurun_out/r2n4_rc.txt
for d in serving random; do
  timeout 600 python tools/k12_scale.py gpurun_out/r2n4_k12_wide_$d.json $d > gpurun_out/r2n4_k12_wide_$d.log 2>&1; echo "wide $d rc=$?" >> gpurun_out/r2n4_rc.txt
  COE_K1_NARROW=1 timeout 600 python tools/k12_scale.py gpurun_out/r2n4_k12_narrow_$d.json $d > gpurun_out/r2n4_k12_narrow_$d.log 2>&1; echo "narrow $d rc=$?" >> gpurun_out/r2n4_rc.txt
done
cat gpurun_out/r2n4_rc.txt; tail -3 gpurun_out/r2n4_k1_tests.log
