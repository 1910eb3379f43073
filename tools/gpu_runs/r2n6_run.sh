# K1 experiment: the sorted tile staged as (key, value) pairs (COE_K1_PACK=1) -- K1 tests, then
# k12_scale A/B on serving-like and random keys, two repetitions
set -u
mkdir -p gpurun_out
COE_K1_PACK=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "group_sort or run_compact" --timeout 300 > gpurun_out/r2n6_k1_tests.log 2>&1; echo "k1 tests pack rc=$?" >> gpurun_out/r2n6_rc.txt
for rep in 1 2; do for d in serving random; do
  COE_K1_PACK=1 timeout 600 python tools/k12_scale.py gpurun_out/r2n6_pack_${d}_$rep.json $d > /dev/null 2>&1; echo "pack $d rc=$?" >> gpurun_out/r2n6_rc.txt
  timeout 600 python tools/k12_scale.py gpurun_out/r2n6_base_${d}_$rep.json $d > /dev/null 2>&1; echo "base $d rc=$?" >> gpurun_out/r2n6_rc.txt
done; done
cat gpurun_out/r2n6_rc.txt; tail -2 gpurun_out/r2n6_k1_tests.log
