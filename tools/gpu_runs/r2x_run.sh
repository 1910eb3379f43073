set -u
mkdir -p gpurun_out
T=tests/test_gpu_parity_full.py::test_c5_pooled_budget_swaps_across_shapes
for v in "X=0" "COE_K3_COORD=0" "COE_POOL_PLAIN_FIT=1" "COE_KEEP_UNTOUCHED=1" "COE_K3_COORD=0 COE_POOL_PLAIN_FIT=1 COE_KEEP_UNTOUCHED=1"; do
  env $v timeout 600 python -m pytest $T -m gpu -q -x > gpurun_out/r2x_$(echo $v | tr ' =' '__').log 2>&1
  echo "$v rc=$?" >> gpurun_out/r2x_rc.txt
done
cat gpurun_out/r2x_rc.txt
