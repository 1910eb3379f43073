set -u
mkdir -p gpurun_out
COE_K3_WIDE=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 120 > gpurun_out/r2n2_kernels_wide.log 2>&1; echo "kernel tests wide rc=$?" >> gpurun_out/r2n2_rc.txt
for rep in 1 2; do
for wd in 0 1; do
  COE_K3_WIDE=$wd timeout 600 bash tools/k3_sweep.sh > gpurun_out/r2n2_sweep_w${wd}_$rep.log 2>&1; echo "sweep w$wd rep$rep rc=$?" >> gpurun_out/r2n2_rc.txt
done
done
COE_K3_WIDE=1 timeout 900 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "c1 or c2 or c3_budgeted or streamed" --timeout 200 > gpurun_out/r2n2_serving_wide.log 2>&1; echo "serving wide rc=$?" >> gpurun_out/r2n2_rc.txt
cat gpurun_out/r2n2_rc.txt
