set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/r2o_kernels_cw1.log 2>&1; echo "kernel tests cw1 rc=$?" >> gpurun_out/r2o_rc.txt
COE_K3_COORD=0 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/r2o_kernels_cw0.log 2>&1; echo "kernel tests cw0 rc=$?" >> gpurun_out/r2o_rc.txt
for rep in 1 2; do
for cw in 0 1; do
  COE_K3_COORD=$cw timeout 900 bash tools/k3_sweep.sh > gpurun_out/r2o_k3_sweep_cw${cw}_$rep.log 2>&1; echo "sweep cw$cw rep$rep rc=$?" >> gpurun_out/r2o_rc.txt
done
done
cat gpurun_out/r2o_rc.txt
