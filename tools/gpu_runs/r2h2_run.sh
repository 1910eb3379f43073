set -u
mkdir -p gpurun_out
COE_K3_TMA_STORE=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/r2h2_kernels_ts.log 2>&1; echo "kernel tests ts rc=$?" >> gpurun_out/r2h2_rc.txt
for rep in 1 2; do
for ts in 0 1; do
  COE_K3_TMA_STORE=$ts timeout 900 bash tools/k3_sweep.sh > gpurun_out/r2h2_sweep_ts${ts}_$rep.log 2>&1; echo "sweep ts$ts rep$rep rc=$?" >> gpurun_out/r2h2_rc.txt
done
done
COE_K3_TMA_STORE=1 timeout 600 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "c1 or c2 or c3_budgeted" > gpurun_out/r2h2_serving_ts.log 2>&1; echo "serving ts rc=$?" >> gpurun_out/r2h2_rc.txt
cat gpurun_out/r2h2_rc.txt
