set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/r2q_kernels.log 2>&1; echo "kernel tests rc=$?" >> gpurun_out/r2q_rc.txt
timeout 900 bash tools/k3_sweep.sh > gpurun_out/r2q_k3_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/r2q_rc.txt
COE_K3_DEBUG=1 timeout 900 bash tools/k3_sweep.sh > gpurun_out/r2q_k3_sweep_nostore.log 2>&1; echo "sweep nostore rc=$?" >> gpurun_out/r2q_rc.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2q_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2q_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2q_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2q_rc.txt
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2q_bench_c2.log 2>&1; echo "bench c2 rc=$?" >> gpurun_out/r2q_rc.txt
cat gpurun_out/r2q_rc.txt
