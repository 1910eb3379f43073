set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/r2n_kernels.log 2>&1; echo "kernel tests rc=$?" >> gpurun_out/r2n_rc.txt
timeout 900 bash tools/k3_sweep.sh > gpurun_out/r2n_k3_sweep.log 2>&1; echo "k3 sweep rc=$?" >> gpurun_out/r2n_rc.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2n_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2n_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline --no-e2e > gpurun_out/r2n_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2n_rc.txt
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/r2n_bench_c2.log 2>&1; echo "bench c2 rc=$?" >> gpurun_out/r2n_rc.txt

for v in 64 148; do
  COE_INPUT_CTAS=$v timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2n_tl_c1_$v.json e2e > gpurun_out/r2n_tl_c1_$v.log 2>&1
  COE_INPUT_CTAS=$v timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2n_tl_c3_$v.json e2e > gpurun_out/r2n_tl_c3_$v.log 2>&1
  echo "tl $v done" >> gpurun_out/r2n_rc.txt
done
cat gpurun_out/r2n_rc.txt
