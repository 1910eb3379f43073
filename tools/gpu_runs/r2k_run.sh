set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_serving.py -m gpu -q -k "e2e" > gpurun_out/r2k_gpu_e2e.log 2>&1; echo "e2e tests rc=$?" >> gpurun_out/r2k_rc.txt
timeout 600 python tools/host_times.py c3 10000 1 > gpurun_out/r2k_host_c3e2e.log 2>&1; echo "host c3 rc=$?" >> gpurun_out/r2k_rc.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2k_bench_c3_gather.log 2>&1; echo "bench c3 gather rc=$?" >> gpurun_out/r2k_rc.txt
COE_INPUT_DMA=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2k_bench_c3_dma.log 2>&1; echo "bench c3 dma rc=$?" >> gpurun_out/r2k_rc.txt
timeout 900 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2k_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2k_rc.txt
timeout 1500 python bench.py --config c5 --alloc-count 201 --steps 3 --warmup 3 > gpurun_out/r2k_bench_c5.log 2>&1; echo "bench c5 rc=$?" >> gpurun_out/r2k_rc.txt
cat gpurun_out/r2k_rc.txt
