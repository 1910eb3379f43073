set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "peer_tier or c5 or multi_executor" > gpurun_out/r2s_peer_tests.log 2>&1; echo "peer tests rc=$?" >> gpurun_out/r2s_rc.txt
COE_INPUT_BULK=1 timeout 900 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "e2e" > gpurun_out/r2s_e2e_bulk.log 2>&1; echo "e2e tests bulk rc=$?" >> gpurun_out/r2s_rc.txt
for v in "X=0" "COE_INPUT_BULK=1" "COE_INPUT_QUEUE=1" "COE_INPUT_BULK=1 COE_INPUT_QUEUE=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2s_tl_c1_$tag.json e2e > gpurun_out/r2s_tl_c1_$tag.log 2>&1
  env $v timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2s_tl_c3_$tag.json e2e > gpurun_out/r2s_tl_c3_$tag.log 2>&1
  echo "$v done" >> gpurun_out/r2s_rc.txt
done
for f in 4096 40000; do
  COE_FUSED_MAX=$f timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2s_tl_c3_fused$f.json > gpurun_out/r2s_tl_c3_fused$f.log 2>&1
  COE_FUSED_MAX=$f timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2s_tl_c1_fused$f.json > gpurun_out/r2s_tl_c1_fused$f.log 2>&1
done
echo "fused done" >> gpurun_out/r2s_rc.txt
COE_MAX_WAVE_ROWS=8192 timeout 900 python bench.py --alloc-count 17 --no-cpu-baseline > gpurun_out/r2s_bench_c3_dev12gb.log 2>&1; echo "dev12gb rc=$?" >> gpurun_out/r2s_rc.txt
ALLOC_COUNT=201 timeout 2400 python tools/rate_sweep.py c5 10000 gpurun_out/r2s_rate_sweep_c5_10000.json > gpurun_out/r2s_rate_sweep_c5.log 2>&1; echo "sweep rc=$?" >> gpurun_out/r2s_rc.txt
cat gpurun_out/r2s_rc.txt
