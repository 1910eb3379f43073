set -u
mkdir -p gpurun_out
COE_INPUT_BULK=1 timeout 900 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "e2e" > gpurun_out/r2s_e2e_bulk.log 2>&1; echo "e2e tests bulk rc=$?" >> gpurun_out/r2s_rc.txt
for v in "X=0" "COE_INPUT_BULK=1" "COE_INPUT_QUEUE=1" "COE_INPUT_BULK=1 COE_INPUT_QUEUE=1" "COE_INPUT_BULK=1 COE_INPUT_CTAS=128"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2s_tl_c1_$tag.json e2e > gpurun_out/r2s_tl_c1_$tag.log 2>&1
  env $v timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2s_tl_c3_$tag.json e2e > gpurun_out/r2s_tl_c3_$tag.log 2>&1
  echo "$v done" >> gpurun_out/r2s_rc.txt
done
cat gpurun_out/r2s_rc.txt
