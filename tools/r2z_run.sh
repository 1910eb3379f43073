set -u
mkdir -p gpurun_out
for v in 0 20 35 50; do
  COE_INPUT_SPLIT=$v timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2z_tl_c1_split$v.json e2e > gpurun_out/r2z_tl_c1_split$v.log 2>&1
  COE_INPUT_SPLIT=$v timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2z_tl_c3_split$v.json e2e > gpurun_out/r2z_tl_c3_split$v.log 2>&1
  echo "split $v done" >> gpurun_out/r2z_rc.txt
done
COE_INPUT_SPLIT=35 timeout 600 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "end_to_end or e2e or streamed" > gpurun_out/r2z_e2e_split.log 2>&1; echo "e2e tests split rc=$?" >> gpurun_out/r2z_rc.txt
cat gpurun_out/r2z_rc.txt
