set -u
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "streamed or back_to_back" --timeout 240 -p no:cacheprovider > gpurun_out/r2i2_e2e_$i.log 2>&1; echo "e2e run $i rc=$?" >> gpurun_out/r2i2_rc.txt
done
COE_INPUT_QUEUE=0 timeout 900 python -m pytest tests/test_gpu_serving.py -m gpu -q -x -k "streamed or back_to_back" --timeout 240 > gpurun_out/r2i2_e2e_q0.log 2>&1; echo "e2e queue0 rc=$?" >> gpurun_out/r2i2_rc.txt
cat gpurun_out/r2i2_rc.txt
