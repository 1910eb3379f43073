set -u
mkdir -p gpurun_out
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/r2j2_gputest_$i.log 2>&1; echo "gpu tests $i rc=$?" >> gpurun_out/r2j2_rc.txt
done
cat gpurun_out/r2j2_rc.txt
