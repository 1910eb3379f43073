set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2u_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2u_rc.txt
for v in "X=0" "COE_INPUT_GATHER=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2u_tl_c1_$tag.json e2e > gpurun_out/r2u_tl_c1_$tag.log 2>&1
  env $v timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2u_tl_c3_$tag.json e2e > gpurun_out/r2u_tl_c3_$tag.log 2>&1
  echo "$v done" >> gpurun_out/r2u_rc.txt
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2u_bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/r2u_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2u_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2u_rc.txt
cat gpurun_out/r2u_rc.txt
