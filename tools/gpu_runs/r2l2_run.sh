set -u
mkdir -p gpurun_out
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2l2_gputest_$i.log 2>&1; echo "gpu tests $i rc=$?" >> gpurun_out/r2l2_rc.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2l2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2l2_rc.txt
timeout 900 python bench.py > gpurun_out/r2l2_bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/r2l2_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2l2_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2l2_rc.txt
cat gpurun_out/r2l2_rc.txt
