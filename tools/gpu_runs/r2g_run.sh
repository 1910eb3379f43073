set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2g_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2g_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2g_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2g_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2g_rc.txt
timeout 900 python bench.py > gpurun_out/r2g_bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/r2g_rc.txt
cat gpurun_out/r2g_rc.txt
