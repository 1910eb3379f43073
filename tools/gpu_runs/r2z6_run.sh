# Final verification after the K2 batch-kernel change: GPU suite, smoke, default bench (C3)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2z6_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2z6_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2z6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2z6_rc.txt
timeout 900 python bench.py > gpurun_out/r2z6_bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/r2z6_rc.txt
cat gpurun_out/r2z6_rc.txt; tail -1 gpurun_out/r2z6_gputest.log
