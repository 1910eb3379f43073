set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2i_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/r2i_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2i_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2i_rc.txt
timeout 900 python bench.py > gpurun_out/r2i_bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2i_rc.txt
bash tools/sanitize.sh > gpurun_out/r2i_san.log 2>&1; echo "san rc=$?" >> gpurun_out/r2i_rc.txt
cat gpurun_out/r2i_rc.txt
