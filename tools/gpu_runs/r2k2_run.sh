set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2k2_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2k2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 900 python bench.py > gpurun_out/r2k2_bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2k2_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2k2_bench_c2.log 2>&1; echo "bench c2 rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2k2_bench_c4.log 2>&1; echo "bench c4 rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 1500 python bench.py --config c5 --alloc-count 201 --steps 3 > gpurun_out/r2k2_bench_c5.log 2>&1; echo "bench c5 rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2k2_bench_ref.log 2>&1; echo "bench ref rc=$?" >> gpurun_out/r2k2_rc.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 40 --log-file gpurun_out/san_memcheck_r2k2.log python tools/sanitize_cases.py smoke swaps e2e hops > gpurun_out/san_memcheck_r2k2.out 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2k2_rc.txt
cat gpurun_out/r2k2_rc.txt
