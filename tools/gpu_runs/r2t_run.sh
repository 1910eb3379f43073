set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2t_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2t_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2t_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2t_rc.txt
timeout 900 python bench.py > gpurun_out/r2t_bench_c3.log 2>&1; echo "bench c3 rc=$?" >> gpurun_out/r2t_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2t_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2t_rc.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 40 --log-file gpurun_out/san_racecheck_smoke3.log python tools/sanitize_cases.py smoke > gpurun_out/san_racecheck_smoke3.out 2>&1; echo "racecheck smoke rc=$?" >> gpurun_out/r2t_rc.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 40 --log-file gpurun_out/san_memcheck_r2t.log python tools/sanitize_cases.py smoke swaps e2e hops > gpurun_out/san_memcheck_r2t.out 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2t_rc.txt
cat gpurun_out/r2t_rc.txt
