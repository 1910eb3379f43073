# Final-code sanitizers: memcheck + synccheck over smoke / swaps / e2e / hops, racecheck over smoke,
# memcheck over the two-process IPC hop test
set -u
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 40 --log-file gpurun_out/r2z3_san_${tool}.log \
    python tools/sanitize_cases.py smoke swaps e2e hops > gpurun_out/r2z3_san_${tool}.out 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2z3_rc.txt
done
timeout 1200 compute-sanitizer --tool racecheck --print-limit 40 --log-file gpurun_out/r2z3_san_racecheck.log \
  python tools/sanitize_cases.py smoke > gpurun_out/r2z3_san_racecheck.out 2>&1
echo "racecheck rc=$?" >> gpurun_out/r2z3_rc.txt
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 40 \
  --log-file gpurun_out/r2z3_san_memcheck_ipc.%p.log \
  python -m pytest tests/test_gpu_serving.py -q -m gpu -k fused_hops_across_processes_ipc > gpurun_out/r2z3_san_ipc.out 2>&1
echo "memcheck_ipc rc=$?" >> gpurun_out/r2z3_rc.txt
cat gpurun_out/r2z3_rc.txt
for f in gpurun_out/r2z3_san_*; do echo "== $f"; tail -4 "$f"; done
