#!/bin/bash
# compute-sanitizer over the serving path (GPU box, repo root).  Summaries -> gpurun_out/san_*.log
#   memcheck: out-of-bounds / misaligned global + shared accesses, API errors
#   racecheck: shared-memory hazards inside the kernels (K1 tiles, K3 smem ring)
#   synccheck: barrier misuse (__syncthreads / named barriers / mbarrier-free paths)
# plus memcheck over the two-process IPC hop test (cross-process peer stores + flags).
set -u
mkdir -p gpurun_out
CASES=${CASES:-"smoke swaps e2e hops"}
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 40 --log-file gpurun_out/san_${tool}.log \
    python tools/sanitize_cases.py $CASES > gpurun_out/san_${tool}.out 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_rc.txt
done
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 40 \
  --log-file gpurun_out/san_memcheck_ipc.%p.log \
  python -m pytest tests/test_gpu_serving.py -q -m gpu -k fused_hops_across_processes_ipc > gpurun_out/san_ipc.out 2>&1
echo "memcheck_ipc rc=$?" >> gpurun_out/san_rc.txt
cat gpurun_out/san_rc.txt
for f in gpurun_out/san_*.log; do echo "== $f"; tail -3 "$f"; done
