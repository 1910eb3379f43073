set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2j_gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/r2j_rc.txt
timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2j_tl_c3_e2e.json e2e > gpurun_out/r2j_tl_c3_e2e.log 2>&1; echo "tl c3 e2e rc=$?" >> gpurun_out/r2j_rc.txt
ALLOC_COUNT=201 timeout 900 python tools/timeline.py c5 10000 gpurun_out/r2j_tl_c5.json > gpurun_out/r2j_tl_c5.log 2>&1; echo "tl c5 rc=$?" >> gpurun_out/r2j_rc.txt
ALLOC_COUNT=201 timeout 900 python tools/host_times.py c5 10000 > gpurun_out/r2j_host_c5.log 2>&1; echo "host c5 rc=$?" >> gpurun_out/r2j_rc.txt
timeout 600 python tools/host_times.py c3 10000 1 > gpurun_out/r2j_host_c3e2e.log 2>&1; echo "host c3 rc=$?" >> gpurun_out/r2j_rc.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 40 --log-file gpurun_out/san_racecheck_smoke.log python tools/sanitize_cases.py smoke > gpurun_out/san_racecheck_smoke.out 2>&1; echo "racecheck smoke rc=$?" >> gpurun_out/r2j_rc.txt
cat gpurun_out/r2j_rc.txt
