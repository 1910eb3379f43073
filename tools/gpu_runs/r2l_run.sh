set -u
mkdir -p gpurun_out
timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2l_tl_c3_e2e.json e2e > gpurun_out/r2l_tl_c3_e2e.log 2>&1; echo "tl c3 e2e rc=$?" >> gpurun_out/r2l_rc.txt
COE_INPUT_DMA=1 timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2l_tl_c3_e2e_dma.json e2e > gpurun_out/r2l_tl_c3_e2e_dma.log 2>&1; echo "tl c3 e2e dma rc=$?" >> gpurun_out/r2l_rc.txt
timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2l_tl_c1_e2e.json e2e > gpurun_out/r2l_tl_c1_e2e.log 2>&1; echo "tl c1 e2e rc=$?" >> gpurun_out/r2l_rc.txt
timeout 600 python tools/e2e_probe.py c1 > gpurun_out/r2l_e2e_probe_c1.log 2>&1; echo "probe c1 rc=$?" >> gpurun_out/r2l_rc.txt
timeout 900 bash tools/k3_sweep.sh > gpurun_out/r2l_k3_sweep.log 2>&1; echo "k3 sweep rc=$?" >> gpurun_out/r2l_rc.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 40 --log-file gpurun_out/san_racecheck_smoke2.log python tools/sanitize_cases.py smoke > gpurun_out/san_racecheck_smoke2.out 2>&1; echo "racecheck smoke rc=$?" >> gpurun_out/r2l_rc.txt
cat gpurun_out/r2l_rc.txt
