# e2e staged inputs (device mirror of the host rows filled by host-order DMAs): e2e tests on both
# input paths, then C1 / C2 bench A/B on one box, C3 (gather path, > 8 GB of inputs) as a check
set -u
mkdir -p gpurun_out
K="end_to_end or ring_reuse"
timeout 900 python -m pytest tests/test_gpu_serving.py tests/test_gpu_parity_full.py -m gpu -q -x -k "$K" --timeout 400 > gpurun_out/r2n5_e2e_tests.log 2>&1; echo "e2e tests staged rc=$?" >> gpurun_out/r2n5_rc.txt
COE_INPUT_STAGE_GB=0 timeout 900 python -m pytest tests/test_gpu_serving.py tests/test_gpu_parity_full.py -m gpu -q -x -k "$K" --timeout 400 > gpurun_out/r2n5_e2e_tests_gather.log 2>&1; echo "e2e tests gather rc=$?" >> gpurun_out/r2n5_rc.txt
for rep in 1 2; do
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2n5_bench_c1_staged_$rep.log 2>&1; echo "c1 staged rc=$?" >> gpurun_out/r2n5_rc.txt
COE_INPUT_STAGE_GB=0 timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2n5_bench_c1_gather_$rep.log 2>&1; echo "c1 gather rc=$?" >> gpurun_out/r2n5_rc.txt
done
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2n5_bench_c2_staged.log 2>&1; echo "c2 staged rc=$?" >> gpurun_out/r2n5_rc.txt
COE_INPUT_STAGE_GB=0 timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2n5_bench_c2_gather.log 2>&1; echo "c2 gather rc=$?" >> gpurun_out/r2n5_rc.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2n5_bench_c3.log 2>&1; echo "c3 rc=$?" >> gpurun_out/r2n5_rc.txt
cat gpurun_out/r2n5_rc.txt
for f in gpurun_out/r2n5_bench_*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["e2e"]["ms_per_step"],2), d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"; done
