#!/bin/bash
# Bench lines for C3 (default, with the CPU baseline), C2 and C1, plus the reference arm.
TAG=${1:-r1}
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c3.log 2>&1
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.log 2>&1
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/${TAG}_bench_c1.log 2>&1
timeout 600 python bench.py --config c3 --requests 1000 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3_1k.log 2>&1
for c in c3 c2 c1 c3_1k; do tail -1 gpurun_out/${TAG}_bench_$c.log | cut -c1-220; done
