#!/bin/bash
# A/B of the runtime's main-stream count and K3 CTA grouping on the K3-bound configs
# (run on the GPU box; timeline summaries land in gpurun_out/ab_<cfg>_<tag>.log).
run() { tag=$1; shift; env "$@" timeout 300 python tools/timeline.py $CFG 10000 gpurun_out/tmp.json > gpurun_out/ab_${CFG}_$tag.log 2>&1; }
for CFG in c2 c1 c3; do
  run s1 COE_MAIN_STREAMS=1
  run s2 COE_MAIN_STREAMS=2
  run s2_cg1 COE_MAIN_STREAMS=2 COE_K3_CG=1
done
