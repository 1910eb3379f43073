run() { tag=$1; shift; env "$@" timeout 300 python tools/timeline.py $CFG 10000 gpurun_out/tmp.json > gpurun_out/ab_${CFG}_$tag.log 2>&1; }
for CFG in c2 c1; do
 for r in 1 2; do
  run s1_r$r COE_MAIN_STREAMS=1
  run s2_r$r COE_MAIN_STREAMS=2
  run s2d_r$r COE_MAIN_STREAMS=2 COE_K3_DYNAMIC=1
 done
done
CFG=c3
run s1 COE_MAIN_STREAMS=1
run s2 COE_MAIN_STREAMS=2
run s2d COE_MAIN_STREAMS=2 COE_K3_DYNAMIC=1
