set -u
mkdir -p gpurun_out
for v in "INPUT_CTAS=64" "INPUT_CTAS=148" "INPUT_CTAS=296" "INPUT_DMA=2" "INPUT_DMA=1"; do
  env COE_$v timeout 600 python tools/timeline.py c1 10000 gpurun_out/r2m_tl_c1_$v.json e2e > gpurun_out/r2m_tl_c1_$v.log 2>&1
  env COE_$v timeout 600 python tools/timeline.py c3 10000 gpurun_out/r2m_tl_c3_$v.json e2e > gpurun_out/r2m_tl_c3_$v.log 2>&1
  echo "$v done" >> gpurun_out/r2m_rc.txt
done
cat gpurun_out/r2m_rc.txt
