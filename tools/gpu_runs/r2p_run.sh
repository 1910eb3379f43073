set -u
mkdir -p gpurun_out
for dbg in 0 1 2 3; do
  for w in "11 44 1024 4096 64" "11 22 2048 8192 128" "16 6 4096 12288 256"; do
    set -- $w
    COE_K3_DEBUG=$dbg timeout 300 python tools/k3_profile.py $1 $2 20 $3 $4 $5 | sed "s/^/dbg$dbg /"
  done
done > gpurun_out/r2p_k3_debug.log 2>&1
echo "debug sweep rc=$?" >> gpurun_out/r2p_rc.txt
timeout 900 bash tools/k3_sweep.sh > gpurun_out/r2p_k3_sweep_auto.log 2>&1; echo "sweep auto rc=$?" >> gpurun_out/r2p_rc.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2p_bench_c1.log 2>&1; echo "bench c1 rc=$?" >> gpurun_out/r2p_rc.txt
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2p_bench_c2.log 2>&1; echo "bench c2 rc=$?" >> gpurun_out/r2p_rc.txt
cat gpurun_out/r2p_rc.txt
