# Final round-2 evidence on the final code: GPU suite, smoke, then tools/profile_round.sh r2z
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2z_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2z_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2z_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2z_rc.txt
bash tools/profile_round.sh r2z > gpurun_out/r2z_profile_round.log 2>&1; echo "profile round rc=$?" >> gpurun_out/r2z_rc.txt
for f in gpurun_out/r2z_bench_*.log; do echo "$f rc-tail: $(tail -c 200 $f | tr '\n' ' ')" >> gpurun_out/r2z_rc.txt; done
cat gpurun_out/r2z_rc.txt
