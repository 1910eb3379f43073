set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2w_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r2w_rc.txt
bash tools/gpu_runs/r2v_run.sh > /dev/null 2>&1; cat gpurun_out/r2v_rc.txt >> gpurun_out/r2w_rc.txt
cat gpurun_out/r2w_rc.txt
