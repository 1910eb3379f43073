set -u
mkdir -p gpurun_out
COE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c4 --requests 1000 --steps 3 --warmup 3 > gpurun_out/r2v_bench_c4_2ranks.log 2>&1; echo "c4 2 ranks rc=$?" >> gpurun_out/r2v_rc.txt
COE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --requests 1000 --steps 3 --warmup 3 > gpurun_out/r2v_bench_c3_2ranks.log 2>&1; echo "c3 2 ranks rc=$?" >> gpurun_out/r2v_rc.txt
COE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2v_bench_ref_2ranks.log 2>&1; echo "ref 2 ranks rc=$?" >> gpurun_out/r2v_rc.txt
cat gpurun_out/r2v_rc.txt
