run() { tag=$1; shift; env "$@" timeout 300 python tools/timeline.py c3 10000 gpurun_out/tmp.json > gpurun_out/sw_$tag.log 2>&1; tail -1 gpurun_out/sw_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['timing']['total_ms'],1), round(d['copies']['busy_ms'],1))"; }
run base
run h1 COE_URGENT_HORIZON=1
run h4 COE_URGENT_HORIZON=4
run w16 COE_COPY_WINDOW=16
run w4 COE_COPY_WINDOW=4
run u4k COE_URGENT_ROWS=4096
run u16k COE_URGENT_ROWS=16384
run base2
