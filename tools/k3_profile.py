"""Run K3 (grouped MLP) in isolation on one expert shape -- the command ncu profiles.

    python tools/k3_profile.py [groups] [requests_per_group] [iters] [d h T]
Default shape: config 3's (d=4096, h=12288, T=256).  Prints achieved TFLOP/s per
projection (CUDA events; never quote a number taken under ncu).
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import runtime

groups = int(sys.argv[1]) if len(sys.argv) > 1 else 16
per = int(sys.argv[2]) if len(sys.argv) > 2 else 8
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
d, h, T = (int(v) for v in sys.argv[4:7]) if len(sys.argv) > 6 else (4096, 12288, 256)
shape = runtime.RuntimeShape(d, h, T)
rt = runtime.B200Runtime(shape, num_experts=16, num_slots=16, max_requests=groups * per, max_admissions=groups * per,
                         max_wave_rows=groups * per * shape.T)
rt.fill_inputs(groups * per)
up, down = rt.bench_mlp(groups, per, iters)
rows = groups * per * shape.T
f = 2.0 * rows * shape.d * shape.h
print(json.dumps({"shape": [d, h, T], "groups": groups, "requests_per_group": per, "rows": rows, "up_ms": up,
                  "down_ms": down, "up_tflops": f / up / 1e9, "down_tflops": f / down / 1e9, "flops_per_launch": f}))
