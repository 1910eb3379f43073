"""Run K3 (grouped MLP) on the C3 expert shape in isolation -- the command ncu profiles.

    python tools/k3_profile.py [groups] [requests_per_group] [iters]
Prints achieved TFLOP/s per projection (CUDA events; never quote a number taken under ncu).
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import runtime

groups = int(sys.argv[1]) if len(sys.argv) > 1 else 16
per = int(sys.argv[2]) if len(sys.argv) > 2 else 8
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
shape = runtime.RuntimeShape(4096, 12288, 256)
rt = runtime.B200Runtime(shape, num_experts=16, num_slots=16, max_requests=groups * per, max_admissions=groups * per,
                         max_wave_rows=groups * per * shape.T)
rt.fill_inputs(groups * per)
up, down = rt.bench_mlp(groups, per, iters)
rows = groups * per * shape.T
f = 2.0 * rows * shape.d * shape.h
print(json.dumps({"groups": groups, "requests_per_group": per, "rows": rows, "up_ms": up, "down_ms": down,
                  "up_tflops": f / up / 1e9, "down_tflops": f / down / 1e9, "flops_per_launch": f}))
