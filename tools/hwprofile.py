"""B200 hardware profiler CLI: ``profiler.measure_b200_device`` over every expert shape of the
committed configs, written to gpurun_out/b200_exec.json for review before it replaces
paper_2503_02354_b200/data/b200_exec.json (which
tools/make_configs.py turns into the shared device documents read by the planner and the oracle).

    python tools/hwprofile.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import configs, profiler  # noqa: E402

shapes = set()
for name in configs.NAMES:
    cfg = json.load(open(os.path.join(configs.CONFIG_DIR, name, "config.json")))
    for s in cfg["shapes"].values():
        shapes.add((s["d"], s["h"], s["T"]))
doc = profiler.measure_b200_device(shapes)
for key, v in sorted(doc["shapes"].items()):
    print(key, v["k_s"], v["b_s"], "swap", v["swap_s"], flush=True)
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/b200_exec.json"  # review, then copy to data/
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc["host_tier"]), "->", out)
