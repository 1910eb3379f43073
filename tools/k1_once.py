"""One coe_group_sort call at n admissions (the command ncu profiles).

    python tools/k1_once.py [n] [serving|random]
serving: run-ranks like a serving queue (a new run every ~5 admissions); random: uniform 22-bit."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import _native  # noqa: E402
from paper_2503_02354_b200._cuda_sigs import check  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
lib = _native.cuda_lib()
rng = np.random.default_rng(n)
if len(sys.argv) > 2 and sys.argv[2] == "random":
    rank = rng.integers(0, 1 << 22, n).astype(np.int32)
else:
    rank = np.cumsum(rng.random(n) < 0.2).astype(np.int32)
bits = max(1, int(rank.max()).bit_length())
dev = torch.device("cuda")
t_ex = torch.zeros(n, dtype=torch.int32, device=dev)
t_rk = torch.from_numpy(rank).to(dev)
perm = torch.empty(n, dtype=torch.int32, device=dev)
keys = torch.empty(n, dtype=torch.int32, device=dev)
scratch = torch.empty(lib.coe_group_sort_scratch_bytes(n), dtype=torch.uint8, device=dev)
for _ in range(2):
    check(lib, lib.coe_group_sort(t_ex.data_ptr(), t_rk.data_ptr(), n, bits, (bits + 7) // 8, perm.data_ptr(),
                                  keys.data_ptr(), scratch.data_ptr(), torch.cuda.current_stream().cuda_stream), "sort")
torch.cuda.synchronize()
