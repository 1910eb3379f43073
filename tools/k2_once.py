"""One coe_group_sort + coe_run_compact call at n admissions (the command ncu profiles).

    python tools/k2_once.py [n]
Serving-like run-ranks (a new run every ~5 admissions), batches of <= 8 per run, as tools/k12_scale.py."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import _native  # noqa: E402
from paper_2503_02354_b200._cuda_sigs import check  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
lib = _native.cuda_lib()
rng = np.random.default_rng(n)
rank = np.cumsum(rng.random(n) < 0.2).astype(np.int32)
bits = max(1, int(rank.max()).bit_length())
starts = np.flatnonzero(np.r_[True, np.diff(rank) != 0])
lens = np.diff(np.r_[starts, n])
order = []
for l in lens:  # each run split into slices of <= 8, in run order
    order.extend([8] * (l // 8) + ([l % 8] if l % 8 else []))
sizes = np.array(order, np.int32)
nb = len(sizes)
dev = torch.device("cuda")
s = torch.cuda.current_stream().cuda_stream
t_ex = torch.zeros(n, dtype=torch.int32, device=dev)
t_rk = torch.from_numpy(rank).to(dev)
perm = torch.empty(n, dtype=torch.int32, device=dev)
keys = torch.empty(n, dtype=torch.int32, device=dev)
scratch = torch.empty(lib.coe_group_sort_scratch_bytes(n), dtype=torch.uint8, device=dev)
t_sizes = torch.from_numpy(sizes).to(dev)
t_bex = torch.zeros(nb, dtype=torch.int32, device=dev)
req = torch.arange(n, dtype=torch.int32, device=dev)
stage = torch.zeros(n, dtype=torch.int32, device=dev)
boff = torch.empty(nb, dtype=torch.int32, device=dev)
mreq = torch.empty(n, dtype=torch.int32, device=dev)
mst = torch.empty(n, dtype=torch.int32, device=dev)
flags = torch.zeros(2, dtype=torch.int32, device=dev)
cscr = torch.empty(max(64, lib.coe_run_compact_scratch_bytes(n, nb, 1)), dtype=torch.uint8, device=dev)
for _ in range(2):
    check(lib, lib.coe_group_sort(t_ex.data_ptr(), t_rk.data_ptr(), n, bits, (bits + 7) // 8, perm.data_ptr(),
                                  keys.data_ptr(), scratch.data_ptr(), s), "sort")
    check(lib, lib.coe_run_compact(perm.data_ptr(), keys.data_ptr(), req.data_ptr(), stage.data_ptr(), n, bits,
                                   t_bex.data_ptr(), t_sizes.data_ptr(), nb, 1, boff.data_ptr(), mreq.data_ptr(),
                                   mst.data_ptr(), flags.data_ptr(), flags[1:].data_ptr(), cscr.data_ptr(), s),
          "compact")
torch.cuda.synchronize()
assert int(flags[1].item()) == 0
