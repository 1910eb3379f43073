"""Quick GPU check of K1/K2/K3 against torch / numpy references (debug tool)."""
import ctypes, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2503_02354_b200 import _native, _cuda_sigs as S

lib = _native.cuda_lib()
dev = torch.device("cuda")
stream = torch.cuda.current_stream().cuda_stream

def ck(code, what):
    S.check(lib, code, what)

# ---------------- K1 / K2 ----------------
rng = np.random.default_rng(0)
n = 50000
X = 3
ex = rng.integers(0, X, n).astype(np.int32)
rank = np.zeros(n, np.int32)
counters = [0] * X
for i in range(n):  # plausible run ranks: non-decreasing new runs, joins of live runs
    x = ex[i]
    if counters[x] == 0 or rng.random() < 0.3:
        rank[i] = counters[x]; counters[x] += 1
    else:
        rank[i] = rng.integers(max(0, counters[x] - 5), counters[x])
rank_bits = int(max(1, int(rank.max()).bit_length()))
passes = (rank_bits + 2 + 7) // 8
t_ex = torch.from_numpy(ex).to(dev); t_rk = torch.from_numpy(rank).to(dev)
perm = torch.empty(n, dtype=torch.int32, device=dev); keys = torch.empty(n, dtype=torch.int32, device=dev)
scratch = torch.empty(lib.coe_group_sort_scratch_bytes(n), dtype=torch.uint8, device=dev)
ck(lib.coe_group_sort(t_ex.data_ptr(), t_rk.data_ptr(), n, rank_bits, passes, perm.data_ptr(), keys.data_ptr(), scratch.data_ptr(), stream), "sort")
torch.cuda.synchronize()
ref = np.lexsort((np.arange(n), rank, ex)).astype(np.int32)
print("K1 sort match:", np.array_equal(perm.cpu().numpy(), ref))

# ---------------- K3 ----------------
def run_k3(d, h, T, nreq, slots, groups_spec):
    act0 = (torch.rand(nreq * T, d, device=dev) * 2 - 1).to(torch.bfloat16)
    act1 = (torch.rand(nreq * T, d, device=dev) * 2 - 1).to(torch.bfloat16)
    slab = torch.empty(slots, 2 * h * d, dtype=torch.bfloat16, device=dev)
    slab.uniform_(-1, 1); slab.mul_(0.05)
    total_rows = sum(len(m) * T for m, _ in groups_spec)
    hs = torch.zeros(max(total_rows, 128), h, dtype=torch.bfloat16, device=dev)
    cfg = S.MlpConfig(d, h, T, act0.data_ptr(), act1.data_ptr(), nreq * T, hs.data_ptr(), hs.shape[0], slab.data_ptr(), slots, 2 * h * d * 2)
    handle = ctypes.c_void_p()
    ck(lib.coe_mlp_create(ctypes.byref(cfg), ctypes.byref(handle)), "create")
    members_req, members_stage, batch_off = [], [], []
    for mem, slot in groups_spec:
        batch_off.append(len(members_req))
        for r, st in mem:
            members_req.append(r); members_stage.append(st)
    G = len(groups_spec)
    up = (S.MlpGroup * G)(); down = (S.MlpGroup * G)()
    tu = td = 0; hrow = 0
    for g, (mem, slot) in enumerate(groups_spec):
        rows = len(mem) * T
        mt = (rows + 127) // 128
        for arr, tstart in ((up, tu), (down, td)):
            arr[g].rows = rows; arr[g].slot = slot; arr[g].batch = g; arr[g].h_row = hrow; arr[g].tile_start = tstart
        tu += mt * (h // 256); td += mt * (d // 256); hrow += rows
    gu = torch.frombuffer(bytearray(bytes(up)), dtype=torch.uint8).to(dev)
    gd = torch.frombuffer(bytearray(bytes(down)), dtype=torch.uint8).to(dev)
    bo = torch.tensor(batch_off, dtype=torch.int32, device=dev)
    mr = torch.tensor(members_req, dtype=torch.int32, device=dev)
    ms = torch.tensor(members_stage, dtype=torch.int32, device=dev)
    a0c, a1c = act0.clone(), act1.clone()
    ck(lib.coe_grouped_mlp(handle, gu.data_ptr(), gd.data_ptr(), G, tu, td, bo.data_ptr(), mr.data_ptr(), ms.data_ptr(), 3, stream), "mlp")
    torch.cuda.synchronize()
    worst = 0.0
    hrow = 0
    for g, (mem, slot) in enumerate(groups_spec):
        W1 = slab[slot, : h * d].view(h, d).float(); W2 = slab[slot, h * d :].view(d, h).float()
        xs = torch.cat([(a0c if st % 2 == 0 else a1c)[r * T:(r + 1) * T] for r, st in mem]).float()
        Href = torch.nn.functional.gelu(xs @ W1.T, approximate="tanh")
        Hgot = hs[hrow: hrow + len(mem) * T].float()
        eh = ((Hgot - Href).norm() / Href.norm()).item()
        Yref = Hgot @ W2.T
        ygot = torch.cat([(act1 if st % 2 == 0 else act0)[r * T:(r + 1) * T] for r, st in mem]).float()
        ey = ((ygot - Yref).norm() / Yref.norm()).item()
        worst = max(worst, eh, ey)
        hrow += len(mem) * T
    lib.coe_mlp_destroy(handle)
    return worst

for (d, h, T) in [(1024, 2048, 128), (1024, 4096, 64), (2048, 1024, 256)]:
    nreq = 24
    spec = [([(0, 0)], 0), ([(1, 0), (2, 1), (3, 0)], 1), ([(4, 1), (5, 1)], 2), ([(6, 0)] , 1),
            ([(7 + i, i % 2) for i in range(9)], 0)]
    err = run_k3(d, h, T, nreq, 3, spec)
    print(f"K3 d={d} h={h} T={T}: worst rel err {err:.3e}")

# timing: one big group, C3 shape
d, h, T = 4096, 12288, 256
nreq = 16
act0 = torch.randn(nreq * T, d, device=dev).to(torch.bfloat16); act1 = torch.zeros_like(act0)
slab = (torch.randn(2, 2 * h * d, device=dev) * 0.02).to(torch.bfloat16)
hs = torch.empty(nreq * T, h, dtype=torch.bfloat16, device=dev)
cfg = S.MlpConfig(d, h, T, act0.data_ptr(), act1.data_ptr(), nreq * T, hs.data_ptr(), hs.shape[0], slab.data_ptr(), 2, 2 * h * d * 2)
handle = ctypes.c_void_p(); ck(lib.coe_mlp_create(ctypes.byref(cfg), ctypes.byref(handle)), "create")
up = (S.MlpGroup * 1)(); down = (S.MlpGroup * 1)()
rows = nreq * T
for arr in (up, down):
    arr[0].rows = rows; arr[0].slot = 1; arr[0].batch = 0; arr[0].h_row = 0; arr[0].tile_start = 0
gu = torch.frombuffer(bytearray(bytes(up)), dtype=torch.uint8).to(dev); gd = torch.frombuffer(bytearray(bytes(down)), dtype=torch.uint8).to(dev)
bo = torch.zeros(1, dtype=torch.int32, device=dev); mr = torch.arange(nreq, dtype=torch.int32, device=dev); ms = torch.zeros(nreq, dtype=torch.int32, device=dev)
tu = (rows // 128) * (h // 256); td = (rows // 128) * (d // 256)
for which, name, flops in ((1, "up", 2 * rows * d * h), (2, "down", 2 * rows * d * h)):
    for _ in range(3):
        ck(lib.coe_grouped_mlp(handle, gu.data_ptr(), gd.data_ptr(), 1, tu, td, bo.data_ptr(), mr.data_ptr(), ms.data_ptr(), which, stream), "mlp")
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ck(lib.coe_grouped_mlp(handle, gu.data_ptr(), gd.data_ptr(), 1, tu, td, bo.data_ptr(), mr.data_ptr(), ms.data_ptr(), which, stream), "mlp")
    e1.record(); torch.cuda.synchronize()
    ms_ = e0.elapsed_time(e1) / 20
    print(f"K3 {name} M={rows} d={d} h={h}: {ms_*1e3:.1f} us, {flops / ms_ / 1e9:.1f} TFLOP/s")
W1 = slab[1, : h * d].view(h, d)
x = act0
for _ in range(3): torch.matmul(x, W1.T)
e0.record()
for _ in range(20): torch.matmul(x, W1.T)
e1.record(); torch.cuda.synchronize()
ms_ = e0.elapsed_time(e1) / 20
print(f"torch matmul up: {ms_*1e3:.1f} us, {2*rows*d*h / ms_ / 1e9:.1f} TFLOP/s")
