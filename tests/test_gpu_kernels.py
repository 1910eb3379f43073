"""Kernel-level GPU tests through the C-ABI (pytest -m gpu).

K1 coe_group_sort: stable segmented radix sort by (executor, run_rank) equals
numpy's stable lexsort, bit-exact, across sizes incl. empty / ragged tiles.
K2 coe_run_compact: batch offsets, members and violation detection.
K3 coe_grouped_mlp: grouped gelu-MLP over gathered request rows vs a plain
PyTorch fp32 reference of the same op (rel-L2 <= 5e-3; bf16 operands / fp32
accumulate), for T in {64, 128, 256}, partial M tiles, mixed stages (X vs
ping-pong buffers), several expert slots per launch.
"""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2503_02354_b200 import _native

    return _native.cuda_lib()


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _ck(lib, code, what=""):
    from paper_2503_02354_b200._cuda_sigs import check

    check(lib, code, what)


def _run_ranks(rng, n, executors):
    ex = rng.integers(0, executors, n).astype(np.int32)
    rank = np.zeros(n, np.int32)
    nxt = [0] * executors
    for i in range(n):
        x = ex[i]
        if nxt[x] == 0 or rng.random() < 0.3:
            rank[i] = nxt[x]
            nxt[x] += 1
        else:
            rank[i] = rng.integers(max(0, nxt[x] - 6), nxt[x])
    return ex, rank


@pytest.mark.parametrize("n, executors", [(1, 1), (7, 1), (2048, 2), (2049, 3), (4097, 1), (50000, 8), (120000, 4),
                                          (1 << 20, 2)])
def test_group_sort_matches_stable_lexsort(lib, n, executors):
    import torch

    rng = np.random.default_rng(n)
    ex, rank = _run_ranks(rng, n, executors)
    bits = max(1, int(rank.max()).bit_length())
    passes = (bits + 3 + 7) // 8
    dev = torch.device("cuda")
    t_ex, t_rk = torch.from_numpy(ex).to(dev), torch.from_numpy(rank).to(dev)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    keys = torch.empty(n, dtype=torch.int32, device=dev)
    scratch = torch.empty(lib.coe_group_sort_scratch_bytes(n), dtype=torch.uint8, device=dev)
    _ck(lib, lib.coe_group_sort(t_ex.data_ptr(), t_rk.data_ptr(), n, bits, passes, perm.data_ptr(), keys.data_ptr(),
                                scratch.data_ptr(), _stream()), "sort")
    torch.cuda.synchronize()
    ref = np.lexsort((np.arange(n), rank, ex))
    assert np.array_equal(perm.cpu().numpy(), ref)
    k = keys.cpu().numpy().astype(np.int64)
    assert np.array_equal(k, (ex[ref].astype(np.int64) << bits) | rank[ref])


@pytest.mark.parametrize("n, executors, rank_bits",
                         [(1_000_000, 2, 20), ((1 << 20) + 1, 3, 18), (3_000_000, 8, 22)])
def test_group_sort_large_tiles_and_four_passes(lib, n, executors, rank_bits):
    """Past 1M admissions K1 switches to 4096-key tiles; 8 executors x 22 rank bits = 4 passes.
    1M and 3M keys have more tiles than the persistent grid has CTAs (977 x 1,024-key tiles vs
    6 per SM; 733 x 4,096-key tiles vs 3 per SM), so CTAs claim several tiles each."""
    import torch

    rng = np.random.default_rng(n)
    ex = rng.integers(0, executors, n).astype(np.int32)
    rank = rng.integers(0, 1 << rank_bits, n).astype(np.int32)
    rank[rng.random(n) < 0.5] = 7  # long equal-key runs: stability across many tiles
    passes = (rank_bits + (executors - 1).bit_length() + 7) // 8
    dev = torch.device("cuda")
    t_ex, t_rk = torch.from_numpy(ex).to(dev), torch.from_numpy(rank).to(dev)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    keys = torch.empty(n, dtype=torch.int32, device=dev)
    scratch = torch.empty(lib.coe_group_sort_scratch_bytes(n), dtype=torch.uint8, device=dev)
    _ck(lib, lib.coe_group_sort(t_ex.data_ptr(), t_rk.data_ptr(), n, rank_bits, passes, perm.data_ptr(),
                                keys.data_ptr(), scratch.data_ptr(), _stream()), "sort")
    torch.cuda.synchronize()
    ref = np.lexsort((np.arange(n), rank, ex))
    assert np.array_equal(perm.cpu().numpy(), ref)
    k = keys.cpu().numpy().astype(np.int64) & 0xFFFFFFFF
    assert np.array_equal(k, (ex[ref].astype(np.int64) << rank_bits) | rank[ref])


@pytest.mark.parametrize("n, X", [(5000, 2), (200000, 3)])
def test_run_compact_offsets_members_and_violations(lib, n, X):
    import torch

    rng = np.random.default_rng(5)
    ex, rank = _run_ranks(rng, n, X)
    bits = max(1, int(rank.max()).bit_length())
    dev = torch.device("cuda")
    order = np.lexsort((np.arange(n), rank, ex))
    # batches: consecutive slices of each executor's run, sizes <= 5, listed interleaved across executors
    per_exec = []
    for x in range(X):
        idx = order[ex[order] == x]
        runs = np.split(idx, np.flatnonzero(np.diff(rank[idx])) + 1)
        sizes = []
        for run in runs:
            left = len(run)
            while left:
                take = int(min(left, rng.integers(1, 6)))
                sizes.append(take)
                left -= take
        per_exec.append(sizes)
    b_exec, b_size = [], []
    cursors = [0] * X
    while any(cursors[x] < len(per_exec[x]) for x in range(X)):
        for x in range(X):
            if cursors[x] < len(per_exec[x]):
                b_exec.append(x)
                b_size.append(per_exec[x][cursors[x]])
                cursors[x] += 1
    req = rng.integers(0, 10**6, n).astype(np.int32)
    stage = rng.integers(0, 3, n).astype(np.int32)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)  # noqa: E731
    perm = T(order)
    keys = T(((ex[order].astype(np.int64) << bits) | rank[order]).astype(np.int32))
    nb = len(b_size)
    boff = torch.empty(nb, dtype=torch.int32, device=dev)
    mreq = torch.empty(n, dtype=torch.int32, device=dev)
    mst = torch.empty(n, dtype=torch.int32, device=dev)
    flags = torch.zeros(2, dtype=torch.int32, device=dev)
    scratch = torch.empty(lib.coe_run_compact_scratch_bytes(n, nb, X), dtype=torch.uint8, device=dev)

    t_req, t_stage, t_exec = T(req), T(stage), T(b_exec)

    def run(sizes):
        t_sizes = T(sizes)  # device arrays must outlive the asynchronous launch
        _ck(lib, lib.coe_run_compact(perm.data_ptr(), keys.data_ptr(), t_req.data_ptr(), t_stage.data_ptr(), n,
                                     bits, t_exec.data_ptr(), t_sizes.data_ptr(), nb, X, boff.data_ptr(),
                                     mreq.data_ptr(), mst.data_ptr(), flags.data_ptr(), flags[1:].data_ptr(),
                                     scratch.data_ptr(), _stream()), "compact")
        torch.cuda.synchronize()
        return boff.cpu().numpy(), flags.cpu().numpy()

    off, fl = run(b_size)
    assert fl[1] == 0
    assert fl[0] == len(set(zip(ex.tolist(), rank.tolist())))
    assert np.array_equal(mreq.cpu().numpy(), req[order]) and np.array_equal(mst.cpu().numpy(), stage[order])
    starts = {x: int(np.flatnonzero(ex[order] == x)[0]) for x in range(X)}
    expect, acc = [], [0] * X
    for x, sz in zip(b_exec, b_size):
        expect.append(starts[x] + acc[x])
        acc[x] += sz
    assert off.tolist() == expect
    # shifting one member across a run boundary must be flagged
    keys_sorted = (ex[order].astype(np.int64) << bits) | rank[order]
    idx0 = [i for i, x in enumerate(b_exec) if x == 0]
    j = next(j for j in range(len(idx0) - 1)
             if keys_sorted[expect[idx0[j]] + b_size[idx0[j]]] != keys_sorted[expect[idx0[j]]])
    bad = list(b_size)
    bad[idx0[j]] += 1
    bad[idx0[j + 1]] -= 1
    _, fl = run(bad)
    assert fl[1] >= 1


def _mlp_case(lib, d, h, T, spec, slots=3):
    """spec: list of (members [(request, stage)], slot). Returns worst rel-L2 vs torch fp32."""
    import torch

    from paper_2503_02354_b200._cuda_sigs import MlpConfig, MlpGroup

    dev = torch.device("cuda")
    nreq = 1 + max(r for mem, _ in spec for r, _ in mem)
    g = torch.Generator(device=dev).manual_seed(d + h + T)
    mk = lambda: (torch.rand(nreq * T, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    x, p0, p1 = mk(), mk(), mk()
    slab = ((torch.rand(slots, 2 * h * d, device=dev, generator=g) * 2 - 1) * 0.05).to(torch.bfloat16)
    rows_total = sum(len(m) * T for m, _ in spec)
    hs = torch.zeros(max(rows_total, 128), h, dtype=torch.bfloat16, device=dev)
    cfg = MlpConfig(d, h, T, x.data_ptr(), p0.data_ptr(), p1.data_ptr(), nreq * T, hs.data_ptr(), hs.shape[0],
                    slab.data_ptr(), slots, 2 * h * d * 2)
    handle = ctypes.c_void_p()
    _ck(lib, lib.coe_mlp_create(ctypes.byref(cfg), ctypes.byref(handle)), "create")
    G = len(spec)
    up, down = (MlpGroup * G)(), (MlpGroup * G)()
    mreq, mst, boff = [], [], []
    tu = td = hrow = 0
    for gi, (mem, slot) in enumerate(spec):
        boff.append(len(mreq))
        mreq += [r for r, _ in mem]
        mst += [s for _, s in mem]
        rows = len(mem) * T
        mt = (rows + 127) // 128
        for arr, ts in ((up, tu), (down, td)):
            arr[gi].rows, arr[gi].slot, arr[gi].batch, arr[gi].h_row, arr[gi].tile_start = rows, slot, gi, hrow, ts
        tu += mt * (h // 256)
        td += mt * (d // 256)
        hrow += rows
    dv = lambda a: torch.tensor(a, dtype=torch.int32, device=dev)  # noqa: E731
    gu = torch.frombuffer(bytearray(bytes(up)), dtype=torch.uint8).to(dev)
    gd = torch.frombuffer(bytearray(bytes(down)), dtype=torch.uint8).to(dev)
    src = {0: x.clone(), 1: p0.clone(), 2: p1.clone()}
    t_boff, t_mreq, t_mst = dv(boff), dv(mreq), dv(mst)  # keep alive until the kernel has run
    _ck(lib, lib.coe_grouped_mlp(handle, gu.data_ptr(), gd.data_ptr(), G, tu, td, t_boff.data_ptr(),
                                 t_mreq.data_ptr(), t_mst.data_ptr(), 3, 0, _stream()), "mlp")
    torch.cuda.synchronize()
    worst, hrow = 0.0, 0
    for mem, slot in spec:
        w1 = slab[slot, : h * d].view(h, d).float()
        w2 = slab[slot, h * d:].view(d, h).float()
        xs = torch.cat([src[0 if s == 0 else 1 + ((s - 1) & 1)][r * T:(r + 1) * T] for r, s in mem]).float()
        h_ref = torch.nn.functional.gelu(xs @ w1.T, approximate="tanh")
        h_got = hs[hrow: hrow + len(mem) * T].float()
        y_iso = h_got @ w2.T  # the down projection alone (from the kernel's own bf16 H)
        y_ref = h_ref @ w2.T  # the whole expert in fp32 (fp32 hidden activations)
        y_got = torch.cat([(p1 if s & 1 else p0)[r * T:(r + 1) * T] for r, s in mem]).float()
        for name, got, ref in (("H", h_got, h_ref), ("Y_down", y_got, y_iso), ("Y", y_got, y_ref)):
            err = ((got - ref).norm() / ref.norm()).item()
            if err > K3_TOL and os.environ.get("COE_DEBUG"):
                print(f"group slot={slot} members={mem} {name} err={err:.3g}")
            worst = max(worst, err)
        hrow += len(mem) * T
    lib.coe_mlp_destroy(handle)
    return worst


# bf16 operands, fp32 accumulation, bf16 H and Y storage: each rounding contributes ~1.1e-3
# rel-L2 (2^-9 / sqrt(3)); H, the down pass alone and the whole expert against fp32 (fp32 H)
K3_TOL = 5e-3

SPEC = [([(0, 0)], 0), ([(1, 0), (2, 1), (3, 2)], 1), ([(4, 1), (5, 3)], 2), ([(6, 0)], 1),
        ([(7 + i, i % 4) for i in range(9)], 0)]


@pytest.mark.parametrize("cg", [2, 1])
@pytest.mark.parametrize("d, h, T", [(1024, 2048, 128), (1024, 4096, 64), (2048, 1024, 256), (512, 768, 32)])
def test_grouped_mlp_matches_torch_fp32(lib, d, h, T, cg, monkeypatch):
    """cg 2: the CTA-pair kernel (tcgen05.mma.cta_group::2, 256 x 256 tiles); cg 1: one CTA."""
    monkeypatch.setenv("COE_K3_CG", str(cg))
    assert _mlp_case(lib, d, h, T, SPEC) <= K3_TOL


@pytest.mark.parametrize("cg", [2, 1])
def test_grouped_mlp_single_row_block_and_many_groups(lib, cg, monkeypatch):
    monkeypatch.setenv("COE_K3_CG", str(cg))
    spec = [([(i, i % 2)], i % 3) for i in range(40)]
    assert _mlp_case(lib, 1024, 1024, 64, spec) <= K3_TOL


def test_swap_in_entry_point(lib):
    """coe_swap_in (K4 alone): pinned host bytes land in the device slot; the event orders them."""
    import torch

    lib.coe_swap_in.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    lib.coe_swap_in.restype = ctypes.c_int
    n = 3 << 20
    src = torch.randint(0, 255, (n,), dtype=torch.uint8).pin_memory()
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    done = torch.cuda.Event()
    done.record(stream)  # materialise the event handle
    _ck(lib, lib.coe_swap_in(dst.data_ptr(), src.data_ptr(), n, stream.cuda_stream, done.cuda_event), "swap_in")
    done.synchronize()
    assert torch.equal(dst.cpu(), src)
    assert lib.coe_swap_in(None, src.data_ptr(), 16, stream.cuda_stream, None) != 0


@pytest.mark.parametrize("world", [2, 3])
def test_hop_all_to_all_entry_point(lib, world):
    """coe_hop (K5 alone): exact-count all-to-all of bf16 activations; ragged and empty
    segments, self copy, one thread per rank over the in-process transport."""
    import threading

    import torch

    lib.coe_local_hub_create.argtypes = [ctypes.c_int]
    lib.coe_local_hub_create.restype = ctypes.c_void_p
    lib.coe_comm_create_local.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    lib.coe_comm_create_local.restype = ctypes.c_int
    lib.coe_hop.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_void_p]
    lib.coe_hop.restype = ctypes.c_int
    lib.coe_comm_destroy.argtypes = [ctypes.c_void_p]
    lib.coe_local_hub_destroy.argtypes = [ctypes.c_void_p]
    hub = lib.coe_local_hub_create(world)
    count = lambda s, d: 0 if (s + d) % 4 == 3 else 64 * (1 + s) + 8 * d  # noqa: E731  (some segments empty)
    send, recv, comms, errs = [], [], [], []
    for r in range(world):
        c = ctypes.c_void_p()
        _ck(lib, lib.coe_comm_create_local(hub, r, ctypes.byref(c)), "comm")
        comms.append(c)
        segs = [torch.full((count(r, d),), float(100 * r + d), dtype=torch.bfloat16, device="cuda")
                for d in range(world)]
        send.append(torch.cat(segs))
        recv.append(torch.zeros(sum(count(s, r) for s in range(world)), dtype=torch.bfloat16, device="cuda"))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(world)]

    def rank(r):
        sc = (ctypes.c_int64 * world)(*[count(r, d) for d in range(world)])
        rc = (ctypes.c_int64 * world)(*[count(s, r) for s in range(world)])
        code = lib.coe_hop(comms[r], send[r].data_ptr(), sc, recv[r].data_ptr(), rc, streams[r].cuda_stream)
        if code:
            errs.append(code)

    threads = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    assert not errs
    for r in range(world):
        expect = torch.cat([torch.full((count(s, r),), float(100 * s + r), dtype=torch.bfloat16, device="cuda")
                            for s in range(world)])
        assert torch.equal(recv[r], expect)
    for c in comms:
        lib.coe_comm_destroy(c)
    lib.coe_local_hub_destroy(hub)


@pytest.mark.parametrize("n", [1, 7, 1000, 8192, 8193, 13642, 16384, 16385, 32768])
def test_group_compact_fused_matches_stable_sort(lib, n):
    """coe_group_compact_fused (K1 + K2 of one executor in one block): the permutation is the
    stable sort by run-rank, members and routes follow it, batch offsets are the scan of the
    sizes, runs are counted, and a batch shifted across a run boundary is flagged."""
    import torch

    lib.coe_group_compact_fused.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                                                     ctypes.c_int] + [ctypes.c_void_p] * 8
    lib.coe_group_compact_fused.restype = ctypes.c_int
    rng = np.random.default_rng(n)
    # serving-shaped steps: at most ~2,000 runs, batches of up to 6 (or more when runs are long)
    # so the step stays inside COE_FUSED_MAX_BATCHES (the runtime falls back to K1 + K2 beyond)
    rank = np.zeros(n, np.int32)
    nxt, p_new = 0, min(0.3, 2000.0 / n)
    for i in range(n):
        if nxt == 0 or rng.random() < p_new:
            rank[i] = nxt
            nxt += 1
        else:
            rank[i] = rng.integers(max(0, nxt - 6), nxt)
    bits = max(1, int(rank.max()).bit_length())
    order = np.argsort(rank, kind="stable")
    runs = np.split(order, np.flatnonzero(np.diff(rank[order])) + 1)
    hi = max(7, 2 * n // 3000 + 2)
    sizes = []
    for run in runs:
        left = len(run)
        while left:
            take = int(min(left, rng.integers(1, hi)))
            sizes.append(take)
            left -= take
    assert len(sizes) <= 4096
    dev = torch.device("cuda")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)  # noqa: E731
    req = rng.integers(0, 10**6, n).astype(np.int32)
    stage = rng.integers(0, 5, n).astype(np.int32)
    rin = rng.integers(0, 2**30, n).astype(np.int32)
    rout = rng.integers(0, 2**30, n).astype(np.int32)
    t = {k: T(v) for k, v in dict(rank=rank, req=req, stage=stage, rin=rin, rout=rout).items()}
    out = {k: torch.empty(max(1, n), dtype=torch.int32, device=dev) for k in ("perm", "mreq", "mst", "min", "mout")}
    nb = len(sizes)
    boff = torch.empty(nb, dtype=torch.int32, device=dev)
    flags = torch.full((2,), -1, dtype=torch.int32, device=dev)

    def run(sz):
        t_sz = T(sz)
        _ck(lib, lib.coe_group_compact_fused(t["rank"].data_ptr(), t["req"].data_ptr(), t["stage"].data_ptr(),
                                             t["rin"].data_ptr(), t["rout"].data_ptr(), n, bits, t_sz.data_ptr(), nb,
                                             out["perm"].data_ptr(), boff.data_ptr(), out["mreq"].data_ptr(),
                                             out["mst"].data_ptr(), out["min"].data_ptr(), out["mout"].data_ptr(),
                                             flags.data_ptr(), _stream()), "fused")
        torch.cuda.synchronize()
        return boff.cpu().numpy(), flags.cpu().numpy()

    off, fl = run(sizes)
    g = lambda k: out[k].cpu().numpy()[:n]  # noqa: E731
    assert np.array_equal(g("perm"), order)
    assert np.array_equal(g("mreq"), req[order]) and np.array_equal(g("mst"), stage[order])
    assert np.array_equal(g("min"), rin[order]) and np.array_equal(g("mout"), rout[order])
    assert fl[0] == len(runs) and fl[1] == 0
    assert off.tolist() == np.concatenate([[0], np.cumsum(sizes)[:-1]]).tolist()
    if len(runs) > 1:  # move one member of the first run into the next batch's run
        bad = list(sizes)
        first_end = next(i for i in range(nb) if sum(sizes[:i + 1]) == len(runs[0]))
        bad[first_end] += 1
        bad[first_end + 1] -= 1
        if bad[first_end + 1] == 0:
            bad[first_end + 1] = 1
            bad[-1] -= 1
        _, fl = run(bad)
        assert fl[1] >= 1
