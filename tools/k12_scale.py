"""K1 (coe_group_sort) and K2 (coe_run_compact) from serving size up to HBM-bound sizes.

    python tools/k12_scale.py [out.json] [serving|random]

Admissions of one executor with run-ranks like a serving queue (a new run every ~5
admissions; or uniform 22-bit run-ranks with "random"), sorted by (executor, run_rank) and compacted into batches of <= 8.  Times are
CUDA events over 20 launches after warm-up; algorithmic bytes: K1 16 B per admission (read
executor + run_rank, write permutation + key), K2 24 B per admission (read permutation, key,
request, stage; write member request + stage) plus 12 B per batch.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import _native  # noqa: E402
from paper_2503_02354_b200._cuda_sigs import check  # noqa: E402


def main() -> None:
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/k12_scale.json"
    dist = sys.argv[2] if len(sys.argv) > 2 else "serving"
    lib = _native.cuda_lib()
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream().cuda_stream
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6539.2)
    cub = None
    cub_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cub_ab", "libcub_sort.so")
    if os.path.exists(cub_path):
        import ctypes

        cub = ctypes.CDLL(cub_path)
        cub.cub_sort_pairs_scratch_bytes.restype = ctypes.c_size_t
        cub.cub_sort_pairs_scratch_bytes.argtypes = [ctypes.c_int64]
        cub.cub_sort_pairs.restype = ctypes.c_int
        cub.cub_sort_pairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                                                ctypes.c_size_t, ctypes.c_void_p]
    rows = []
    for n in (13642, 262144, 1 << 20, 1 << 22, 1 << 24):
        rng = np.random.default_rng(n)
        if dist == "random":  # uniform 22-bit run-ranks: every tile touches every digit
            rank = rng.integers(0, 1 << 22, n).astype(np.int32)
        else:
            rank = np.cumsum(rng.random(n) < 0.2).astype(np.int32)
            rank = np.minimum(rank, (1 << 23) - 1)
        ex = np.zeros(n, np.int32)
        bits = max(1, int(rank.max()).bit_length())
        passes = (bits + 7) // 8
        t_ex, t_rk = torch.from_numpy(ex).to(dev), torch.from_numpy(rank).to(dev)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        keys = torch.empty(n, dtype=torch.int32, device=dev)
        scratch = torch.empty(lib.coe_group_sort_scratch_bytes(n), dtype=torch.uint8, device=dev)
        # batches: each run split into slices of <= 8, in run order
        starts = np.flatnonzero(np.r_[True, np.diff(np.sort(rank)) != 0])
        lens = np.diff(np.r_[starts, n])
        sizes = np.concatenate([np.r_[np.full(l // 8, 8), [l % 8] if l % 8 else []] for l in lens]).astype(np.int32)
        nb = len(sizes)
        t_sizes = torch.from_numpy(sizes).to(dev)
        t_bex = torch.zeros(nb, dtype=torch.int32, device=dev)
        req = torch.arange(n, dtype=torch.int32, device=dev)
        stage = torch.zeros(n, dtype=torch.int32, device=dev)
        boff = torch.empty(nb, dtype=torch.int32, device=dev)
        mreq = torch.empty(n, dtype=torch.int32, device=dev)
        mst = torch.empty(n, dtype=torch.int32, device=dev)
        flags = torch.zeros(2, dtype=torch.int32, device=dev)
        cscr = torch.empty(max(64, lib.coe_run_compact_scratch_bytes(n, nb, 1)), dtype=torch.uint8, device=dev)

        def k1():
            check(lib, lib.coe_group_sort(t_ex.data_ptr(), t_rk.data_ptr(), n, bits, passes, perm.data_ptr(),
                                          keys.data_ptr(), scratch.data_ptr(), stream), "sort")

        def k2():
            check(lib, lib.coe_run_compact(perm.data_ptr(), keys.data_ptr(), req.data_ptr(), stage.data_ptr(), n,
                                           bits, t_bex.data_ptr(), t_sizes.data_ptr(), nb, 1, boff.data_ptr(),
                                           mreq.data_ptr(), mst.data_ptr(), flags.data_ptr(), flags[1:].data_ptr(),
                                           cscr.data_ptr(), stream), "compact")

        res = {"admissions": n, "batches": nb, "rank_bits": bits, "passes": passes, "keys": dist}
        cases = [("k1", k1, 16 * n), ("k2", k2, 24 * n + 12 * nb)]
        if cub is not None:  # library baseline: CUB SortPairs on the same keys, values and bit range
            ck_in = t_rk.clone()  # executor 0: the key is the run-rank
            cv_in = torch.arange(n, dtype=torch.int32, device=dev)
            ck_out, cv_out = torch.empty_like(ck_in), torch.empty_like(cv_in)
            cbytes = cub.cub_sort_pairs_scratch_bytes(n)
            cscratch = torch.empty(max(1, cbytes), dtype=torch.uint8, device=dev)

            def cub_sort():
                assert cub.cub_sort_pairs(ck_in.data_ptr(), ck_out.data_ptr(), cv_in.data_ptr(), cv_out.data_ptr(),
                                          n, bits, cscratch.data_ptr(), cbytes, stream) == 0

            cases.append(("cub_sort_pairs", cub_sort, 16 * n))
        for name, fn, byts in cases:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                fn()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            res[name] = {"us": us, "algorithmic_bytes": byts, "gbs": byts / (us * 1e-6) / 1e9,
                         "frac_of_hbm": byts / (us * 1e-6) / 1e9 / peak}
        torch.cuda.synchronize()
        assert int(flags[1].item()) == 0, "batch straddles a run"
        ref = np.lexsort((np.arange(n), rank, ex))
        assert np.array_equal(perm.cpu().numpy(), ref)
        if cub is not None:
            assert np.array_equal(cv_out.cpu().numpy(), ref), "CUB baseline order differs"
            res["k1_speedup_vs_cub"] = res["cub_sort_pairs"]["us"] / res["k1"]["us"]
        rows.append(res)
        print(json.dumps(res), flush=True)
    json.dump({"rows": rows, "hbm_peak_gbs": peak, "keys": dist}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
