"""World-size-2 CPU test (gloo) of the multi-GPU path's host protocol.

Each rank runs the same deterministic planner (no control traffic), executes
only its executor's batches, and exchanges hopped activations point-to-point
in the global hop order (coe_plan_hops, hops.h) -- the protocol the CUDA
runtime follows over NCCL.  Activations are tiny numpy MLPs (oracle.mlp) so
the test checks ordering, deadlock-freedom and data correctness: every
request's final output equals a single-process chain forward.
"""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

D, H, T = 64, 128, 4
SEED = 7


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup_plan(world, n_req):
    from paper_2503_02354_b200 import configs, engine

    w = configs.load("c4", 1000, gpu_executors=world)
    w.stream = w.stream[:n_req]
    return engine.plan(configs.run_config(w, trace=False))


def _weights(e):
    from oracle import synth

    return synth.expert_weights(SEED, e, D, H)


def _worker(rank, world, port, n_req, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mlp, synth
        from paper_2503_02354_b200 import runtime

        plan = _setup_plan(world, n_req)
        raw = plan.ops().tobytes() + plan.op_args().tobytes() + plan.admissions().tobytes()
        digest = torch.tensor([int.from_bytes(hashlib.sha256(raw).digest()[:7], "big")], dtype=torch.int64)
        gathered = [torch.zeros_like(digest) for _ in range(world)]
        dist.all_gather(gathered, digest)
        assert all(int(g) == int(digest) for g in gathered), "ranks planned differently"

        hops = runtime.hops_from_plan(plan)
        mine = [h for h in hops if h[1] == rank or h[2] == rank]
        # activation store: output of (request, stage) held on this rank
        act = {}
        cursor = 0

        def run_hops(limit):
            nonlocal cursor
            while cursor < len(mine) and mine[cursor][0] <= limit:
                _idx, src, dst, req, stage = mine[cursor]
                if src == rank:
                    dist.send(torch.from_numpy(act[(req, stage)]), dst=dst)
                else:
                    buf = torch.empty(T, D, dtype=torch.float32)
                    dist.recv(buf, src=src)
                    act[(req, stage)] = buf.numpy()
                cursor += 1

        incoming = {(h[3], h[4] + 1): h[0] for h in mine if h[2] == rank}
        for expert, members in runtime.batches_from_plan(plan, executor=rank):
            need = [incoming[(r, s)] for r, s in members if (r, s) in incoming]
            if need:
                run_hops(max(need))
            w1, w2 = _weights(expert)
            xs = np.concatenate([synth.request_inputs(SEED, r, T, D) if s == 0 else act[(r, s - 1)]
                                 for r, s in members])
            ys = mlp.expert_forward(xs, w1, w2)
            for k, (r, s) in enumerate(members):
                act[(r, s)] = ys[k * T:(k + 1) * T]
        run_hops(1 << 62)
        assert cursor == len(mine)
        chains = plan.resolved.chains
        finals = {r: act[(r, len(chains[r]) - 1)] for r in range(len(chains)) if (r, len(chains[r]) - 1) in act}
        np.save(result_path.format(rank=rank), np.array([finals], dtype=object), allow_pickle=True)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_ranks_exchange_hops_and_match_single_process(tmp_path, world):
    from oracle import mlp, synth

    n_req = 160
    plan = _setup_plan(world, n_req)
    from paper_2503_02354_b200 import runtime

    hops = runtime.hops_from_plan(plan)
    assert len(hops) > 0, "config must exercise cross-executor hops"
    path = str(tmp_path / "out_{rank}.npy")
    mp.start_processes(_worker, args=(world, _free_port(), n_req, path), nprocs=world, join=True,
                       start_method="spawn")
    finals = {}
    for r in range(world):
        finals.update(np.load(path.format(rank=r), allow_pickle=True)[0])
    chains = plan.resolved.chains
    assert sorted(finals) == list(range(len(chains)))
    for r in range(0, len(chains), 7):
        ref = mlp.chain_forward(synth.request_inputs(SEED, r, T, D), chains[r], _weights)
        assert mlp.rel_l2(finals[r], ref) < 1e-5
