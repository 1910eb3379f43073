"""Worker for tests/test_gpu_serving.py::test_fused_hops_across_processes_ipc (one rank).

Serves the trimmed config-4 plan as executor RANK of 2 with fused peer hops whose buffers
were exchanged as CUDA IPC handles, two steps, and saves the final outputs of the requests
that finish on this rank to <dir>/rank<RANK>.npz.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_02354_b200 import configs, engine, runtime  # noqa: E402


PEER_TIER = {"read_bandwidth_bytes_per_s": 720e9, "fixed_load_overhead_s": 1e-5}


def workload(mode: str, world: int):
    """"hops": config 4 (240 requests); "peer": config 5 (300 requests) with the peer-GPU tier."""
    name, n = ("c5", 300) if mode == "peer" else ("c4", 240)
    w = configs.load(name, 1000, gpu_executors=world)
    w.stream = w.stream[:n]
    w.docs = dict(w.docs, stream={"schema_version": 1, "requests": w.docs["stream"]["requests"][:n]})
    kw = {"peer_tier": PEER_TIER} if mode == "peer" else {}
    return w, engine.plan(configs.run_config(w, trace=False, **kw))


def main(out_dir: str, mode: str = "hops") -> None:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w, plan = workload(mode, world)
    shape = runtime.RuntimeShape(1024, 2048, 64)
    rt = runtime.B200Runtime.for_plan(plan, shape, executor=rank)
    n = len(plan.resolved.request_ids)
    rt.fill_inputs(n)
    rt.attach_peers_ipc(rank, world)
    dist.barrier()
    chains = plan.resolved.chains
    mine = sorted({r for _e, members in runtime.batches_from_plan(plan, executor=rank)
                   for r, s in members if s == len(chains[r]) - 1})
    outs, peer = [], []
    for _ in range(3 if mode == "peer" else 2):
        st = rt.step(plan, rank)
        peer.append((st["peer_loads"], st["peer_tier_loads"]))
        rt.synchronize()
        host = torch.empty(n * shape.T * shape.d, dtype=torch.bfloat16).pin_memory()
        rt.download_outputs(runtime.last_stages(plan), host.data_ptr())
        rt.synchronize()
        outs.append(host.view(n, shape.T, shape.d).float().numpy()[mine].copy())
        dist.barrier()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), requests=np.array(mine, np.int64), outputs=np.stack(outs),
             peer=np.array(peer, np.int64))
    dist.barrier()
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "hops")
