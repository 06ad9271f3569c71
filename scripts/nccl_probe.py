"""NCCL send/recv bandwidth between the GPUs of one box, alone (no augment
running): each rank exchanges `mb` MB with every other rank in one grouped
send/recv, as the cfg4 exchange does.  Measurement aid for DESIGN.md 8.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      scripts/nccl_probe.py [mb ...]
"""
import json
import os
import sys

import torch
import torch.distributed as dist

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
for mb in [float(x) for x in sys.argv[1:]] or [10.0, 40.0, 80.0, 160.0]:
    n = int(mb * 1e6)
    send = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(world)]
    recv = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(world)]

    def once():
        ops = []
        for r in range(world):
            if r == rank:
                continue
            ops.append(dist.P2POp(dist.isend, send[r], r))
            ops.append(dist.P2POp(dist.irecv, recv[r], r))
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    for _ in range(5):
        once()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 30
    e0.record()
    for _ in range(it):
        once()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / it
    gbs = n * (world - 1) / (ms / 1e3) / 1e9  # received bytes per GPU per second
    t = torch.tensor([gbs], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": world, "mb_per_peer": mb, "ms": ms,
                          "recv_gbs_per_gpu": float(t.item())}), flush=True)
dist.destroy_process_group()
