"""Host-path probe over NCCL (torchrun, N ranks, cfg2 shapes): per-call host
time of submit_host / wait_host at prefetch depth 4.  Measurement aid only."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import paper_1910_01196_b200 as ll  # noqa: E402
from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
d, B, seed = 160_000 * world, 1024 * world, 42
ld = DeviceLoader(LoaderConfig(d=d, learners=world, rank=rank, batch_size=B, seed=seed,
                               data_seed=seed, exchange="nccl", prefetch_depth=4,
                               augment=AugmentConfig(out_dtype="fp32")), device=rank)
ld.populate()
uid = [DeviceLoader.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
ld.comm_init(uid[0])
order = ll.permute_epoch(seed, 1, d).order
ids = np.empty(B, np.uint64)
for s in range(8):
    ld.submit_host(1, s, order[s * B:(s + 1) * B])
    ld.wait_host(ids)
dist.barrier()
n, depth = 120, 4
ts, tw = [], []
out = 0
t0 = time.perf_counter()
for s in range(n):
    a = time.perf_counter()
    ld.submit_host(1, s, order[s * B:(s + 1) * B])
    ts.append(time.perf_counter() - a)
    out += 1
    if out == depth:
        a = time.perf_counter()
        ld.wait_host(ids)
        tw.append(time.perf_counter() - a)
        out -= 1
while out:
    ld.wait_host(ids)
    out -= 1
wall = time.perf_counter() - t0
print(f"rank {rank}: {n * B / world / wall / 1e6:.2f} M samples/s/GPU, us/step {wall / n * 1e6:.1f}, "
      f"submit median {np.median(ts) * 1e6:.1f} us p90 {np.percentile(ts, 90) * 1e6:.1f}, "
      f"wait median {np.median(tw) * 1e6:.1f} us", flush=True)
dist.barrier()
ld.close()
