"""N > 1 host logic on CPU: two processes over torch.distributed (gloo).

Each rank plans the same steps independently (the replicated plan,
sampling.hpp:11-14 -- here from the oracle, as the device plan equals it bit
for bit, tests/test_gpu_parity.py), asks the library's exchange planner
(ll_exchange_plan: pure host code of liblocload_b200.so, the same function the
loader uses before its NCCL calls) which sends/receives it owns, performs them
over gloo with sample bytes from its own shard, and assembles its final list:
kept samples from the shard + received ones in buffer order.  Every assembled
sample must be the right sample.  Also checks that the ranks agree on the plan
without communicating (digest all-gather) and the max-over-ranks timing rule.
"""
import ctypes as C
import hashlib
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAMPLE = 3 * 16 * 16  # small synthetic samples keep the test in seconds


def _rdzv(tmp_path) -> str:
    """A fresh file:// rendezvous for torch.distributed (no TCP port to race
    for between tests)."""
    import uuid
    return "file://" + str(tmp_path / f"rdzv_{uuid.uuid4().hex}")


def _worker(rank, world, rdzv, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import oracle
    from paper_1910_01196_b200 import _capi

    dist.init_process_group("gloo", init_method=rdzv, rank=rank, world_size=world)
    d, B, seed = 4000, 200, 7
    cached = d
    first = oracle.owned_begin(rank, world, cached)
    last = oracle.owned_begin(rank + 1, world, cached)
    shard = {s: oracle.gen_sample(seed, s, SAMPLE) for s in range(first, last)}
    order = oracle.permute_epoch(seed, 3, d)
    errors = []
    digests = []
    moved = 0
    for t in range(d // B):
        r = oracle.assign_step(order[t * B:(t + 1) * B], world, cached,
                               oracle.MODE_LOCALITY_BALANCED)
        digests.append(hashlib.sha256(r["final_ids"].tobytes()).hexdigest())
        mv = (_capi.Move * max(len(r["moves"]), 1))()
        for i, m in enumerate(r["moves"]):
            mv[i].sender, mv[i].receiver, mv[i].count = m[0], m[1], m[2]
            mv[i].src_off, mv[i].dst_off = m[3], m[4]
        off = np.ascontiguousarray(r["final_off"], dtype=np.uint64)
        xs = (_capi.Xfer * (2 * world))()
        nx = C.c_uint32()
        _capi.check(_capi.lib().ll_exchange_plan(mv, len(r["moves"]),
                                                 _capi.ptr(off, C.c_uint64), world, rank, xs,
                                                 C.byref(nx)))
        final = r["final_ids"]
        kept = int(r["kept"][rank])
        n_local = int(off[rank + 1] - off[rank])
        recv = torch.zeros((n_local - kept, SAMPLE), dtype=torch.uint8)
        reqs = []
        for x in xs[:nx.value]:
            if x.is_send:
                ids = final[x.list_first:x.list_first + x.count]
                buf = torch.from_numpy(np.stack([shard[int(s)] for s in ids]))
                reqs.append(dist.isend(buf, dst=int(x.peer)))
            else:
                view = recv[x.buf_first:x.buf_first + x.count]
                tmp = torch.zeros_like(view)
                reqs.append((dist.irecv(tmp, src=int(x.peer)), view, tmp))
                moved += x.count
        for q in reqs:
            if isinstance(q, tuple):
                q[0].wait()
                q[1].copy_(q[2])
            else:
                q.wait()
        mine = final[off[rank]:off[rank + 1]]
        for k, s in enumerate(mine):
            got = shard[int(s)] if k < kept else recv[k - kept].numpy()
            if not np.array_equal(got, oracle.gen_sample(seed, int(s), SAMPLE)):
                errors.append(f"step {t} slot {k} id {int(s)}")
                break
    # ranks agree on every step's plan without having exchanged it
    all_digests = [None] * world
    dist.all_gather_object(all_digests, digests)
    agree = all(dg == digests for dg in all_digests)
    # max-over-ranks timing reduction used by bench.py
    v = torch.tensor([float(rank + 1)])
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(f"{moved} {int(agree)} {v.item()}\n" + "\n".join(errors))
    dist.destroy_process_group()


def test_two_rank_exchange_over_gloo(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _rdzv(tmp_path), str(tmp_path)), nprocs=world, join=True)
    total = 0
    for r in range(world):
        lines = open(tmp_path / f"rank{r}.txt").read().splitlines()
        moved, agree, vmax = lines[0].split()
        assert lines[1:] == [], lines[1:]
        assert agree == "1"
        assert float(vmax) == world
        total += int(moved)
    assert total > 0
