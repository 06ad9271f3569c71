"""Multi-GPU loader: one process per GPU, NCCL and P2P (CUDA IPC) exchange,
every learner's delivered batch checked against the oracle.  Needs >= 2 GPUs
(skipped otherwise)."""
import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, exchange, dtype, out_dir, scheme="locality_balanced",
            host=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    import oracle
    from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, B, seed = 6000 * world, 192 * world, 42
    ld = DeviceLoader(LoaderConfig(d=d, learners=world, rank=rank, batch_size=B, seed=seed,
                                   data_seed=seed, exchange=exchange, scheme=scheme,
                                   augment=AugmentConfig(out_dtype=dtype)), device=rank)
    ld.populate()
    if exchange == "p2p":
        hs = [None] * world
        dist.all_gather_object(hs, ld.ipc_handle())
        ld.open_peers(hs)
    else:
        uid = [DeviceLoader.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ld.comm_init(uid[0])
    dist.barrier()
    order = oracle.permute_epoch(seed, 1, d)
    bad = []
    received = 0
    steps = [0, 1, 17, ld.steps_per_epoch - 1]
    if host:
        # host-driven path (ll_loader_submit_host / wait_host), two steps in
        # flight: the next step's plan is staged while the previous one runs
        host_ids = np.empty(B, np.uint64)
        ld.submit_host(1, steps[0], order[steps[0] * B:(steps[0] + 1) * B])
    for i, t in enumerate(steps):
        if host:
            if i + 1 < len(steps):
                n = steps[i + 1]
                ld.submit_host(1, n, order[n * B:(n + 1) * B])
            info = ld.wait_host(host_ids)
        else:
            info = ld.step(1, t)
        mode = (oracle.MODE_REGULAR if scheme == "regular" else oracle.MODE_LOCALITY_BALANCED)
        r = oracle.assign_step(order[t * B:(t + 1) * B], world, d, mode)
        lst = r["final_ids"][r["final_off"][rank]:r["final_off"][rank + 1]]
        got_ids = ld.fetch_ids(info)
        if host and not np.array_equal(host_ids[:info.n_local], lst):
            bad.append(f"step {t}: host ids differ")
            continue
        if not np.array_equal(got_ids, lst):
            bad.append(f"step {t}: ids differ")
            continue
        received += info.received
        got = ld.fetch(info)
        src = oracle.gen_samples(seed, lst, 256 * 256 * 3)
        for k, sid in enumerate(lst):
            want = oracle.augment(src[k].reshape(256, 256, 3), int(sid), seed, 1,
                                  bf16=dtype == "bf16")
            if not np.array_equal(got[k], want):
                bad.append(f"step {t} sample {k} (id {sid}, kept {info.kept})")
                break
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(f"received {received}\n" + "\n".join(bad))
    dist.barrier()
    ld.close()
    dist.destroy_process_group()


def _n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("exchange,dtype,scheme", [
    ("nccl", "fp32", "locality_balanced"), ("p2p", "fp32", "locality_balanced"),
    ("p2p", "bf16", "locality_balanced"),
    # reg_slice (sampling.cpp:27-42) at full volume: about half of every slice
    # comes from the other learner
    ("nccl", "bf16", "regular"), ("p2p", "fp32", "regular")])
def test_two_learners_exchange(tmp_path, exchange, dtype, scheme):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), exchange, dtype, str(tmp_path), scheme),
             nprocs=world, join=True)
    total_recv = 0
    for r in range(world):
        lines = open(tmp_path / f"rank{r}.txt").read().splitlines()
        total_recv += int(lines[0].split()[1])
        assert lines[1:] == [], lines[1:]
    assert total_recv > 0  # the steps really exercised the exchange


@pytest.mark.skipif(_n_gpus() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("exchange,scheme", [("p2p", "locality_balanced"),
                                             ("nccl", "locality_balanced"),
                                             ("nccl", "regular")])
def test_four_learners_exchange(tmp_path, exchange, scheme):
    """The same checks with four learners: moves between several peer pairs
    per step, every learner's batch against the oracle."""
    import torch.multiprocessing as mp
    world = 4
    mp.spawn(_worker, args=(world, _free_port(), exchange, "bf16", str(tmp_path), scheme),
             nprocs=world, join=True)
    total_recv = 0
    for r in range(world):
        lines = open(tmp_path / f"rank{r}.txt").read().splitlines()
        total_recv += int(lines[0].split()[1])
        assert lines[1:] == [], lines[1:]
    assert total_recv > 0


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("exchange,scheme", [("nccl", "locality_balanced"),
                                             ("nccl", "regular"),
                                             ("p2p", "locality_balanced")])
def test_two_learners_host_path(tmp_path, exchange, scheme):
    """The reference-facing host call (GlobalBatch from host memory, two steps
    in flight) with the exchange: same outputs as the device-driven steps."""
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), exchange, "bf16", str(tmp_path), scheme, True),
             nprocs=world, join=True)
    total_recv = 0
    for r in range(world):
        lines = open(tmp_path / f"rank{r}.txt").read().splitlines()
        total_recv += int(lines[0].split()[1])
        assert lines[1:] == [], lines[1:]
    assert total_recv > 0
