"""Multi-GPU loader: one process per GPU, NCCL and P2P (CUDA IPC) exchange,
every learner's delivered batch checked against the oracle.  Needs >= 2 GPUs
(skipped otherwise)."""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _rdzv(tmp_path) -> str:
    """A fresh file:// rendezvous for torch.distributed (no TCP port to race
    for between tests)."""
    import uuid
    return "file://" + str(tmp_path / f"rdzv_{uuid.uuid4().hex}")


def _worker(rank, world, rdzv, exchange, dtype, out_dir, scheme="locality_balanced",
            host=False, opts=None):
    """opts: alpha (storage tier for ids >= alpha*d), hw (fixed source
    geometry, default 256x256), variable (cfg5 geometry, resize mode)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import oracle
    from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig
    opts = opts or {}
    alpha = opts.get("alpha", 1.0)
    H, W = opts.get("hw", (256, 256))
    variable = opts.get("variable", False)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method=rdzv, rank=rank, world_size=world)
    d, B, seed = opts.get("d_per", 6000) * world, opts.get("b_per", 192) * world, 42
    aug = AugmentConfig(mode="resize" if variable else "crop", out_dtype=dtype)
    ld = DeviceLoader(LoaderConfig(d=d, height=H, width=W, learners=world, rank=rank,
                                   batch_size=B, alpha=alpha, seed=seed, data_seed=seed,
                                   exchange=exchange, scheme=scheme,
                                   geometry="variable" if variable else "fixed", augment=aug),
                      device=rank)
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
    cached = oracle.cached_count(d, alpha)
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
        r = oracle.assign_step(order[t * B:(t + 1) * B], world, cached, mode)
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
        for k, sid in enumerate(lst):
            if variable:
                h, w = oracle.sample_hw(seed, int(sid))
                src = oracle.gen_sample(seed, int(sid), h * w * 3).reshape(h, w, 3)
                want = oracle.augment(src, int(sid), seed, 1, mode=oracle.AUG_RESIZE,
                                      bf16=dtype == "bf16")
            else:
                src = oracle.gen_sample(seed, int(sid), H * W * 3).reshape(H, W, 3)
                want = oracle.augment(src, int(sid), seed, 1, bf16=dtype == "bf16")
            if not np.array_equal(got[k], want):
                bad.append(f"step {t} sample {k} (id {sid}, kept {info.kept})")
                break
    xs = ld.exchange_stats() if exchange == "nccl" else {}
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(f"received {received} wire {xs.get('bytes_recv', 0)}\n" + "\n".join(bad))
    dist.barrier()
    ld.close()
    dist.destroy_process_group()


def _run(tmp_path, world, exchange, dtype, scheme="locality_balanced", host=False, opts=None):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _rdzv(tmp_path), exchange, dtype, str(tmp_path), scheme, host,
                            opts), nprocs=world, join=True)
    total_recv = wire = 0
    for r in range(world):
        lines = open(tmp_path / f"rank{r}.txt").read().splitlines()
        head = lines[0].split()
        total_recv += int(head[1])
        wire += int(head[3])
        assert lines[1:] == [], lines[1:]
    assert total_recv > 0  # the steps really exercised the exchange
    return total_recv, wire


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
    _run(tmp_path, 2, exchange, dtype, scheme)


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("scheme,register", [("locality_balanced", "1"), ("regular", "0")])
def test_two_learners_nccl_buffer_kinds(tmp_path, monkeypatch, scheme, register):
    """The NCCL exchange on the buffer kind its scheme does not use by default
    (comm_init: registered ncclMemAlloc buffers for the regular scheme,
    cudaMalloc for the balanced one; LL_NCCL_REGISTER forces either): same
    outputs against the oracle."""
    monkeypatch.setenv("LL_NCCL_REGISTER", register)
    _run(tmp_path, 2, "nccl", "bf16", scheme)


@pytest.mark.skipif(_n_gpus() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("exchange,scheme", [("p2p", "locality_balanced"),
                                             ("nccl", "locality_balanced"),
                                             ("nccl", "regular")])
def test_four_learners_exchange(tmp_path, exchange, scheme):
    """The same checks with four learners: moves between several peer pairs
    per step, every learner's batch against the oracle."""
    _run(tmp_path, 4, exchange, "bf16", scheme)


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("exchange,scheme,opts", [
    ("nccl", "locality_balanced", None), ("nccl", "regular", None),
    ("p2p", "locality_balanced", None),
    ("nccl", "locality_balanced", {"alpha": 0.5}), ("nccl", "regular", {"alpha": 0.5}),
    ("nccl", "locality_balanced", {"variable": True, "d_per": 3000, "b_per": 128})],
    ids=["nccl-bal", "nccl-reg", "p2p-bal", "nccl-bal-storage", "nccl-reg-storage",
         "nccl-bal-variable"])
def test_two_learners_host_path(tmp_path, exchange, scheme, opts):
    """The reference-facing host call (GlobalBatch from host memory, two steps
    in flight) with the exchange: same outputs as the device-driven steps,
    also with the storage tier and with variable-size sources over NCCL."""
    _run(tmp_path, 2, exchange, "bf16", scheme, host=True, opts=opts)


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("exchange,scheme", [("nccl", "locality_balanced"),
                                             ("nccl", "regular"),
                                             ("p2p", "locality_balanced")])
def test_two_learners_storage_tier(tmp_path, exchange, scheme):
    """alpha = 0.5 (cfg3 at p = 2): half of the ids are uncached and read from
    every learner's storage tier; over NCCL only the moved cached samples
    cross the wire (a move's run hands cached samples over first)."""
    _run(tmp_path, 2, exchange, "fp32", scheme, opts={"alpha": 0.5})


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_two_learners_variable_resize(tmp_path, exchange):
    """cfg5 over both exchanges: variable-size sources, bilinear resize to
    224, bf16; NCCL messages carry each moved sample's resize window."""
    recv, wire = _run(tmp_path, 2, exchange, "bf16",
                      opts={"variable": True, "d_per": 3000, "b_per": 128})
    if exchange == "nccl":
        assert wire > 0


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("hw", [(224, 224), (232, 224), (250, 250)])
def test_two_learners_nccl_small_sources(tmp_path, hw):
    """Sources whose whole sample is smaller than a crop-window message slot
    (224 x 224, 232 x 224): the exchange buffers are sized by the slot at
    comm_init and never grow on the step path."""
    _run(tmp_path, 2, "nccl", "fp32", "locality_balanced", opts={"hw": hw})
    _run(tmp_path, 2, "nccl", "bf16", "regular", opts={"hw": hw})


def _train_worker(rank, world, rdzv, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_1910_01196_b200 import locload as ll
    from paper_1910_01196_b200.train_dist import DistributedTrainer
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=rdzv, rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    obj = ll.ToyObjective.synthesize(4096, 16, 7)
    for i, (scheme, agg) in enumerate([("locality_balanced", "canonical"),
                                       ("regular", "learner_order"),
                                       ("locality", "canonical"),
                                       ("locality_balanced", "allreduce")]):
        run = DistributedTrainer(obj, scheme, 2 * world, 512, 4, 0.001,
                                 aggregation=agg, device=rank).run(24)
        np.save(os.path.join(out_dir, f"w{i}_{rank}.npy"), run.final_weights)
        np.save(os.path.join(out_dir, f"g{i}_{rank}.npy"), run.step_gradients)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs")
def test_distributed_trainer_nccl_vs_reference(tmp_path):
    """The gradient all-reduce across GPUs (NCCL all-gather + ordered device
    sums): every rank ends with the reference's run_training weights and step
    gradients bit for bit under canonical and learner_order aggregation
    (equivalence.cpp:132-148); NCCL all_reduce(SUM) agrees to rounding."""
    import torch.multiprocessing as mp
    import oracle
    world = 2
    mp.spawn(_train_worker, args=(world, _rdzv(tmp_path), str(tmp_path)), nprocs=world, join=True)
    for i, (scheme, agg) in enumerate([("locality_balanced", "canonical"),
                                       ("regular", "learner_order"),
                                       ("locality", "canonical"),
                                       ("locality_balanced", "allreduce")]):
        ref_agg = "canonical" if agg == "canonical" else "learner_order"
        w, g = oracle.ref_run_training(4096, 16, 7, scheme, 2 * world, 512, 24, 4, 0.001,
                                       ref_agg)
        ws = [np.load(tmp_path / f"w{i}_{r}.npy") for r in range(world)]
        assert np.array_equal(ws[0], ws[1])
        if agg == "allreduce":
            np.testing.assert_allclose(ws[0], w, rtol=1e-12, atol=1e-15)
        else:
            assert np.array_equal(ws[0], w), (scheme, agg)
            assert np.array_equal(np.load(tmp_path / f"g{i}_0.npy"), g), (scheme, agg)
