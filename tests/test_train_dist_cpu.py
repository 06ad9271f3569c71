"""Gradient all-reduce of the distributed consumer, host logic on CPU.

Two processes over torch.distributed (gloo), each playing half of the p
learners of run_training (equivalence.cpp:95-174) through
paper_1910_01196_b200.train_dist.DistributedTrainer.  The per-rank compute
(plan lists, per-sample gradients, ordered sums, update) comes from the
oracle here -- the reference's own sample_gradient, the C oracle's
assignment and a sequential numpy sum -- because there is no GPU; the
trainer's collectives and ordering rules are what is under test.  Under
canonical and learner_order aggregation every rank must end with the
reference's weights and step gradients bit for bit (equivalence.cpp:132-148);
under the NCCL-style all-reduce they agree to rounding.  The device kernels
behind the same protocol are covered by tests/test_gpu_train.py.
"""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, DIMS, OBJ_SEED, SEED, LR = 640, 6, 3, 11, 0.05


def _rdzv(tmp_path) -> str:
    """A fresh file:// rendezvous for torch.distributed (no TCP port to race
    for between tests)."""
    import uuid
    return "file://" + str(tmp_path / f"rdzv_{uuid.uuid4().hex}")


class RefOps:
    """CPU stand-in for DeviceOps: same interface, reference arithmetic."""

    def __init__(self, obj_seed, dims, n):
        import torch
        self.torch, self.obj_seed, self.dims, self.n = torch, obj_seed, dims, n
        self._orders = {}

    def zeros(self, *shape):
        return self.torch.zeros(*shape, dtype=self.torch.float64)

    def lists(self, seed, epoch, n, p, B, scheme, step):
        import oracle
        if (seed, epoch) not in self._orders:
            self._orders = {(seed, epoch): oracle.ref_permute_epoch(seed, epoch, n)}
        batch = self._orders[(seed, epoch)][step * B:(step + 1) * B]
        mode = {"regular": oracle.MODE_REGULAR, "locality": oracle.MODE_LOCALITY,
                "locality_balanced": oracle.MODE_LOCALITY_BALANCED}[scheme]
        r = oracle.assign_step(batch, p, n, mode)
        return [r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]] for j in range(p)]

    def ids(self, ids):
        return self.torch.as_tensor(np.ascontiguousarray(ids, np.int64))

    def grads(self, w, ids):
        import oracle
        G = np.zeros((int(ids.numel()), self.dims))
        for i, s in enumerate(ids.tolist()):
            G[i] = oracle.ref_sample_gradient(self.n, self.dims, self.obj_seed, w.numpy(), s)[0]
        return self.torch.as_tensor(G)

    def ordered_sum(self, G, order=None):
        g = np.zeros(self.dims)
        rows = G.numpy()
        for r in (range(rows.shape[0]) if order is None else order.tolist()):
            g = g + rows[r]  # one IEEE add per coordinate, in this order
        return self.torch.as_tensor(g)

    def apply(self, gsum, scale, lr, w):
        g = gsum.numpy() * scale
        w.copy_(self.torch.as_tensor(w.numpy() - lr * g))
        return self.torch.as_tensor(g)

    def argsort(self, ids):
        return self.torch.argsort(ids, stable=True)

    def host(self, t):
        return t.numpy().copy()

    def stream_ctx(self):
        import contextlib
        return contextlib.nullcontext()


def _worker(rank, world, rdzv, cases, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_1910_01196_b200.locload import ToyObjective
    from paper_1910_01196_b200.train_dist import DistributedTrainer
    dist.init_process_group("gloo", init_method=rdzv, rank=rank, world_size=world)
    obj = ToyObjective.synthesize(N, DIMS, OBJ_SEED)  # host-only library call
    for i, (scheme, agg, p, B, steps) in enumerate(cases):
        tr = DistributedTrainer(obj, scheme, p, B, SEED, LR, aggregation=agg,
                                ops=RefOps(OBJ_SEED, DIMS, N))
        run = tr.run(steps)
        np.save(os.path.join(out_dir, f"w_{i}_{rank}.npy"), run.final_weights)
        np.save(os.path.join(out_dir, f"g_{i}_{rank}.npy"), run.step_gradients)
    dist.barrier()
    dist.destroy_process_group()


CASES = [("locality_balanced", "canonical", 4, 64, 14), ("locality", "canonical", 2, 48, 14),
         ("regular", "canonical", 2, 64, 12), ("locality_balanced", "learner_order", 4, 64, 14),
         ("regular", "learner_order", 2, 32, 22), ("locality_balanced", "allreduce", 2, 64, 12)]


def test_distributed_sgd_matches_reference(tmp_path, ref_lib):
    import oracle
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _rdzv(tmp_path), CASES, str(tmp_path)), nprocs=world, join=True)
    for i, (scheme, agg, p, B, steps) in enumerate(CASES):
        ref_agg = "canonical" if agg == "canonical" else "learner_order"
        want_w, want_g = oracle.ref_run_training(N, DIMS, OBJ_SEED, scheme, p, B, steps, SEED,
                                                 LR, ref_agg)
        ws = [np.load(tmp_path / f"w_{i}_{r}.npy") for r in range(world)]
        gs = [np.load(tmp_path / f"g_{i}_{r}.npy") for r in range(world)]
        for r in range(world):  # every rank holds the same model
            assert np.array_equal(ws[r], ws[0]) and np.array_equal(gs[r], gs[0])
        if agg == "allreduce":
            np.testing.assert_allclose(ws[0], want_w, rtol=1e-12, atol=1e-15)
        else:
            assert np.array_equal(ws[0], want_w), (scheme, agg)
            assert np.array_equal(gs[0], want_g), (scheme, agg)


def test_trainer_argument_errors():
    from paper_1910_01196_b200._capi import InvalidArgument
    from paper_1910_01196_b200.locload import ToyObjective
    from paper_1910_01196_b200.train_dist import DistributedTrainer
    obj = ToyObjective.synthesize(100, 3, 1)
    ops = RefOps(1, 3, 100)
    with pytest.raises(InvalidArgument, match="batch size must be in"):
        DistributedTrainer(obj, "locality", 2, 0, 1, 0.1, ops=ops)
    with pytest.raises(InvalidArgument, match="need at least one learner"):
        DistributedTrainer(obj, "locality", 0, 10, 1, 0.1, ops=ops)
    with pytest.raises(InvalidArgument, match="learner count must divide"):
        DistributedTrainer(obj, "regular", 3, 10, 1, 0.1, ops=ops)
    with pytest.raises(InvalidArgument, match="unknown aggregation"):
        DistributedTrainer(obj, "regular", 2, 10, 1, 0.1, aggregation="mean", ops=ops)
