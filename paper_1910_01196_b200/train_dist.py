"""Distributed consumer: synchronous SGD with one (or more) learners per
process and a gradient all-reduce across the processes.

The reference simulates p learners in one thread (run_training,
proj/src/equivalence.cpp:95-174).  Here each process of a torch.distributed
group plays p / world of them: every step it takes its learners' lists from
the replicated device plan (ll_plan_epoch -- the loader's K2+K3 permutation
and K4 assignment), computes their per-sample gradients on its GPU, and the
processes combine them with a gradient all-reduce before the identical update
w -= lr * g on every rank.

Aggregation (equivalence.hpp:40-48):
  * "canonical": per-sample gradients are all-gathered with their sample ids
    and summed in ascending id on every rank (equivalence.cpp:132-143) --
    the deterministic all-reduce; bit-identical to the reference;
  * "learner_order": each learner's list is summed in list order, the
    per-learner partials are all-gathered and summed in learner order
    (:144-155) -- also bit-identical;
  * "allreduce": per-process partials combined by one NCCL all_reduce(SUM):
    the production collective, whose summation order NCCL chooses, so the
    trajectory matches the reference only up to rounding (the reference's
    learner_order comment: "like a real all-reduce").

The sums in a prescribed order run on the device (ll_ordered_sum_device,
one thread per coordinate, IEEE-rounded adds in that order); the collectives
are torch.distributed's (NCCL on GPUs, gloo on CPU for the host-logic tests).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import _capi
from ._capi import InvalidArgument, check
from .locload import SchemeKind, ToyObjective, TrainingRun, context, plan_epoch

AGGREGATIONS = ("canonical", "learner_order", "allreduce")


class DeviceOps:
    """The per-rank compute of a step on this process's GPU (C-ABI kernels on
    torch tensors, issued on the library context's stream, which is torch's
    current stream while the trainer runs)."""

    def __init__(self, obj: ToyObjective, device: int):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.ctx = context(device)
        sp = C.c_size_t()
        check(_capi.lib().ll_ctx_stream(self.ctx, C.byref(sp)))
        self.stream = torch.cuda.ExternalStream(sp.value, device=self.device)
        with torch.cuda.stream(self.stream):
            self.xs = torch.as_tensor(np.ascontiguousarray(obj.xs, np.float64)).to(self.device)
            self.ys = torch.as_tensor(np.ascontiguousarray(obj.ys, np.float64)).to(self.device)
        self.dims = obj.dims()
        self._plans = {}

    def zeros(self, *shape):
        return self.torch.zeros(*shape, dtype=self.torch.float64, device=self.device)

    def lists(self, seed: int, epoch: int, n: int, p: int, B: int, scheme: str,
              step: int) -> List[np.ndarray]:
        key = (seed, epoch, n, p, B, scheme)
        if key not in self._plans:
            self._plans = {key: plan_epoch(seed, epoch, n, p, B, scheme=scheme,
                                           device=self.device.index)}
        return self._plans[key].lists(step)

    def ids(self, ids: np.ndarray):
        return self.torch.as_tensor(np.ascontiguousarray(ids, np.int64)).to(self.device)

    def grads(self, w, ids):
        m = int(ids.numel())
        G = self.torch.empty((m, self.dims), dtype=self.torch.float64, device=self.device)
        if m:
            check(_capi.lib().ll_toy_grads_device(self.ctx, self.xs.data_ptr(),
                                                  self.ys.data_ptr(), self.dims, w.data_ptr(),
                                                  ids.data_ptr(), m, G.data_ptr()))
        return G

    def ordered_sum(self, G, order=None):
        out = self.torch.empty(self.dims, dtype=self.torch.float64, device=self.device)
        check(_capi.lib().ll_ordered_sum_device(self.ctx, G.data_ptr(), int(G.shape[0]),
                                                self.dims,
                                                0 if order is None else order.data_ptr(),
                                                out.data_ptr()))
        return out

    def apply(self, gsum, scale: float, lr: float, w):
        g = self.torch.empty(self.dims, dtype=self.torch.float64, device=self.device)
        check(_capi.lib().ll_sgd_apply_device(self.ctx, gsum.data_ptr(), self.dims, scale, lr,
                                              w.data_ptr(), g.data_ptr()))
        return g

    def argsort(self, ids):
        return self.torch.argsort(ids, stable=True)

    def host(self, t) -> np.ndarray:
        return t.cpu().numpy()

    def stream_ctx(self):
        return self.torch.cuda.stream(self.stream)


class DistributedTrainer:
    """run_training with the learners spread over a torch.distributed group:
    process r plays learners [r * p/world, (r+1) * p/world).  Every rank ends
    with the same weights; under canonical and learner_order aggregation they
    equal the reference's run_training bit for bit."""

    def __init__(self, obj: ToyObjective, scheme: str, p: int, batch_size: int, seed: int,
                 learning_rate: float, aggregation: str = "canonical", group=None,
                 device: Optional[int] = None, ops=None):
        import torch.distributed as dist
        if scheme not in SchemeKind:
            raise InvalidArgument(f"run_training: unknown scheme {scheme!r}")
        if aggregation not in AGGREGATIONS:
            raise InvalidArgument(f"run_training: unknown aggregation {aggregation!r}")
        if p == 0:
            raise InvalidArgument("run_training: need at least one learner")
        n = obj.samples()
        if batch_size == 0 or batch_size > n:
            raise InvalidArgument("run_training: batch size must be in [1, n]")
        if scheme == "regular" and batch_size % p:
            raise InvalidArgument("reg_slice: learner count must divide the batch size")
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        if p % self.world:
            raise InvalidArgument("DistributedTrainer: the learner count must be a multiple "
                                  "of the process count")
        per = p // self.world
        self.mine = list(range(self.rank * per, (self.rank + 1) * per))
        self.obj, self.scheme, self.p, self.B = obj, scheme, p, batch_size
        self.seed, self.lr, self.agg = seed, learning_rate, aggregation
        if ops is None:
            import torch
            ops = DeviceOps(obj, torch.cuda.current_device() if device is None else device)
        self.ops = ops

    # -- collectives ---------------------------------------------------------
    def _all_gather_rows(self, t):
        """All-gather a [rows][...] tensor with rows varying per rank."""
        import torch
        if self.world == 1:
            return t
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        counts = [int(x.item()) for x in ns]
        mx = max(counts)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        outs = [torch.zeros_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return torch.cat([o[:c] for o, c in zip(outs, counts)])

    # -- one step ------------------------------------------------------------
    def step_gradient(self, w, lists: List[np.ndarray]):
        """The aggregated (unnormalised) gradient of one global batch."""
        ops = self.ops
        if self.agg == "canonical":
            ids = ops.ids(np.concatenate([lists[j] for j in self.mine]) if self.mine else
                          np.zeros(0, np.int64))
            G = ops.grads(w, ids)
            all_ids = self._all_gather_rows(ids)
            all_G = self._all_gather_rows(G)
            return ops.ordered_sum(all_G, ops.argsort(all_ids))
        import torch
        partials = [ops.ordered_sum(ops.grads(w, ops.ids(lists[j]))) for j in self.mine]
        if self.agg == "learner_order":
            P = torch.stack(partials)
            return ops.ordered_sum(self._all_gather_rows(P))
        mine = ops.ordered_sum(torch.stack(partials))
        if self.world > 1:
            self.dist.all_reduce(mine, op=self.dist.ReduceOp.SUM, group=self.group)
        return mine

    def run(self, steps: int) -> TrainingRun:
        """steps of synchronous SGD from w = 0 (equivalence.cpp:113-172)."""
        ops = self.ops
        n = self.obj.samples()
        spe = n // self.B
        with ops.stream_ctx():
            w = ops.zeros(self.obj.dims())
            grads = []
            for t in range(steps):
                epoch, st = divmod(t, spe)
                lists = ops.lists(self.seed, epoch, n, self.p, self.B, self.scheme, st)
                gsum = self.step_gradient(w, lists)
                grads.append(ops.apply(gsum, 1.0 / float(self.B), self.lr, w))
            final = ops.host(w)
            sg = np.stack([ops.host(g) for g in grads]) if grads else \
                np.zeros((0, self.obj.dims()))
        return TrainingRun(final, sg)
