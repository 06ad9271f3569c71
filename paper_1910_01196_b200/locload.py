"""Python mirror of the reference's locload API for the hot path, backed by the
B200 C-ABI (include/locload_b200.h).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/locload/{core,sampling,balance,pipeline}.hpp so
the parity tests read like the reference's own doctest suites.  Reference
std::invalid_argument -> InvalidArgument (a ValueError) with the reference's
message text; std::runtime_error -> RuntimeError.

Every function that is part of the hot path runs on the GPU (permute_epoch,
permutation_prefix, reg_slice, loc_distribution, balance, assign, plan_epoch
-- a whole epoch's plan, the sampler half of Loader::run_epoch -- and the
loader).
Pure closed forms that the reference itself defines inline in its headers
(CacheDirectory.owner, sampling.hpp:22-25) or as O(p) arithmetic (targets,
deficit_fraction, counts_with_uncached over an existing distribution) are
plain host code here too.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi
from ._capi import InvalidArgument, check, ptr

SampleId = int
LearnerId = int

_ctx_by_device: dict = {}


def context(device: int = 0) -> C.c_void_p:
    """Process-wide default ll_ctx for `device` (created lazily)."""
    h = _ctx_by_device.get(device)
    if h is None:
        h = C.c_void_p()
        check(_capi.lib().ll_ctx_create(C.byref(h), device))
        _ctx_by_device[device] = h
    return h


# ---------------------------------------------------------------- core.hpp
@dataclass
class EpochPermutation:  # core.hpp:13-17
    seed: int = 0
    epoch: int = 0
    order: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


@dataclass
class GlobalBatch:  # core.hpp:20-23
    step: int = 0
    samples: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


def permute_epoch(seed: int, epoch: int, d: int, device: int = 0) -> EpochPermutation:
    """core.hpp:25-28: Fisher-Yates over SplitMix64(derive_seed(seed, epoch))."""
    out = np.empty(max(d, 1), np.uint64)
    check(_capi.lib().ll_permute_epoch(context(device), seed, epoch, d, ptr(out, C.c_uint64)))
    return EpochPermutation(seed, epoch, out[:d])


def permutation_prefix(seed: int, epoch: int, d: int, k: int, device: int = 0) -> np.ndarray:
    """core.hpp:30-33."""
    out = np.empty(max(k, 1), np.uint64)
    check(_capi.lib().ll_permutation_prefix(context(device), seed, epoch, d, k,
                                            ptr(out, C.c_uint64)))
    return out[:k]


def batches(perm: EpochPermutation, b: int) -> List[GlobalBatch]:
    """core.hpp:35-38 / core.cpp:57-73: consecutive windows, remainder dropped.
    Windows are views of the permutation (no copy)."""
    d = len(perm.order)
    if b == 0 or b > d:
        raise InvalidArgument("batches: batch size must be in [1, dataset size]")
    return [GlobalBatch(t, perm.order[t * b:(t + 1) * b]) for t in range(d // b)]


# ------------------------------------------------------------ sampling.hpp
class CacheDirectory:
    """sampling.hpp:15-39 / sampling.cpp:7-25 (closed form, replicated)."""

    def __init__(self, d: int, p: int, alpha: float):
        if p == 0:
            raise InvalidArgument("CacheDirectory: learner count must be >= 1")
        if not (alpha > 0.0) or alpha > 1.0:
            raise InvalidArgument("CacheDirectory: cached fraction must be in (0, 1]")
        self._d, self._p, self._alpha = int(d), int(p), float(alpha)
        c = int(np.float64(alpha) * np.float64(d))  # sampling.cpp:15, truncation toward 0
        self._cached = min(c, self._d)

    def owner(self, s: int) -> Optional[LearnerId]:
        if s >= self._cached:
            return None
        return s * self._p // self._cached

    def owned_count(self, j: int) -> int:
        if j >= self._p:
            return 0
        up = lambda k: (k * self._cached + self._p - 1) // self._p  # noqa: E731
        return up(j + 1) - up(j)

    def owned_begin(self, j: int) -> int:
        return (j * self._cached + self._p - 1) // self._p

    def dataset_size(self) -> int:
        return self._d

    def learners(self) -> int:
        return self._p

    def cached_fraction(self) -> float:
        return self._alpha

    def cached_count(self) -> int:
        return self._cached


@dataclass
class LocalAssignment:  # sampling.hpp:42-46
    learner: int = 0
    step: int = 0
    samples: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


@dataclass
class LocDistribution:  # sampling.hpp:51-56
    step: int = 0
    assignments: List[LocalAssignment] = field(default_factory=list)
    uncached: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    counts: List[int] = field(default_factory=list)


@dataclass
class Assignment:
    """Device result of one step (ll_assign)."""
    final_ids: np.ndarray
    final_off: np.ndarray
    kept: np.ndarray
    counts: np.ndarray
    moves: list
    stats: np.ndarray

    def lists(self) -> List[np.ndarray]:
        return [self.final_ids[self.final_off[j]:self.final_off[j + 1]]
                for j in range(len(self.kept))]


def assign_batch(batch_samples, d: int, p: int, alpha: float, scheme: int,
                 device: int = 0) -> Assignment:
    """One global batch through the device assignment kernel (K4)."""
    b = np.ascontiguousarray(batch_samples, dtype=np.uint64)
    B = len(b)
    ids = np.empty(max(B, 1), np.uint64)
    off = np.empty(p + 1 if p else 1, np.uint64)
    kept = np.empty(max(p, 1), np.uint64)
    counts = np.empty(max(p, 1), np.uint64)
    moves = (_capi.Move * max(p, 1))()
    nm = C.c_uint32()
    stats = np.zeros(4, np.uint64)
    check(_capi.lib().ll_assign(context(device), ptr(b, C.c_uint64) if B else None, B, d, p,
                                alpha, scheme, ptr(ids, C.c_uint64), ptr(off, C.c_uint64),
                                ptr(kept, C.c_uint64), ptr(counts, C.c_uint64), moves,
                                C.byref(nm), ptr(stats, C.c_uint64)))
    mv = [(m.sender, m.receiver, m.count, m.src_off, m.dst_off, m.nvlink)
          for m in moves[:nm.value]]
    return Assignment(ids[:B], off[:p + 1], kept[:p], counts[:p], mv, stats)


@dataclass
class EpochPlan:
    """A whole epoch's device plan (ll_plan_epoch): permute_epoch + batches +
    the per-step assignment of every global batch."""
    steps: int
    B: int
    p: int
    final_ids: np.ndarray  # [steps][B]
    final_off: np.ndarray  # [steps][p+1]
    kept: np.ndarray       # [steps][p]
    counts: np.ndarray     # [steps][p]
    moves: list            # per step: [(sender, receiver, count, src_off, dst_off, nvlink)]
    totals: np.ndarray     # {moved, nvlink, uncached, reg_remote}

    def lists(self, step: int) -> List[np.ndarray]:
        o = self.final_off[step]
        return [self.final_ids[step, o[j]:o[j + 1]] for j in range(self.p)]


def plan_epoch(seed: int, epoch: int, d: int, p: int, B: int, alpha: float = 1.0,
               scheme: str = "locality_balanced", device: int = 0,
               with_ids: bool = True) -> EpochPlan:
    """The sampler half of Loader::run_epoch (pipeline.cpp:251-252) composed
    with equivalence.cpp:66-91 for every step: K2+K3 then K4, on the device."""
    if B == 0 or B > d:
        raise InvalidArgument("batches: batch size must be in [1, dataset size]")
    steps = d // B
    sc = SchemeKind[scheme] if isinstance(scheme, str) else int(scheme)
    ids = np.empty((steps, B), np.uint64) if with_ids else None
    off = np.empty((steps, p + 1), np.uint64)
    kept = np.empty((steps, max(p, 1)), np.uint64)
    counts = np.empty((steps, max(p, 1)), np.uint64)
    moves = (_capi.Move * (steps * max(p, 1)))()
    nm = np.zeros(steps, np.uint32)
    tot = np.zeros(4, np.uint64)
    n_steps = C.c_uint64()
    check(_capi.lib().ll_plan_epoch(context(device), seed, epoch, d, p, B, alpha, sc,
                                    C.byref(n_steps), ptr(ids, C.c_uint64) if with_ids else None,
                                    ptr(off, C.c_uint64), ptr(kept, C.c_uint64),
                                    ptr(counts, C.c_uint64), moves, ptr(nm, C.c_uint32),
                                    ptr(tot, C.c_uint64)))
    mv = [[(m.sender, m.receiver, m.count, m.src_off, m.dst_off, m.nvlink)
           for m in moves[s * p:s * p + int(nm[s])]] for s in range(steps)]
    return EpochPlan(steps, B, p, ids, off, kept[:, :p], counts[:, :p], mv, tot)


def reg_slice(batch: GlobalBatch, p: int, j: int, device: int = 0) -> LocalAssignment:
    """sampling.cpp:27-42."""
    if p == 0 or j >= p:
        raise InvalidArgument("reg_slice: learner rank out of range")
    B = len(batch.samples)
    if B % p != 0:
        raise InvalidArgument("reg_slice: learner count must divide the batch size")
    a = assign_batch(batch.samples, 2 ** 32 - 2, p, 1.0, _capi.SCHEME_REGULAR, device)
    return LocalAssignment(j, batch.step, a.lists()[j].copy())


def loc_distribution(batch: GlobalBatch, dir: CacheDirectory, device: int = 0) -> LocDistribution:
    """sampling.cpp:44-63.  The device list of learner j holds its cached
    samples (batch order) followed by its round-robin share of the uncached
    ones; the reference's separate `uncached` list is re-interleaved from those
    shares (the k-th uncached sample is entry k // p of learner k % p's share)."""
    p = dir.learners()
    a = assign_batch(batch.samples, dir.dataset_size(), p, dir.cached_fraction(),
                     _capi.SCHEME_LOCALITY, device)
    U = int(a.stats[2])
    lists = a.lists()
    dealt = [U // p + (1 if j < U % p else 0) for j in range(p)]
    owned = [int(a.counts[j]) - dealt[j] for j in range(p)]
    unc = np.empty(U, np.uint64)
    for j in range(p):
        unc[j::p] = lists[j][owned[j]:]
    dist = LocDistribution(batch.step)
    dist.assignments = [LocalAssignment(j, batch.step, lists[j][:owned[j]].copy())
                        for j in range(p)]
    dist.uncached = unc
    dist.counts = owned
    return dist


def counts_with_uncached(dist: LocDistribution, p: int) -> List[int]:
    """sampling.cpp:65-72."""
    counts = list(dist.counts) + [0] * max(0, p - len(dist.counts))
    counts = counts[:p]
    for k in range(len(dist.uncached)):
        counts[k % p] += 1
    return counts


# ------------------------------------------------------------- balance.hpp
@dataclass
class ImbalanceVector:  # balance.hpp:12-18
    counts: List[int] = field(default_factory=list)
    targets: List[int] = field(default_factory=list)

    def total(self) -> int:
        return int(sum(self.counts))

    def learners(self) -> int:
        return len(self.counts)


@dataclass
class Move:  # balance.hpp:24-28
    sender: int = 0
    receiver: int = 0
    count: int = 0


@dataclass
class TransferSchedule:  # balance.hpp:30-34
    moves: List[Move] = field(default_factory=list)


def targets(b: int, p: int) -> List[int]:
    """balance.cpp:14-28."""
    if p == 0:
        raise InvalidArgument("targets: learner count must be >= 1")
    if b < 0:
        raise InvalidArgument("targets: batch size must be non-negative")
    return [b // p + (1 if j < b % p else 0) for j in range(p)]


def _validate(iv: ImbalanceVector) -> None:  # balance.cpp:32-41
    if len(iv.counts) != len(iv.targets):
        raise InvalidArgument("balance: counts and targets must have equal length")
    if sum(iv.counts) != sum(iv.targets):
        raise InvalidArgument("balance: counts and targets must sum to the same total")


def balance_many(ivs: List[ImbalanceVector], device: int = 0) -> List[TransferSchedule]:
    """Algorithm 1 (balance.cpp:58-84) for many equal-p instances in one launch."""
    if not ivs:
        return []
    for iv in ivs:
        _validate(iv)
    p = len(ivs[0].counts)
    assert all(len(iv.counts) == p for iv in ivs)
    n = len(ivs)
    if p == 0:
        return [TransferSchedule() for _ in ivs]
    cnt = np.ascontiguousarray([iv.counts for iv in ivs], dtype=np.int64)
    tg = np.ascontiguousarray([iv.targets for iv in ivs], dtype=np.int64)
    moves = (_capi.Move * (n * p))()
    nm = np.zeros(n, np.uint32)
    check(_capi.lib().ll_balance_batch(context(device), ptr(cnt, C.c_int64), ptr(tg, C.c_int64),
                                       p, n, moves, ptr(nm, C.c_uint32)))
    out = []
    for i in range(n):
        out.append(TransferSchedule([Move(m.sender, m.receiver, m.count)
                                     for m in moves[i * p:i * p + int(nm[i])]]))
    return out


def balance(iv: ImbalanceVector, device: int = 0) -> TransferSchedule:
    """balance.hpp:36-41."""
    _validate(iv)
    if len(iv.counts) == 0:
        return TransferSchedule()
    return balance_many([iv], device)[0]


def deficit_fraction(iv: ImbalanceVector) -> float:
    """balance.cpp:126-135."""
    _validate(iv)
    b = iv.total()
    if b == 0:
        return 0.0
    return sum(max(0, t - c) for c, t in zip(iv.counts, iv.targets)) / b


SchemeKind = {"regular": _capi.SCHEME_REGULAR, "locality": _capi.SCHEME_LOCALITY,
              "locality_balanced": _capi.SCHEME_LOCALITY_BALANCED}


def assign(batch: GlobalBatch, scheme: str, p: int, dir: CacheDirectory,
           device: int = 0) -> List[LocalAssignment]:
    """equivalence.cpp:66-91 (the reference's private per-step assignment)."""
    if scheme == "regular":
        return [reg_slice(batch, p, j, device) for j in range(p)]
    a = assign_batch(batch.samples, dir.dataset_size(), p, dir.cached_fraction(),
                     SchemeKind[scheme], device)
    return [LocalAssignment(j, batch.step, lst.copy()) for j, lst in enumerate(a.lists())]


# --------------------------------------------------------- equivalence.hpp
class ToyObjective:
    """equivalence.hpp:12-33: least-squares data, synthesised on the host by
    the library (ll_toy_synthesize, bit-identical to equivalence.cpp:12-37)."""

    def __init__(self, xs: np.ndarray, ys: np.ndarray):
        self.xs = xs
        self.ys = ys

    @staticmethod
    def synthesize(n: int, dims: int, seed: int) -> "ToyObjective":
        if n <= 0 or dims <= 0:
            raise InvalidArgument("ToyObjective: need n >= 1 and dims >= 1")
        xs = np.empty(n * dims, np.float64)
        ys = np.empty(n, np.float64)
        check(_capi.lib().ll_toy_synthesize(n, dims, seed, ptr(xs, C.c_double),
                                            ptr(ys, C.c_double)))
        return ToyObjective(xs.reshape(n, dims), ys)

    def samples(self) -> int:
        return self.ys.shape[0]

    def dims(self) -> int:
        return self.xs.shape[1]


@dataclass
class TrainingRun:  # equivalence.hpp:52-55
    final_weights: np.ndarray
    step_gradients: np.ndarray  # [steps][dims], each normalised by B


Aggregation = {"canonical": _capi.AGG_CANONICAL, "learner_order": _capi.AGG_LEARNER_ORDER}


def run_training(obj: ToyObjective, scheme: str, p: int, batch_size: int, steps: int, seed: int,
                 learning_rate: float, agg: str = "canonical", device: int = 0) -> TrainingRun:
    """equivalence.cpp:95-174 on the device (ll_train_run)."""
    if scheme not in SchemeKind:
        raise InvalidArgument(f"run_training: unknown scheme {scheme!r}")
    xs = np.ascontiguousarray(obj.xs, np.float64)
    ys = np.ascontiguousarray(obj.ys, np.float64)
    w = np.empty(obj.dims(), np.float64)
    g = np.empty((max(steps, 1), obj.dims()), np.float64)
    check(_capi.lib().ll_train_run(context(device), ptr(xs, C.c_double), ptr(ys, C.c_double),
                                   obj.samples(), obj.dims(), SchemeKind[scheme], p, batch_size,
                                   steps, seed, learning_rate, Aggregation[agg],
                                   ptr(w, C.c_double), ptr(g, C.c_double)))
    return TrainingRun(w, g[:steps])


def run_training_imbalanced_vs_balanced(obj: ToyObjective, p: int, batch_size: int, steps: int,
                                        seed: int, learning_rate: float, device: int = 0):
    """equivalence.hpp:64-67."""
    return (run_training(obj, "locality", p, batch_size, steps, seed, learning_rate,
                         device=device),
            run_training(obj, "locality_balanced", p, batch_size, steps, seed, learning_rate,
                         device=device))


def full_batch_gradient(obj: ToyObjective, w, batch: GlobalBatch, device: int = 0) -> np.ndarray:
    """equivalence.cpp:190-205 on the device."""
    xs = np.ascontiguousarray(obj.xs, np.float64)
    ys = np.ascontiguousarray(obj.ys, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    ids = np.ascontiguousarray(batch.samples, np.uint64)
    out = np.empty(obj.dims(), np.float64)
    check(_capi.lib().ll_full_batch_gradient(context(device), ptr(xs, C.c_double),
                                             ptr(ys, C.c_double), obj.samples(), obj.dims(),
                                             ptr(w, C.c_double), ptr(ids, C.c_uint64), len(ids),
                                             ptr(out, C.c_double)))
    return out
