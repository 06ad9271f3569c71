"""Generate tests/golden/golden.json by RUNNING THE REFERENCE.

Every value below comes from oracle/_ref/liblocload_ref.so, i.e. the
unmodified reference sources in /root/reference/proj compiled by
oracle/Makefile (plus ref_shim.cpp's extern "C" wrappers).  Run in the build
container (the only place /root/reference exists):

    python tests/golden/make_golden.py

The fixture is committed; tests on the GPU box only read it.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def splitmix_draws(seed, k):
    import ctypes as C
    out = np.empty(k, np.uint64)
    oracle.ref().ref_splitmix_draws(seed, k, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return [int(x) for x in out]


def splitmix_bounded(seed, n, k):
    import ctypes as C
    out = np.empty(k, np.uint64)
    oracle.ref().ref_splitmix_bounded(seed, n, k, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return [int(x) for x in out]


def reg_remote(batch, d, p):
    """samples of the batch whose reg_slice learner is not their owner."""
    import ctypes as C
    owners = np.empty(len(batch), np.uint32)
    b = np.ascontiguousarray(batch, dtype=np.uint64)
    oracle.ref().ref_owner(d, p, 1.0, b.ctypes.data_as(C.POINTER(C.c_uint64)), len(b),
                           owners.ctypes.data_as(C.POINTER(C.c_uint32)))
    slice_ = len(batch) // p
    pos_learner = np.arange(len(batch)) // slice_
    return int((owners != pos_learner).sum())


def plan_step_digest(lists, off, moves) -> str:
    """sha256 over one step's plan: the final lists (u64, learner-major), the
    offsets[p+1] (u64) and the moves as (sender, receiver, count) i64 triples.
    The GPU tests digest ll_plan_epoch's tables the same way."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(lists, dtype=np.uint64).tobytes())
    h.update(np.ascontiguousarray(off, dtype=np.uint64).tobytes())
    h.update(np.asarray([x for m in moves for x in m[:3]], dtype=np.int64).tobytes())
    return h.hexdigest()


def ref_epoch_plan(d, p, B, seed, epoch):
    """The reference's plan of one epoch (alpha = 1), step by step."""
    order = oracle.ref_permute_epoch(seed, epoch, d)
    steps = []
    moved = reg = 0
    for t in range(d // B):
        batch = order[t * B:(t + 1) * B]
        lists, off, mv = oracle.ref_assign_balanced(batch, d, p)
        steps.append((lists, off, mv))
        moved += sum(m[2] for m in mv)
        reg += reg_remote(batch, d, p)
    return order, steps, moved, reg


def main() -> None:
    R = oracle.ref()
    g: dict = {"source": "oracle/_ref (reference sources compiled in place)"}

    g["rng"] = {
        "mix64": {str(z): int(R.ref_mix64(z)) for z in [0, 1, 42, 2 ** 63, 2 ** 64 - 1]},
        "derive_seed": [[s, a, int(R.ref_derive_seed(s, a))]
                        for s, a in [(42, 0), (42, 1), (7, 0), (0, 0), (123, 4)]],
        "derive_seed3": [[s, a, b, int(R.ref_derive_seed3(s, a, b))]
                         for s, a, b in [(42, 0, 0), (42, 1, 5), (7, 3, 1)]],
        "draws": {"seed": int(R.ref_derive_seed(42, 0)),
                  "values": splitmix_draws(int(R.ref_derive_seed(42, 0)), 16)},
        "bounded": [{"seed": s, "n": n, "values": splitmix_bounded(s, n, 32)}
                    for s, n in [(1, 33), (2, 1000), (3, 1), (4, 2 ** 40 + 7)]],
    }

    perms = []
    for d in [1, 2, 13, 1000, 10000]:
        for seed, epoch in [(123, 4), (42, 0), (7, 1), (99, 3)]:
            o = oracle.ref_permute_epoch(seed, epoch, d)
            perms.append({"seed": seed, "epoch": epoch, "d": d, "order": [int(x) for x in o]})
    for d, seed, epoch in [(160000, 42, 1), (640000, 42, 0), (1280000, 42, 0),
                           (1280000, 7, 2)]:
        o = oracle.ref_permute_epoch(seed, epoch, d)
        perms.append({"seed": seed, "epoch": epoch, "d": d, "head": [int(x) for x in o[:64]],
                      "sha256": sha(o)})
    g["permutations"] = perms

    # locality-balanced assignment of whole epochs' batches (alpha = 1)
    cases = []
    for d, p, B, seed, epoch, steps in [(48, 4, 16, 7, 0, 1), (10000, 4, 256, 42, 0, 6),
                                        (10000, 4, 256, 42, 1, 3), (5000, 3, 999, 5, 2, 3),
                                        (20000, 8, 1024, 42, 0, 3), (4096, 2, 64, 11, 0, 4),
                                        (1000, 7, 13, 3, 0, 5), (3000, 1, 100, 1, 0, 2),
                                        (64, 64, 64, 9, 0, 1), (100000, 5, 2000, 17, 3, 2)]:
        order = oracle.ref_permute_epoch(seed, epoch, d)
        for t in range(steps):
            batch = order[t * B:(t + 1) * B]
            lists, off, mv = oracle.ref_assign_balanced(batch, d, p)
            cases.append({"d": d, "p": p, "B": B, "seed": seed, "epoch": epoch, "step": t,
                          "batch": [int(x) for x in batch], "lists": [int(x) for x in lists],
                          "off": [int(x) for x in off], "moves": mv})
    g["assign_balanced"] = cases

    # loc_distribution with a partial cache (counts and cached lists)
    part = []
    rng = np.random.default_rng(2024)
    for _ in range(40):
        d = int(rng.integers(64, 5000))
        p = int(rng.integers(1, 17))
        alpha = float(int(rng.integers(1, 101)) / 100.0)
        B = int(rng.integers(1, min(d, 512)))
        batch = rng.choice(d, B, replace=False).astype(np.uint64)
        r = oracle.ref_loc_distribution(batch, d, p, alpha)
        tg = oracle.ref_targets(B, p)
        mv = oracle.ref_balance(r["cwu"].astype(np.int64), tg)
        part.append({"d": d, "p": p, "alpha": alpha, "batch": [int(x) for x in batch],
                     "lists": [[int(x) for x in l] for l in r["lists"]],
                     "uncached": [int(x) for x in r["uncached"]],
                     "counts": [int(x) for x in r["counts"]],
                     "cwu": [int(x) for x in r["cwu"]], "targets": tg, "moves": mv})
    g["loc_distribution_partial"] = part

    # Algorithm 1 on random instances (the shape of test_balance.cpp:20-29)
    bal = []
    for max_p, n in [(64, 400), (8, 600)]:
        for _ in range(n):
            p = int(rng.integers(1, max_p + 1))
            b = int(rng.integers(0, 8 * p + 1))
            counts = np.bincount(rng.integers(0, p, b), minlength=p).astype(np.int64)
            tg = oracle.ref_targets(b, p)
            bal.append({"counts": counts.tolist(), "targets": tg,
                        "moves": oracle.ref_balance(counts, tg)})
    g["balance"] = bal

    # generate_dataset bytes
    samples = []
    with tempfile.TemporaryDirectory() as tmp:
        for seed, sid, nbytes in [(42, 0, 196608), (42, 1, 196608), (42, 3, 196608),
                                  (1, 7, 1024), (9, 13, 512), (42, 0, 13)]:
            b = oracle.ref_gen_sample(seed, sid, nbytes, tmp)
            samples.append({"seed": seed, "id": sid, "bytes": nbytes,
                            "head": b[:32].tobytes().hex(),
                            "sha256": hashlib.sha256(b.tobytes()).hexdigest()})
    g["samples"] = samples

    # remote samples per epoch, Loc (moved) vs Reg (remote) -- SURVEY 8(d)
    remote = []
    for d, p, B, seed, epoch in [(10000, 4, 256, 42, 0), (160000, 2, 2048, 42, 0),
                                 (320000, 4, 4096, 42, 1)]:
        order = oracle.ref_permute_epoch(seed, epoch, d)
        moved = reg = 0
        for t in range(d // B):
            batch = order[t * B:(t + 1) * B]
            _, _, mv = oracle.ref_assign_balanced(batch, d, p)
            moved += sum(m[2] for m in mv)
            reg += reg_remote(batch, d, p)
        remote.append({"d": d, "p": p, "B": B, "seed": seed, "epoch": epoch, "loc_moved": moved,
                       "reg_remote": reg})
    g["remote_per_epoch"] = remote

    # the headline configuration's plan (cfg2 shape: d = 1.28 M, B = 1,024 p),
    # whole epochs, per-step digests -- SURVEY 8(d), BASELINE.md section 4
    plans = []
    for d, p, B, seed, epoch in [(1280000, 2, 2048, 42, 0), (1280000, 4, 4096, 42, 0),
                                 (1280000, 8, 8192, 42, 0), (1280000, 8, 8192, 7, 2)]:
        _, steps, moved, reg = ref_epoch_plan(d, p, B, seed, epoch)
        plans.append({"d": d, "p": p, "B": B, "seed": seed, "epoch": epoch, "steps": len(steps),
                      "loc_moved": moved, "reg_remote": reg,
                      "n_moves": [len(mv) for _, _, mv in steps],
                      "step_sha256": [plan_step_digest(*st) for st in steps]})
    g["epoch_plans"] = plans

    # Eq. 8's predicted beta: simulate_imbalance the way `locload imbalance`
    # runs it (500 steps, seed derive_seed(seed, p, local_batch))
    g["simulate_imbalance"] = [
        {"d": 1280000, "p": p, "local_batch": 1024, "steps": 500, "seed": 42,
         "beta_median": oracle.eq8_beta_median(1280000, p, 1024, 42)} for p in (2, 4, 8)]

    with open(OUT, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
