"""CUDA path vs the oracle / the reference's golden vectors, through the C-ABI.

Bars (north_star): permutation, per-learner assignment and remote-fetch lists
bit-exact; augmented tensors within 1e-5 abs (fp32) / 1 ulp (bf16) after
normalisation -- the kernels are in fact bit-exact with the oracle and the
tests assert that too.  Mirrors the reference suites test_core.cpp,
test_sampling.cpp, test_balance.cpp, test_pipeline.cpp (cited per test).
"""
import hashlib

import numpy as np
import pytest

import oracle
import paper_1910_01196_b200 as ll
from paper_1910_01196_b200 import _capi
from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5


def bf16_ulps(a: np.ndarray, b: np.ndarray) -> int:
    """max distance in bf16 ulps between two arrays of bf16 bit patterns"""
    def key(x):
        x = x.astype(np.int32)
        return np.where(x & 0x8000, 0x8000 - (x & 0x7FFF), x + 0x8000)
    return int(np.abs(key(a) - key(b)).max()) if a.size else 0


# ------------------------------------------------------------- core (K2+K3)
def test_permute_matches_reference_golden(golden):
    for c in golden["permutations"]:
        o = ll.permute_epoch(c["seed"], c["epoch"], c["d"]).order
        if "order" in c:
            assert o.tolist() == c["order"], (c["seed"], c["epoch"], c["d"])
        else:
            assert o[:64].tolist() == c["head"]
            assert hashlib.sha256(o.tobytes()).hexdigest() == c["sha256"], c["d"]


def test_permute_random_vs_oracle():
    rng = np.random.default_rng(11)
    for d in [1, 2, 3, 31, 32, 33, 511, 512, 513, 16383, 16384, 16385, 65537, 200003]:
        s, e = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, 1000))
        assert np.array_equal(ll.permute_epoch(s, e, d).order, oracle.permute_epoch(s, e, d)), d


@pytest.mark.parametrize("forced", [[0], [5], [999], [3, 4, 5], [10, 500, 998], [998, 999],
                                    [1, 1000, 1500]])
def test_permute_forced_rejections_vs_oracle(forced):
    """The Lemire retry path (rng.hpp:41-50): draw indices forced to reject."""
    d = 1000
    f = np.ascontiguousarray(sorted(forced), dtype=np.uint64)
    out = np.empty(d, np.uint64)
    import ctypes as C
    _capi.check(_capi.lib().ll_permute_epoch_forced(ll.locload.context(), 5, 1, d,
                                                    _capi.ptr(f, C.c_uint64), len(f),
                                                    _capi.ptr(out, C.c_uint64)))
    assert np.array_equal(out, oracle.permute_epoch(5, 1, d, forced=forced))


def test_permute_large_forced_vs_oracle():
    import ctypes as C
    d = 300000
    forced = [7, 123456, 123457, 299990]
    f = np.ascontiguousarray(forced, dtype=np.uint64)
    out = np.empty(d, np.uint64)
    _capi.check(_capi.lib().ll_permute_epoch_forced(ll.locload.context(), 9, 0, d,
                                                    _capi.ptr(f, C.c_uint64), len(f),
                                                    _capi.ptr(out, C.c_uint64)))
    assert np.array_equal(out, oracle.permute_epoch(9, 0, d, forced=forced))


def test_single_sample_and_errors():
    assert ll.permute_epoch(7, 0, 1).order.tolist() == [0]  # test_core.cpp:12-15
    with pytest.raises(ValueError, match="permute_epoch: dataset must contain"):
        ll.permute_epoch(7, 0, 0)  # test_core.cpp:41-44
    with pytest.raises(ValueError, match="permutation_prefix"):
        ll.permutation_prefix(7, 0, 0, 0)


def test_determinism_and_bijection():
    """test_core.cpp:17-39"""
    a, b = ll.permute_epoch(7, 0, 12).order, ll.permute_epoch(7, 0, 12).order
    assert np.array_equal(a, b)
    assert not np.array_equal(a, ll.permute_epoch(7, 1, 12).order)
    assert not np.array_equal(a, ll.permute_epoch(8, 0, 12).order)
    for d in [1, 2, 13, 1000, 10000]:
        o = ll.permute_epoch(123, 4, d).order
        assert sorted(o.tolist()) == list(range(d))


def test_positions_uniform_across_seeds():
    """test_core.cpp:49-73: chi-square over 20 bins, 1000 seeds, crit 43.82."""
    d, bins, seeds = 10000, 20, 1000
    pos = {0: [], 1234: [], 9999: []}
    for s in range(seeds):
        o = ll.permute_epoch(s, 0, d).order
        inv = np.empty(d, np.int64)
        inv[o.astype(np.int64)] = np.arange(d)
        for t in pos:
            pos[t].append(inv[t])
    for t, ps in pos.items():
        h = np.bincount(np.array(ps) * bins // d, minlength=bins)
        exp = seeds / bins
        assert ((h - exp) ** 2 / exp).sum() < 43.82, t


def test_prefix_matches_dense():
    """test_core.cpp:75-85"""
    d = 5000
    full = ll.permute_epoch(99, 3, d).order
    for k in [0, 1, 64, 4096, d]:
        assert np.array_equal(ll.permutation_prefix(99, 3, d, k), full[:k])
    with pytest.raises(ValueError):
        ll.permutation_prefix(99, 3, d, d + 1)


def test_batches():
    """test_core.cpp:87-122"""
    perm = ll.permute_epoch(7, 0, 10)
    bs = ll.batches(perm, 4)
    assert len(bs) == 2 and all(len(b.samples) == 4 for b in bs)
    perm = ll.permute_epoch(11, 2, 1024)
    bs = ll.batches(perm, 64)
    assert len(bs) == 16
    assert sorted(np.concatenate([b.samples for b in bs]).tolist()) == list(range(1024))
    with pytest.raises(ValueError):
        ll.batches(perm, 0)
    with pytest.raises(ValueError):
        ll.batches(perm, 1025)


def test_permute_rounds_reported():
    ll.permute_epoch(42, 0, 1280000)
    import ctypes as C
    r = C.c_uint32()
    _capi.check(_capi.lib().ll_last_permute_rounds(ll.locload.context(), C.byref(r)))
    assert 10 < r.value < 200


# ---------------------------------------------------- sampling + balance (K4)
def test_assign_matches_reference_golden(golden):
    for c in golden["assign_balanced"]:
        a = ll.assign_batch(c["batch"], c["d"], c["p"], 1.0, _capi.SCHEME_LOCALITY_BALANCED)
        assert a.final_ids.tolist() == c["lists"], (c["d"], c["p"], c["B"], c["step"])
        assert a.final_off.tolist() == c["off"]
        assert [m[:3] for m in a.moves] == [tuple(m) for m in c["moves"]]


def test_assign_vs_oracle_random_all_schemes():
    rng = np.random.default_rng(5)
    for _ in range(150):
        p = int(rng.integers(1, 65))
        d = int(rng.integers(max(p, 64), 20000))
        B = int(rng.integers(1, min(d, 5000)))
        alpha = float(rng.choice([1.0, 1.0, 0.5, 0.25, 0.73, 0.01]))
        batch = rng.choice(d, B, replace=False).astype(np.uint64)
        cached = oracle.cached_count(d, alpha)
        for scheme in [_capi.SCHEME_LOCALITY, _capi.SCHEME_LOCALITY_BALANCED]:
            a = ll.assign_batch(batch, d, p, alpha, scheme)
            r = oracle.assign_step(batch, p, cached, scheme)
            assert np.array_equal(a.final_ids, r["final_ids"])
            assert np.array_equal(a.final_off, r["final_off"])
            assert np.array_equal(a.kept, r["kept"])
            assert np.array_equal(a.counts, r["counts"])
            assert [m[:5] for m in a.moves] == [tuple(int(x) for x in m) for m in r["moves"]]
            # NVLink count per move = cached samples in the moved run
            for m in a.moves:
                run = a.final_ids[a.final_off[m[1]] + m[4]:a.final_off[m[1]] + m[4] + m[2]]
                assert m[5] == int((run < cached).sum())
        if B % p == 0:
            a = ll.assign_batch(batch, d, p, alpha, _capi.SCHEME_REGULAR)
            assert np.array_equal(a.final_ids, batch)
            owners = np.array([oracle.lib().lo_owner(int(s), p, cached) for s in batch])
            reg_learner = np.arange(B) // (B // p)
            assert a.stats[3] == int(((owners != reg_learner) & (owners < p)).sum())


def test_loc_distribution_reference_cases():
    """test_sampling.cpp:85-123, 195-203"""
    batch = ll.GlobalBatch(0, np.array([0, 13, 25, 14, 26, 15, 27, 16, 28, 17, 1, 18], np.uint64))
    dist = ll.loc_distribution(batch, ll.CacheDirectory(36, 3, 1.0))
    assert dist.counts == [2, 6, 4] and len(dist.uncached) == 0
    assert dist.assignments[0].samples.tolist() == [0, 1]
    assert dist.assignments[1].samples.tolist() == [13, 14, 15, 16, 17, 18]
    assert dist.assignments[2].samples.tolist() == [25, 26, 27, 28]
    b2 = ll.GlobalBatch(0, np.array([0, 6, 7, 8, 9, 5], np.uint64))
    dist = ll.loc_distribution(b2, ll.CacheDirectory(12, 3, 0.5))
    assert dist.counts == [1, 0, 1]
    assert dist.uncached.tolist() == [6, 7, 8, 9]
    assert ll.counts_with_uncached(dist, 3) == [3, 1, 2]
    rb = ll.GlobalBatch(0, np.array([5, 9, 1, 7, 0, 3, 11, 2, 8, 10, 4, 6], np.uint64))
    assert ll.reg_slice(rb, 3, 0).samples.tolist() == [5, 9, 1, 7]
    assert ll.reg_slice(rb, 1, 0).samples.tolist() == rb.samples.tolist()
    with pytest.raises(ValueError, match="reg_slice: learner count must divide"):
        ll.reg_slice(rb, 5, 0)
    with pytest.raises(ValueError, match="reg_slice: learner rank out of range"):
        ll.reg_slice(rb, 3, 3)


def test_partial_cache_vs_reference_golden(golden):
    for c in golden["loc_distribution_partial"]:
        dist = ll.loc_distribution(ll.GlobalBatch(0, np.array(c["batch"], np.uint64)),
                                   ll.CacheDirectory(c["d"], c["p"], c["alpha"]))
        assert dist.counts == c["counts"]
        assert dist.uncached.tolist() == c["uncached"]
        assert [a.samples.tolist() for a in dist.assignments] == c["lists"]
        assert ll.counts_with_uncached(dist, c["p"]) == c["cwu"]


def test_balance_matches_reference_golden(golden):
    by_p = {}
    for c in golden["balance"]:
        by_p.setdefault(len(c["counts"]), []).append(c)
    for p, cases in by_p.items():
        ivs = [ll.ImbalanceVector(c["counts"], c["targets"]) for c in cases]
        got = ll.balance_many(ivs)
        for c, s in zip(cases, got):
            assert [(m.sender, m.receiver, m.count) for m in s.moves] == \
                [tuple(m) for m in c["moves"]]


def test_balance_reference_examples_and_properties():
    """test_balance.cpp:55-101"""
    def mv(c, t):
        return [(m.sender, m.receiver, m.count)
                for m in ll.balance(ll.ImbalanceVector(c, t)).moves]
    assert mv([2, 6, 4], [4, 4, 4]) == [(1, 0, 2)]
    assert mv([10, 0, 2], [4, 4, 4]) == [(0, 1, 4), (0, 2, 2)]
    assert mv([6, 6, 2, 2], [4, 4, 4, 4]) == [(0, 2, 2), (1, 3, 2)]
    assert mv([4, 4, 4], [4, 4, 4]) == [] and mv([], []) == []
    with pytest.raises(ValueError):
        mv([1, 2], [4, 4])
    with pytest.raises(ValueError):
        mv([1, 2, 3], [3, 3])
    rng = np.random.default_rng(404)
    for p in range(1, 65):
        ivs = []
        for _ in range(32):
            b = int(rng.integers(0, 8 * p + 1))
            cnt = np.bincount(rng.integers(0, p, b), minlength=p).tolist()
            ivs.append(ll.ImbalanceVector(cnt, ll.targets(b, p)))
        for iv, s in zip(ivs, ll.balance_many(ivs)):
            net = [0] * p
            for m in s.moves:
                assert m.count >= 1 and m.sender != m.receiver
                net[m.sender] -= m.count
                net[m.receiver] += m.count
            assert net == [t - c for c, t in zip(iv.counts, iv.targets)]
            assert len(s.moves) <= max(p - 1, 0)


# ------------------------------------------------------------- dataset (K1)
def test_generated_bytes_match_reference_golden(golden):
    import ctypes as C
    for c in golden["samples"]:
        ids = np.array([c["id"]], np.uint64)
        out = np.empty(c["bytes"], np.uint8)
        _capi.check(_capi.lib().ll_generate_samples(ll.locload.context(), c["seed"],
                                                    _capi.ptr(ids, C.c_uint64), 1, c["bytes"],
                                                    _capi.ptr(out, C.c_uint8)))
        assert out[:32].tobytes().hex() == c["head"]
        assert hashlib.sha256(out.tobytes()).hexdigest() == c["sha256"]


@pytest.mark.parametrize("nbytes", [187500, 1000, 17, 150528 + 8])
def test_generated_bytes_unaligned_sizes_vs_oracle(nbytes):
    """K1 with sample sizes that are not multiples of 16 (250 x 250 x 3 =
    187,500 B, ...): every 16-byte chunk writes exactly its own bytes."""
    import ctypes as C
    ids = np.array([0, 5, 77, 123456], np.uint64)
    out = np.empty(len(ids) * nbytes, np.uint8)
    _capi.check(_capi.lib().ll_generate_samples(ll.locload.context(), 42,
                                                _capi.ptr(ids, C.c_uint64), len(ids), nbytes,
                                                _capi.ptr(out, C.c_uint8)))
    want = oracle.gen_samples(42, ids, nbytes)
    assert np.array_equal(out.reshape(len(ids), nbytes), want)


# ------------------------------------------------------------- augment (K6/K7)
def device_augment(src, ids, H, W, seed, epoch, mode="crop", dtype="fp32", oh=224, ow=224):
    import ctypes as C
    spec = AugmentConfig(mode=mode, out_dtype=dtype, out_h=oh, out_w=ow).to_c()
    n = len(ids)
    out = np.empty((n, 3, oh, ow), np.float32 if dtype == "fp32" else np.uint16)
    s = np.ascontiguousarray(src, dtype=np.uint8)
    i = np.ascontiguousarray(ids, dtype=np.uint64)
    _capi.check(_capi.lib().ll_augment(ll.locload.context(), C.byref(spec), seed, epoch,
                                       _capi.ptr(s, C.c_uint8), _capi.ptr(i, C.c_uint64), n, H,
                                       W, out.ctypes.data_as(C.c_void_p)))
    return out


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_crop_augment_vs_oracle(dtype):
    rng = np.random.default_rng(1)
    ids = rng.choice(10 ** 6, 40, replace=False).astype(np.uint64)
    src = oracle.gen_samples(42, ids, 256 * 256 * 3)
    got = device_augment(src, ids, 256, 256, 42, 1, dtype=dtype)
    for k, sid in enumerate(ids):
        want = oracle.augment(src[k].reshape(256, 256, 3), int(sid), 42, 1, bf16=dtype == "bf16")
        if dtype == "fp32":
            assert np.abs(got[k] - want).max() <= FP32_TOL
        else:
            assert bf16_ulps(got[k], want) <= 1
        assert np.array_equal(got[k], want)  # bit-exact in practice


def test_crop_augment_non_square_source():
    ids = np.arange(9, dtype=np.uint64)
    H, W = 240, 320
    src = oracle.gen_samples(3, ids, H * W * 3)
    got = device_augment(src, ids, H, W, 5, 0)
    for k in range(len(ids)):
        assert np.array_equal(got[k], oracle.augment(src[k].reshape(H, W, 3), k, 5, 0))


@pytest.mark.parametrize("hw", [(250, 250), (230, 229), (224, 225), (301, 226)])
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_crop_augment_unaligned_rows(hw, dtype):
    """Sources whose rows are not a multiple of 16 bytes (750, 687, 675, 678
    bytes): K6 stages every row from the aligned address below its own window
    start; bit-exact vs the oracle (the 256-px layout keeps one phase)."""
    H, W = hw
    ids = np.arange(11, dtype=np.uint64) * 7 + 3
    src = oracle.gen_samples(9, ids, H * W * 3)
    got = device_augment(src, ids, H, W, 13, 2, dtype=dtype)
    for k, sid in enumerate(ids):
        want = oracle.augment(src[k].reshape(H, W, 3), int(sid), 13, 2, bf16=dtype == "bf16")
        assert np.array_equal(got[k], want), (hw, k)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_loader_unaligned_rows_p2p_and_storage(dtype, alpha):
    """250 x 250 sources through the loader: own shard, a peer shard over the
    P2P path (TMA row copies from the aligned address) and, with alpha = 0.5,
    the host storage tier."""
    d, p, B, seed, H = 2000, 2, 96, 42, 250
    lds = []
    for j in range(p):
        ld = DeviceLoader(LoaderConfig(d=d, height=H, width=H, learners=p, rank=j, batch_size=B,
                                       alpha=alpha, seed=seed, data_seed=seed, exchange="p2p",
                                       augment=AugmentConfig(out_dtype=dtype)))
        ld.populate()
        lds.append(ld)
    DeviceLoader.link_peers(lds)
    order = oracle.permute_epoch(seed, 1, d)
    cached = oracle.cached_count(d, alpha)
    far = 0
    for t in [0, 5]:
        r = oracle.assign_step(order[t * B:(t + 1) * B], p, cached, oracle.MODE_LOCALITY_BALANCED)
        for j, ld in enumerate(lds):
            info = ld.step(1, t)
            lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]]
            assert np.array_equal(ld.fetch_ids(info), lst)
            got = ld.fetch(info)
            src = oracle.gen_samples(seed, lst, H * H * 3)
            for k, sid in enumerate(lst):
                want = oracle.augment(src[k].reshape(H, H, 3), int(sid), seed, 1,
                                      bf16=dtype == "bf16")
                assert np.array_equal(got[k], want), (t, j, k)
            far += len(lst) - info.kept
    assert far > 0
    for ld in lds:
        ld.close()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_resize_augment_vs_oracle(dtype):
    for sid in [1, 2, 3, 4]:
        H, W = oracle.sample_hw(42, sid)
        src = oracle.gen_sample(42, sid, H * W * 3)
        got = device_augment(src[None], np.array([sid], np.uint64), H, W, 42, 2, mode="resize",
                             dtype=dtype)[0]
        want = oracle.augment(src.reshape(H, W, 3), sid, 42, 2, mode=oracle.AUG_RESIZE,
                              bf16=dtype == "bf16")
        if dtype == "fp32":
            assert np.abs(got - want).max() <= FP32_TOL
        else:
            assert bf16_ulps(got, want) <= 1
        assert np.array_equal(got, want)


@pytest.mark.parametrize("oh,ow", [(37, 45), (5, 1), (230, 300), (96, 600), (448, 512)])
def test_resize_augment_odd_shapes_vs_oracle(oh, ow):
    """Banded K7 with partial warps / odd band heights / upscaling, and the
    unbanded kernel (out_w > 512); both bit-exact vs the oracle."""
    for sid in [5, 6]:
        H, W = oracle.sample_hw(42, sid)
        src = oracle.gen_sample(42, sid, H * W * 3)
        got = device_augment(src[None], np.array([sid], np.uint64), H, W, 42, 1, mode="resize",
                             oh=oh, ow=ow)[0]
        want = oracle.augment(src.reshape(H, W, 3), sid, 42, 1, oh, ow, mode=oracle.AUG_RESIZE)
        assert np.array_equal(got, want), (oh, ow, H, W)


def test_augment_params_vs_oracle():
    import ctypes as C
    ids = np.arange(1000, dtype=np.uint64) * 7919
    spec = AugmentConfig().to_c()
    out = np.empty((1000, 5), np.uint32)
    _capi.check(_capi.lib().ll_augment_params(ll.locload.context(), C.byref(spec), 42, 3,
                                              _capi.ptr(ids, C.c_uint64), 1000, 256, 256,
                                              _capi.ptr(out, C.c_uint32)))
    for k in range(1000):
        assert tuple(out[k]) == oracle.aug_params(42, 3, int(ids[k]), 256, 256)


# ------------------------------------------------------------- loader
def make_learners(d, p, B, exchange="p2p", scheme="locality_balanced", dtype="fp32", seed=42):
    lds = []
    for j in range(p):
        cfg = LoaderConfig(d=d, learners=p, rank=j, batch_size=B, seed=seed, data_seed=seed,
                           scheme=scheme, exchange=exchange,
                           augment=AugmentConfig(out_dtype=dtype))
        ld = DeviceLoader(cfg)
        ld.populate()
        lds.append(ld)
    if p > 1 and exchange == "p2p":
        DeviceLoader.link_peers(lds)
    return lds


def test_loader_cfg1_plan_vs_oracle(golden):
    """cfg1 (d=10k, p=4, B=256): every step of epochs 0 and 1 vs the oracle,
    and the epoch's moved / regular-remote totals vs the reference."""
    ld = make_learners(10000, 4, 256)[0]
    for epoch in [0, 1]:
        ld.plan_epoch(epoch)
        order = oracle.permute_epoch(42, epoch, 10000)
        for t in range(ld.steps_per_epoch):
            ids, off, kept, counts, mv = ld.plan_step(t)
            r = oracle.assign_step(order[t * 256:(t + 1) * 256], 4, 10000,
                                   oracle.MODE_LOCALITY_BALANCED)
            assert np.array_equal(ids, r["final_ids"]) and np.array_equal(off, r["final_off"])
            assert [m[:5] for m in mv] == [tuple(int(x) for x in m) for m in r["moves"]]
        if epoch == 0:
            tot = ld.epoch_totals()
            ref = golden["remote_per_epoch"][0]
            assert tot["moved"] == ref["loc_moved"] == 417
            assert tot["reg_remote"] == ref["reg_remote"] == 7468


def _plan_step_digest(lists, off, moves) -> str:
    # tests/golden/make_golden.py:plan_step_digest
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(lists, dtype=np.uint64).tobytes())
    h.update(np.ascontiguousarray(off, dtype=np.uint64).tobytes())
    h.update(np.asarray([x for m in moves for x in m[:3]], dtype=np.int64).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("case", range(4), ids=["p2", "p4", "p8", "p8-seed7-epoch2"])
def test_headline_plan_vs_reference(golden, case):
    """cfg2's plan pinned on the device: the whole epoch at d = 1.28 M,
    B = 1,024 p (K2+K3 permutation, K4 distribution + Algorithm 1 + tail moves
    for all 625 / 312 / 156 steps) equals the reference step by step -- the
    committed per-step digests of oracle/_ref's loc_distribution, balance and
    equivalence.cpp:77-88 tail moves, and, where oracle/_ref is present, a
    live list-by-list comparison.  Epoch totals equal BASELINE.md section 4:
    11,102 / 13,652 / 15,059 moved, 640,140 / 958,300 / 1,119,042 Reg remote."""
    c = golden["epoch_plans"][case]
    d, p, B, seed, epoch = c["d"], c["p"], c["B"], c["seed"], c["epoch"]
    plan = ll.plan_epoch(seed, epoch, d, p, B)
    assert plan.steps == c["steps"] == d // B
    got = [_plan_step_digest(plan.final_ids[t], plan.final_off[t], plan.moves[t])
           for t in range(plan.steps)]
    bad = [t for t in range(plan.steps) if got[t] != c["step_sha256"][t]]
    assert not bad, f"steps differing from the reference: {bad[:10]}"
    assert [len(m) for m in plan.moves] == c["n_moves"]
    assert int(plan.totals[0]) == c["loc_moved"]
    assert int(plan.totals[1]) == c["loc_moved"]  # alpha = 1: every move crosses NVLink
    assert int(plan.totals[2]) == 0
    assert int(plan.totals[3]) == c["reg_remote"]
    want = {(2, 42): (11102, 640140), (4, 42): (13652, 958300), (8, 42): (15059, 1119042)}
    if (p, seed) in want:
        assert (c["loc_moved"], c["reg_remote"]) == want[(p, seed)]
    # every learner keeps >= 90 % of its samples local (north_star target)
    assert 1 - c["loc_moved"] / (plan.steps * B) >= 0.90
    if oracle.ref_available():
        order = oracle.ref_permute_epoch(seed, epoch, d)
        for t in range(0, plan.steps, 7):
            lists, off, mv = oracle.ref_assign_balanced(order[t * B:(t + 1) * B], d, p)
            assert np.array_equal(plan.final_ids[t], lists), t
            assert np.array_equal(plan.final_off[t], off), t
            assert [m[:3] for m in plan.moves[t]] == mv, t
            for j in range(p):  # kept = the learner's own samples left after its tail moves
                sent = sum(m[2] for m in mv if m[0] == j)
                assert plan.kept[t][j] == plan.counts[t][j] - sent


def test_headline_plan_regular_scheme_vs_reference():
    """cfg4's comparator at the headline shape: the regular scheme's lists are
    reg_slice (sampling.cpp:27-42) of every batch of the epoch."""
    d, p, B = 1280000, 8, 8192
    plan = ll.plan_epoch(42, 0, d, p, B, scheme="regular")
    order = oracle.ref_permute_epoch(42, 0, d) if oracle.ref_available() else \
        oracle.permute_epoch(42, 0, d)
    for t in [0, 1, 77, 155]:
        for j in range(p):
            want = order[t * B + j * (B // p):t * B + (j + 1) * (B // p)]
            assert np.array_equal(plan.lists(t)[j], want)
    assert int(plan.totals[0]) == 0


def test_remote_per_epoch_reference_goldens(golden):
    """golden remote_per_epoch: Loc moved / Reg remote of whole epochs, counted
    by running the reference, equal the device plan's totals."""
    for c in golden["remote_per_epoch"]:
        plan = ll.plan_epoch(c["seed"], c["epoch"], c["d"], c["p"], c["B"], with_ids=False)
        assert int(plan.totals[0]) == c["loc_moved"], c
        assert int(plan.totals[3]) == c["reg_remote"], c


@pytest.mark.parametrize("scheme,alpha,p,B", [("locality_balanced", 0.4, 3, 999),
                                               ("locality", 0.75, 5, 640),
                                               ("regular", 0.5, 4, 512)])
def test_plan_epoch_partial_cache_vs_oracle(scheme, alpha, p, B):
    """ll_plan_epoch with alpha < 1 and the other schemes: every step's final
    lists equal the C oracle's assignment of the same permutation."""
    d, seed, epoch = 30000, 9, 1
    plan = ll.plan_epoch(seed, epoch, d, p, B, alpha=alpha, scheme=scheme)
    order = oracle.permute_epoch(seed, epoch, d)
    cached = oracle.cached_count(d, alpha)
    mode = {"regular": oracle.MODE_REGULAR, "locality": oracle.MODE_LOCALITY,
            "locality_balanced": oracle.MODE_LOCALITY_BALANCED}[scheme]
    uncached = 0
    for t in range(plan.steps):
        r = oracle.assign_step(order[t * B:(t + 1) * B], p, cached, mode)
        assert np.array_equal(plan.final_ids[t], r["final_ids"]), t
        assert np.array_equal(plan.final_off[t], r["final_off"]), t
        uncached += int(np.sum(order[t * B:(t + 1) * B] >= cached))
    assert int(plan.totals[2]) == uncached


def test_plan_epoch_errors():
    with pytest.raises(_capi.InvalidArgument, match="batches: batch size must be in"):
        ll.plan_epoch(1, 0, 10, 2, 11)
    with pytest.raises(_capi.InvalidArgument, match="reg_slice: learner count must divide"):
        ll.plan_epoch(1, 0, 100, 3, 10, scheme="regular")
    with pytest.raises(_capi.InvalidArgument, match="cached fraction"):
        ll.plan_epoch(1, 0, 100, 2, 10, alpha=0.0)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_loader_cfg1_outputs_vs_oracle(dtype):
    """Four learners on one GPU (P2P exchange over shared HBM): each learner's
    augmented batch equals the oracle's augment of its final list."""
    d, p, B = 10000, 4, 256
    lds = make_learners(d, p, B, dtype=dtype)
    order = oracle.permute_epoch(42, 1, d)
    for t in [0, 7, 38]:
        r = oracle.assign_step(order[t * B:(t + 1) * B], p, d, oracle.MODE_LOCALITY_BALANCED)
        for j, ld in enumerate(lds):
            info = ld.step(1, t)
            lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]]
            assert np.array_equal(ld.fetch_ids(info), lst)
            assert info.kept == r["kept"][j] and info.n_local == len(lst)
            got = ld.fetch(info)
            src = oracle.gen_samples(42, lst, 256 * 256 * 3)
            for k, sid in enumerate(lst):
                want = oracle.augment(src[k].reshape(256, 256, 3), int(sid), 42, 1,
                                      bf16=dtype == "bf16")
                assert np.array_equal(got[k], want), (t, j, k)


def test_loader_regular_scheme_outputs():
    d, p, B = 4096, 2, 128
    lds = make_learners(d, p, B, scheme="regular")
    order = oracle.permute_epoch(42, 0, d)
    for t in [0, 5]:
        batch = order[t * B:(t + 1) * B]
        for j, ld in enumerate(lds):
            info = ld.step(0, t)
            lst = batch[j * B // p:(j + 1) * B // p]
            assert np.array_equal(ld.fetch_ids(info), lst)
            got = ld.fetch(info)
            src = oracle.gen_samples(42, lst, 256 * 256 * 3)
            for k, sid in enumerate(lst):
                assert np.array_equal(got[k], oracle.augment(src[k].reshape(256, 256, 3),
                                                             int(sid), 42, 0))


def test_loader_host_step_equals_device_step():
    """The reference-facing host call (GlobalBatch in, local ids out) delivers
    exactly what the device-planned step delivers."""
    d, p, B = 8192, 2, 512
    lds = make_learners(d, p, B)
    order = ll.permute_epoch(42, 2, d).order
    for t in [0, 3]:
        batch = np.ascontiguousarray(order[t * B:(t + 1) * B])
        for ld in lds:
            dev = ld.step(2, t)
            a = ld.fetch(dev)
            out_ids = np.empty(B, np.uint64)
            host = ld.step_host(2, t, batch, out_ids)
            assert host.n_local == dev.n_local and host.kept == dev.kept
            assert np.array_equal(out_ids[:host.n_local], ld.fetch_ids(dev))
            assert np.array_equal(ld.fetch(host), a)


def test_loader_run_epoch_report():
    """pipeline.hpp:55-64 accounting over a whole epoch (test_pipeline.cpp:125-133)."""
    lds = make_learners(2000, 2, 64)
    reps = [ld.run_epoch(0) for ld in lds]
    assert all(r.batches == 31 for r in reps)
    assert sum(r.samples for r in reps) == 31 * 64
    assert all(r.cache_hits + r.cache_misses == r.samples for r in reps)
    assert all(len(r.batch_latency_s) == 31 for r in reps)


def test_loader_config_errors():
    with pytest.raises(ValueError, match="CacheDirectory: cached fraction"):
        DeviceLoader(LoaderConfig(alpha=1.5))
    with pytest.raises(ValueError, match="batches: batch size"):
        DeviceLoader(LoaderConfig(d=10, batch_size=11))
    with pytest.raises(ValueError, match="reg_slice"):
        DeviceLoader(LoaderConfig(d=100, learners=3, batch_size=10, scheme="regular"))
    with pytest.raises(ValueError, match="Loader: workers, parallelism"):
        DeviceLoader(LoaderConfig(prefetch_depth=0))
    ld = DeviceLoader(LoaderConfig(d=1000, learners=2, batch_size=100))
    with pytest.raises(ValueError, match="not populated"):
        ld.step(0, 0)
    ld.populate()
    with pytest.raises(ValueError, match="exchange"):
        for t in range(10):
            ld.step(0, t)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_loader_variable_size_resize_vs_oracle(dtype):
    """cfg5: variable 128-512 px sources (geometry from the id), bilinear resize
    to 224, two learners with P2P exchange; every delivered sample equals the
    oracle's restatement bit for bit (tolerance 1 ulp bf16 / 1e-5 fp32)."""
    d, p, B, seed = 3000, 2, 96, 42
    lds = []
    for j in range(p):
        ld = DeviceLoader(LoaderConfig(d=d, height=0, width=0, learners=p, rank=j, batch_size=B,
                                       seed=seed, data_seed=seed, exchange="p2p",
                                       geometry="variable",
                                       augment=AugmentConfig(mode="resize", out_dtype=dtype)))
        ld.populate()
        lds.append(ld)
    DeviceLoader.link_peers(lds)
    order = oracle.permute_epoch(seed, 2, d)
    for t in [0, 9]:
        r = oracle.assign_step(order[t * B:(t + 1) * B], p, d, oracle.MODE_LOCALITY_BALANCED)
        for j, ld in enumerate(lds):
            info = ld.step(2, t)
            lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]]
            assert np.array_equal(ld.fetch_ids(info), lst)
            got = ld.fetch(info)
            for k, sid in enumerate(lst[:24]):
                H, W = oracle.sample_hw(seed, int(sid))
                src = oracle.gen_sample(seed, int(sid), H * W * 3).reshape(H, W, 3)
                want = oracle.augment(src, int(sid), seed, 2, mode=oracle.AUG_RESIZE,
                                      bf16=dtype == "bf16")
                if dtype == "fp32":
                    assert np.abs(got[k] - want).max() <= FP32_TOL
                else:
                    assert bf16_ulps(got[k], want) <= 1
                assert np.array_equal(got[k], want), (t, j, k, H, W)


def test_loader_variable_size_consecutive_steps_prefetched_prologue():
    """cfg5 over consecutive steps: from step 1 on, K7's prologue (per-sample
    geometry and the pull of far windows from the peer's shard) was issued on
    the side stream under the previous step's augment.  A host-path step in
    between (its own buffer set) must not disturb the prefetched one."""
    d, p, B, seed, epoch = 2400, 2, 64, 7, 1
    lds = []
    for j in range(p):
        ld = DeviceLoader(LoaderConfig(d=d, height=0, width=0, learners=p, rank=j, batch_size=B,
                                       seed=seed, data_seed=seed, exchange="p2p",
                                       geometry="variable",
                                       augment=AugmentConfig(mode="resize", out_dtype="bf16")))
        ld.populate()
        lds.append(ld)
    DeviceLoader.link_peers(lds)
    order = oracle.permute_epoch(seed, epoch, d)

    def check(got, lst, kept):
        ks = sorted(set(range(min(3, len(lst)))) | set(range(kept, len(lst))))
        for k in ks:
            sid = int(lst[k])
            H, W = oracle.sample_hw(seed, sid)
            src = oracle.gen_sample(seed, sid, H * W * 3).reshape(H, W, 3)
            want = oracle.augment(src, sid, seed, epoch, mode=oracle.AUG_RESIZE, bf16=True)
            assert np.array_equal(got[k], want), (k, sid, H, W)

    far = 0
    for t in range(6):
        r = oracle.assign_step(order[t * B:(t + 1) * B], p, d, oracle.MODE_LOCALITY_BALANCED)
        if t == 3:  # host path on learner 0 between two device-planned steps
            ids = np.empty(B, np.uint64)
            lds[0].submit_host(epoch, t, order[t * B:(t + 1) * B])
            info = lds[0].wait_host(ids)
            lst = r["final_ids"][r["final_off"][0]:r["final_off"][1]]
            assert np.array_equal(ids[:info.n_local], lst)
            check(lds[0].fetch(info), lst, info.kept)
        for j, ld in enumerate(lds):
            info = ld.step(epoch, t)
            lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]]
            assert np.array_equal(ld.fetch_ids(info), lst)
            check(ld.fetch(info), lst, info.kept)
            far += len(lst) - info.kept
    assert far > 0  # the steps really pulled windows from the peer
    for ld in lds:
        ld.close()


def test_loader_host_submit_wait_pipelined():
    """Prefetching host API (prefetch_depth 2): in-order delivery, identical
    to the synchronous call and to the device-planned step."""
    d, p, B = 8192, 2, 512
    lds = make_learners(d, p, B)
    order = ll.permute_epoch(42, 4, d).order
    ld = lds[0]
    want = []
    for t in range(5):
        want.append(ld.fetch_ids(ld.step(4, t)).copy())
    ld.submit_host(4, 0, order[0:B])
    ld.submit_host(4, 1, order[B:2 * B])
    with pytest.raises(ValueError, match="outstanding"):
        ld.submit_host(4, 2, order[2 * B:3 * B])
    ids = np.empty(B, np.uint64)
    for t in range(5):
        info = ld.wait_host(ids)
        assert info.step == t
        assert np.array_equal(ids[:info.n_local], want[t])
        assert info.h2d_bytes == 8 * B and info.d2h_bytes >= 8 * info.n_local
        if t + 2 < 5:
            ld.submit_host(4, t + 2, order[(t + 2) * B:(t + 3) * B])
    with pytest.raises(ValueError, match="no host step"):
        ld.wait_host(ids)


def test_loader_host_batch_validation():
    """A caller's GlobalBatch is range-checked before the device reads the
    shard with it: ids >= d, a short batch or a too-small out_ids buffer are
    refused (nothing is queued), and the loader stays usable afterwards."""
    d, p, B = 4096, 2, 256
    lds = make_learners(d, p, B)
    ld = lds[0]
    order = ll.permute_epoch(42, 0, d).order
    bad = order[:B].copy()
    bad[17] = d
    with pytest.raises(_capi.InvalidArgument, match="out of range"):
        ld.submit_host(0, 0, bad)
    bad[17] = 2 ** 32 + 5  # would truncate to a valid u32 id on the device
    with pytest.raises(_capi.InvalidArgument, match="out of range"):
        ld.submit_host(0, 0, bad)
    with pytest.raises(_capi.InvalidArgument, match="batch_size"):
        ld.submit_host(0, 0, order[:B - 1])
    with pytest.raises(_capi.InvalidArgument, match="out_ids"):
        ld.step_host(0, 0, order[:B], np.empty(B - 1, np.uint64))
    with pytest.raises(_capi.InvalidArgument, match="out_ids"):
        ld.step_host(0, 0, order[:B], np.empty(B, np.int64))
    ids = np.empty(B, np.uint64)
    info = ld.step_host(0, 0, order[:B], ids)
    r = oracle.assign_step(order[:B], p, d, oracle.MODE_LOCALITY_BALANCED)
    assert np.array_equal(ids[:info.n_local], r["final_ids"][r["final_off"][0]:r["final_off"][1]])


@pytest.mark.parametrize("p,alpha", [(1, 0.25), (2, 0.5), (3, 0.37)])
def test_loader_storage_tier_vs_oracle(p, alpha):
    """alpha < 1 (cfg3): uncached samples are dealt round-robin (counts as the
    reference, order as DESIGN.md section 3) and read from the pinned host
    storage tier; every learner's batch equals the oracle's."""
    d, B, seed = 3000, 120, 42
    lds = []
    for j in range(p):
        ld = DeviceLoader(LoaderConfig(d=d, learners=p, rank=j, batch_size=B, alpha=alpha,
                                       seed=seed, data_seed=seed, exchange="p2p"))
        ld.populate()
        lds.append(ld)
    if p > 1:
        DeviceLoader.link_peers(lds)
    cached = oracle.cached_count(d, alpha)
    order = oracle.permute_epoch(seed, 1, d)
    for t in [0, 13]:
        r = oracle.assign_step(order[t * B:(t + 1) * B], p, cached, oracle.MODE_LOCALITY_BALANCED)
        for j, ld in enumerate(lds):
            info = ld.step(1, t)
            lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]]
            assert np.array_equal(ld.fetch_ids(info), lst)
            assert info.uncached == int((order[t * B:(t + 1) * B] >= cached).sum())
            got = ld.fetch(info)
            src = oracle.gen_samples(seed, lst, 256 * 256 * 3)
            for k, sid in enumerate(lst):
                want = oracle.augment(src[k].reshape(256, 256, 3), int(sid), seed, 1)
                assert np.array_equal(got[k], want), (t, j, k, int(sid) >= cached)


def test_loader_resize_far_sources_vs_oracle():
    """K7 with far sources: a peer's shard (P2P) and the host storage tier
    (alpha < 1) are pulled into local HBM before the tap gathers; every
    delivered sample equals the oracle (fixed 256 x 256 sources, resize to
    160 x 192)."""
    d, p, B, seed, alpha = 3000, 2, 120, 42, 0.5
    aug = AugmentConfig(mode="resize", out_h=160, out_w=192)
    lds = []
    for j in range(p):
        ld = DeviceLoader(LoaderConfig(d=d, learners=p, rank=j, batch_size=B, alpha=alpha,
                                       seed=seed, data_seed=seed, exchange="p2p", augment=aug))
        ld.populate()
        lds.append(ld)
    DeviceLoader.link_peers(lds)
    cached = oracle.cached_count(d, alpha)
    order = oracle.permute_epoch(seed, 1, d)
    far = 0
    for t in [0, 7]:
        r = oracle.assign_step(order[t * B:(t + 1) * B], p, cached, oracle.MODE_LOCALITY_BALANCED)
        for j, ld in enumerate(lds):
            info = ld.step(1, t)
            lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]]
            assert np.array_equal(ld.fetch_ids(info), lst)
            got = ld.fetch(info)
            src = oracle.gen_samples(seed, lst, 256 * 256 * 3)
            for k, sid in enumerate(lst):
                far += int(int(sid) >= cached or k >= info.kept)
                want = oracle.augment(src[k].reshape(256, 256, 3), int(sid), seed, 1, 160, 192,
                                      mode=oracle.AUG_RESIZE)
                assert np.array_equal(got[k], want), (t, j, k)
    assert far > 0


def test_loader_populate_from_reference_files(tmp_path):
    """Cache population from a dataset written by the REFERENCE's
    generate_dataset (oracle/_ref): the learner serves exactly the oracle's
    samples; missing and truncated files raise errors naming the sample like
    read_sample (test_pipeline.cpp:177-192)."""
    import os
    d, p, B, seed = 600, 2, 64, 9
    root = str(tmp_path / "ds")
    oracle._ref_check(oracle.ref().ref_generate_dataset(root.encode(), d, 256 * 256 * 3, seed))
    lds = []
    for j in range(p):
        ld = DeviceLoader(LoaderConfig(d=d, learners=p, rank=j, batch_size=B, seed=seed,
                                       data_seed=seed, exchange="p2p"))
        ld.populate_from_files(root, threads=4)
        lds.append(ld)
    DeviceLoader.link_peers(lds)
    order = oracle.permute_epoch(seed, 0, d)
    r = oracle.assign_step(order[:B], p, d, oracle.MODE_LOCALITY_BALANCED)
    for j, ld in enumerate(lds):
        info = ld.step(0, 0)
        lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]]
        got = ld.fetch(info)
        src = oracle.gen_samples(seed, lst, 256 * 256 * 3)
        for k, sid in enumerate(lst):
            assert np.array_equal(got[k], oracle.augment(src[k].reshape(256, 256, 3), int(sid), seed, 0))
    os.remove(os.path.join(root, "00000017.bin"))
    with open(os.path.join(root, "00000403.bin"), "wb") as f:
        f.write(b"xy")
    ld0 = DeviceLoader(LoaderConfig(d=d, learners=2, rank=0, batch_size=B))
    with pytest.raises(RuntimeError, match="sample 17: cannot open"):
        ld0.populate_from_files(root)
    ld1 = DeviceLoader(LoaderConfig(d=d, learners=2, rank=1, batch_size=B))
    with pytest.raises(RuntimeError, match=r"sample 403: truncated file .* \(read 2 of 196608 bytes\)"):
        ld1.populate_from_files(root)


def test_loader_populate_from_files_variable_and_storage(tmp_path):
    """Variable-size files (cfg5 geometry) into the HBM shard, and alpha < 1
    ids into the host storage tier."""
    import os
    d, B, seed = 300, 32, 5
    root = str(tmp_path / "var")
    os.makedirs(root)
    for s in range(d):
        h, w = oracle.sample_hw(seed, s)
        with open(os.path.join(root, f"{s:08d}.bin"), "wb") as f:
            f.write(oracle.gen_sample(seed, s, h * w * 3).tobytes())
    ld = DeviceLoader(LoaderConfig(d=d, height=0, width=0, batch_size=B, seed=seed, data_seed=seed,
                                   geometry="variable",
                                   augment=AugmentConfig(mode="resize", out_dtype="bf16")))
    ld.populate_from_files(root)
    info = ld.step(1, 2)
    lst = ld.fetch_ids(info)
    got = ld.fetch(info)
    for k, sid in enumerate(lst[:8]):
        h, w = oracle.sample_hw(seed, int(sid))
        src = oracle.gen_sample(seed, int(sid), h * w * 3).reshape(h, w, 3)
        assert np.array_equal(got[k], oracle.augment(src, int(sid), seed, 1, mode=oracle.AUG_RESIZE,
                                                     bf16=True))
    # fixed-size files with a storage tier
    root2 = str(tmp_path / "fix")
    oracle._ref_check(oracle.ref().ref_generate_dataset(root2.encode(), d, 256 * 256 * 3, seed))
    ld2 = DeviceLoader(LoaderConfig(d=d, batch_size=B, alpha=0.4, seed=seed, data_seed=seed))
    ld2.populate_from_files(root2)
    info = ld2.step(0, 1)
    lst = ld2.fetch_ids(info)
    got = ld2.fetch(info)
    assert info.uncached > 0
    src = oracle.gen_samples(seed, lst, 256 * 256 * 3)
    for k, sid in enumerate(lst):
        assert np.array_equal(got[k], oracle.augment(src[k].reshape(256, 256, 3), int(sid), seed, 0))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_torch_handoff_zero_copy_train_step(dtype):
    """Trainer hand-off: the step's batch as a zero-copy
    torch tensor on the loader's GPU, ordered after the loader stream, equal
    to the library's own copy, and usable by a training step."""
    import torch
    ld = make_learners(4096, 1, 128, dtype=dtype)[0]
    info = ld.step(0, 3)
    t = ld.torch_batch(info)
    assert t.shape == (128, 3, 224, 224)
    assert t.dtype == (torch.float32 if dtype == "fp32" else torch.bfloat16)
    assert t.data_ptr() == info.device_out
    host = ld.fetch(info)
    if dtype == "fp32":
        assert np.array_equal(t.cpu().numpy(), host)
    else:
        assert np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), host)
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 8, 7, stride=4), torch.nn.ReLU(),
                              torch.nn.AdaptiveAvgPool2d(1), torch.nn.Flatten(),
                              torch.nn.Linear(8, 10)).cuda()
    loss = net(t.float()).logsumexp(1).mean()
    loss.backward()
    assert torch.isfinite(loss).item()
    assert all(p.grad is not None for p in net.parameters())


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_dlpack_handoff(dtype):
    """The C-ABI's DLPack export (ll_loader_batch_dlpack): a framework-neutral
    zero-copy view of the step's batch, taken here by torch.utils.dlpack."""
    import torch
    import torch.utils.dlpack
    ld = make_learners(4096, 1, 128, dtype=dtype)[0]
    info = ld.step(0, 5)
    stream = torch.cuda.ExternalStream(ld.stream_ptr(), device=torch.device("cuda", 0))
    torch.cuda.current_stream().wait_stream(stream)
    t = torch.utils.dlpack.from_dlpack(ld.dlpack_batch(info))
    assert t.shape == (128, 3, 224, 224) and t.is_cuda and t.is_contiguous()
    assert t.dtype == (torch.float32 if dtype == "fp32" else torch.bfloat16)
    assert t.data_ptr() == info.device_out
    host = ld.fetch(info)
    if dtype == "fp32":
        assert np.array_equal(t.cpu().numpy(), host)
    else:
        assert np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), host)
    del t  # the view's deleter runs; the loader's memory stays
    assert np.array_equal(ld.fetch(info), host)


# ------------------------------------------------- HBM sample store (SampleCache)
def _store(capacity):
    import ctypes as C
    h = C.c_void_p()
    _capi.check(_capi.lib().ll_store_create(C.byref(h), 0, capacity))
    return h


def _store_insert(h, ids, samples):
    import ctypes as C
    ids = np.ascontiguousarray(ids, np.uint64)
    ptrs = (C.c_void_p * len(ids))(*[s.ctypes.data for s in samples])
    ins = np.zeros(len(ids), np.uint8)
    _capi.check(_capi.lib().ll_store_insert(h, ll.locload.context(), _capi.ptr(ids, C.c_uint64),
                                            len(ids), samples[0].size, ptrs,
                                            _capi.ptr(ins, C.c_uint8)))
    return ins


def test_store_populate_on_first_touch_no_replacement():
    """ll_store_* = SampleCache (pipeline.hpp:68-94) in HBM: inserts beyond the
    capacity are skipped, a held id is never replaced, lookups and gathers
    return the inserted bytes, a gather of an absent id is refused."""
    import ctypes as C
    rng = np.random.default_rng(5)
    S = 3 * 250 * 250  # not a multiple of 16
    samples = [rng.integers(0, 256, S, dtype=np.uint8) for _ in range(6)]
    h = _store(4)
    try:
        assert _store_insert(h, [10, 11, 12], samples[:3]).tolist() == [1, 1, 1]
        # 11 again (other bytes): no replacement; 13 fits; 14 is past capacity
        assert _store_insert(h, [11, 13, 14], samples[3:6]).tolist() == [0, 1, 0]
        n = C.c_uint64()
        _capi.check(_capi.lib().ll_store_size(h, C.byref(n)))
        assert n.value == 4
        ids = np.array([13, 10, 11, 12, 14, 99], np.uint64)
        found = np.zeros(len(ids), np.uint8)
        _capi.check(_capi.lib().ll_store_lookup(h, _capi.ptr(ids, C.c_uint64), len(ids),
                                                _capi.ptr(found, C.c_uint8)))
        assert found.tolist() == [1, 1, 1, 1, 0, 0]
        out = np.empty(4 * S, np.uint8)
        _capi.check(_capi.lib().ll_store_gather(h, ll.locload.context(),
                                                _capi.ptr(ids, C.c_uint64), 4,
                                                _capi.ptr(out, C.c_uint8)))
        want = [samples[4], samples[0], samples[1], samples[2]]
        for k in range(4):
            assert np.array_equal(out[k * S:(k + 1) * S], want[k]), k
        with pytest.raises(_capi.InvalidArgument, match="not held"):
            _capi.check(_capi.lib().ll_store_gather(h, ll.locload.context(),
                                                    _capi.ptr(ids[4:], C.c_uint64), 1,
                                                    _capi.ptr(out, C.c_uint8)))
        with pytest.raises(_capi.InvalidArgument, match="same size"):
            _store_insert(h, [50], [np.zeros(16, np.uint8)])
    finally:
        _capi.lib().ll_store_destroy(h)


def test_store_zero_capacity_and_many_slabs():
    """Capacity 0 never holds anything; 3,000 samples of 1 MB span three
    1-GiB slabs and all gather back intact."""
    import ctypes as C
    h = _store(0)
    try:
        assert _store_insert(h, [1], [np.ones(64, np.uint8)]).tolist() == [0]
    finally:
        _capi.lib().ll_store_destroy(h)
    S = 1 << 20
    h = _store(3000)
    try:
        base = np.arange(S, dtype=np.uint32).astype(np.uint8)
        for c0 in range(0, 3000, 500):
            ids = np.arange(c0, c0 + 500, dtype=np.uint64)
            samples = [np.roll(base, int(i)) for i in ids]
            assert _store_insert(h, ids, samples).all()
        ids = np.array([0, 1023, 1024, 2047, 2048, 2999], np.uint64)
        out = np.empty(len(ids) * S, np.uint8)
        _capi.check(_capi.lib().ll_store_gather(h, ll.locload.context(),
                                                _capi.ptr(ids, C.c_uint64), len(ids),
                                                _capi.ptr(out, C.c_uint8)))
        for k, i in enumerate(ids):
            assert np.array_equal(out[k * S:(k + 1) * S], np.roll(base, int(i))), i
    finally:
        _capi.lib().ll_store_destroy(h)
