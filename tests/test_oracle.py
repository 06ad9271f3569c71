"""Pin the CPU oracle (oracle/locload_oracle.c) before trusting it.

Checked against (a) the known-answer tests of the reference's own suites
(proj/tests/test_*.cpp, cited per test), (b) golden vectors produced by
running the compiled reference (tests/golden/make_golden.py), and (c) the live
reference build when it is present.  CPU only.
"""
import hashlib

import numpy as np
import pytest

import oracle

L = oracle.lib


def test_rng_known_answers(golden):
    g = golden["rng"]
    for z, v in g["mix64"].items():
        assert L().lo_mix64(int(z)) == v
    for s, a, v in g["derive_seed"]:
        assert L().lo_derive_seed(s, a) == v
    for s, a, b, v in g["derive_seed3"]:
        assert L().lo_derive_seed3(s, a, b) == v
    # SURVEY appendix A (measured on the compiled reference)
    assert L().lo_derive_seed(42, 0) == 0x32514187b3135a8e
    assert L().lo_derive_seed3(42, 0, 0) == 0x293560a19ccdf13b


def test_permutations_match_reference_golden(golden):
    for case in golden["permutations"]:
        o = oracle.permute_epoch(case["seed"], case["epoch"], case["d"])
        if "order" in case:
            assert o.tolist() == case["order"], case["d"]
        else:
            assert o[:64].tolist() == case["head"]
            assert hashlib.sha256(o.tobytes()).hexdigest() == case["sha256"]


def test_permutation_appendix_values():
    assert oracle.permute_epoch(42, 0, 10000)[:5].tolist() == [8649, 1, 6490, 1477, 7937]
    assert oracle.permute_epoch(7, 0, 1).tolist() == [0]  # test_core.cpp:12-15


def test_permutation_rejects_empty():
    with pytest.raises(ValueError):  # test_core.cpp:41-44
        oracle.permute_epoch(7, 0, 0)


def test_forced_rejection_is_a_shifted_stream():
    """Forcing draw k to reject makes index k use draw k+1 and every later
    index use draw index + 1 (rng.hpp:41-50 retry)."""
    base = oracle.permute_epoch(5, 0, 1000)
    forced = oracle.permute_epoch(5, 0, 1000, forced=[10])
    assert sorted(forced.tolist()) == list(range(1000))
    assert not np.array_equal(base, forced)
    none = oracle.permute_epoch(5, 0, 1000, forced=[])
    assert np.array_equal(base, none)


def test_assign_balanced_matches_reference_golden(golden):
    for c in golden["assign_balanced"]:
        r = oracle.assign_step(c["batch"], c["p"], c["d"], oracle.MODE_LOCALITY_BALANCED)
        assert r["final_ids"].tolist() == c["lists"]
        assert r["final_off"].tolist() == c["off"]
        assert [m[:3] for m in r["moves"]] == [tuple(m) for m in c["moves"]]


def test_worked_tail_move_example():
    """d=48, p=4, B=16, seed 7, epoch 0, step 0."""
    batch = oracle.permute_epoch(7, 0, 48)[:16]
    assert batch.tolist() == [32, 4, 30, 41, 38, 22, 47, 45, 42, 35, 14, 28, 21, 46, 8, 31]
    r = oracle.assign_step(batch, 4, 48, oracle.MODE_LOCALITY_BALANCED)
    lists = [r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]].tolist() for j in range(4)]
    assert lists == [[4, 8, 42, 46], [22, 14, 21, 31], [32, 30, 35, 28], [41, 38, 47, 45]]
    assert [m[:3] for m in r["moves"]] == [(3, 0, 2), (2, 1, 1)]


def test_loc_distribution_2_6_4():
    """test_sampling.cpp:113-123 (the paper's Fig. 4 split)."""
    batch = [0, 13, 25, 14, 26, 15, 27, 16, 28, 17, 1, 18]
    r = oracle.assign_step(batch, 3, 36, oracle.MODE_LOCALITY)
    lists = [r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]].tolist() for j in range(3)]
    assert r["counts"].tolist() == [2, 6, 4]
    assert lists == [[0, 1], [13, 14, 15, 16, 17, 18], [25, 26, 27, 28]]
    # balanced: test_balance.cpp:55-61 -> one move (1 -> 0, 2)
    r = oracle.assign_step(batch, 3, 36, oracle.MODE_LOCALITY_BALANCED)
    assert [m[:3] for m in r["moves"]] == [(1, 0, 2)]


def test_uncached_round_robin_counts():
    """test_sampling.cpp:195-203: counts_with_uncached == {3, 1, 2}."""
    r = oracle.assign_step([0, 6, 7, 8, 9, 5], 3, 6, oracle.MODE_LOCALITY)
    assert r["counts"].tolist() == [3, 1, 2]
    lists = [r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]].tolist() for j in range(3)]
    # cached first (batch order), then the dealt uncached (6->0, 7->1, 8->2, 9->0)
    assert lists == [[0, 6, 9], [7], [5, 8]]


def test_partial_cache_matches_reference(golden):
    """alpha < 1: cached lists, counts_with_uncached and the schedule equal the
    reference; the dealt-uncached placement is this build's definition."""
    for c in golden["loc_distribution_partial"]:
        cached = oracle.cached_count(c["d"], c["alpha"])
        p = c["p"]
        r = oracle.assign_step(c["batch"], p, cached, oracle.MODE_LOCALITY)
        assert r["counts"].tolist() == c["cwu"]
        U = len(c["uncached"])
        for j in range(p):
            lst = r["final_ids"][r["final_off"][j]:r["final_off"][j + 1]].tolist()
            own = c["counts"][j]
            assert lst[:own] == c["lists"][j]
            assert lst[own:] == c["uncached"][j::p]
        assert sum(U // p + (1 if j < U % p else 0) for j in range(p)) == U
        rb = oracle.assign_step(c["batch"], p, cached, oracle.MODE_LOCALITY_BALANCED)
        assert [m[:3] for m in rb["moves"]] == [tuple(m) for m in c["moves"]]


def test_balance_matches_reference_golden(golden):
    for c in golden["balance"]:
        assert oracle.balance(c["counts"], c["targets"]) == [tuple(m) for m in c["moves"]]


def test_balance_reference_examples():
    assert oracle.targets(13, 3) == [5, 4, 4]  # test_balance.cpp:47-53
    assert oracle.targets(0, 2) == [0, 0]
    assert oracle.balance([2, 6, 4], [4, 4, 4]) == [(1, 0, 2)]
    assert oracle.balance([10, 0, 2], [4, 4, 4]) == [(0, 1, 4), (0, 2, 2)]
    assert oracle.balance([6, 6, 2, 2], [4, 4, 4, 4]) == [(0, 2, 2), (1, 3, 2)]
    assert oracle.balance([4, 4, 4], [4, 4, 4]) == []
    with pytest.raises(ValueError):
        oracle.balance([1, 2], [4, 4])


def test_generated_bytes_match_reference_golden(golden):
    for c in golden["samples"]:
        b = oracle.gen_sample(c["seed"], c["id"], c["bytes"])
        assert b[:32].tobytes().hex() == c["head"]
        assert hashlib.sha256(b.tobytes()).hexdigest() == c["sha256"]


def test_remote_per_epoch_matches_reference(golden):
    """Loc moved samples per epoch from the oracle."""
    for c in golden["remote_per_epoch"][:1]:
        order = oracle.permute_epoch(c["seed"], c["epoch"], c["d"])
        moved = 0
        for t in range(c["d"] // c["B"]):
            r = oracle.assign_step(order[t * c["B"]:(t + 1) * c["B"]], c["p"], c["d"],
                                   oracle.MODE_LOCALITY_BALANCED)
            moved += sum(m[2] for m in r["moves"])
        assert moved == c["loc_moved"]


# ---- augment: cross-check the C restatement against an independent numpy one
def _np_crop(src, prm, bf16):
    y0, x0, ch, cw, flip = prm
    m255, inv = oracle.norm_constants()
    win = src[y0:y0 + ch, x0:x0 + cw, :].astype(np.float32)
    if flip:
        win = win[:, ::-1, :]
    out = ((win - m255[None, None, :]) * inv[None, None, :]).astype(np.float32)
    out = np.ascontiguousarray(out.transpose(2, 0, 1))
    if bf16:
        u = out.view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
        return u.astype(np.uint16)
    return out


@pytest.mark.parametrize("bf16", [False, True])
def test_crop_oracle_matches_numpy(bf16):
    for sid in [0, 1, 17, 12345]:
        src = oracle.gen_sample(42, sid, 256 * 256 * 3).reshape(256, 256, 3)
        prm = oracle.aug_params(42, 3, sid, 256, 256)
        assert prm[2:4] == (224, 224) and 0 <= prm[0] <= 32 and 0 <= prm[1] <= 32
        got = oracle.augment(src, sid, 42, 3, bf16=bf16)
        assert np.array_equal(got, _np_crop(src, prm, bf16))


def test_aug_params_cover_range_and_flip():
    prms = [oracle.aug_params(1, 0, i, 256, 256) for i in range(4000)]
    ys = {p[0] for p in prms}
    xs = {p[1] for p in prms}
    fl = [p[4] for p in prms]
    assert ys == set(range(33)) and xs == set(range(33))
    assert 0.45 < np.mean(fl) < 0.55


def _np_resize(src, prm, out_h, out_w):
    """Independent numpy restatement of the fixed-point bilinear."""
    y0, x0, ch, cw, flip = prm
    m255, inv = oracle.norm_constants()

    def taps(n_out, extent):
        o = np.arange(n_out, dtype=np.int64)
        f = np.maximum((2 * o + 1) * extent * 64 // n_out - 64, 0)
        lo, w = f >> 7, f & 127
        edge = lo >= extent - 1
        lo[edge], w[edge] = extent - 1, 0
        return lo, w, np.where(w > 0, lo + 1, lo)

    ylo, wy, yhi = taps(out_h, ch)
    xlo, wx, xhi = taps(out_w, cw)
    if flip:
        xlo, wx, xhi = xlo[::-1], wx[::-1], xhi[::-1]
    s = src[y0:y0 + ch, x0:x0 + cw].astype(np.int64)
    wy, wx = wy[:, None, None], wx[None, :, None]
    v = ((128 - wy) * (128 - wx) * s[ylo][:, xlo] + (128 - wy) * wx * s[ylo][:, xhi]
         + wy * (128 - wx) * s[yhi][:, xlo] + wy * wx * s[yhi][:, xhi])
    assert v.max() < 2 ** 22
    val = v.astype(np.float32) * np.float32(2.0 ** -14)
    return ((val - m255) * inv).astype(np.float32).transpose(2, 0, 1)


def test_resize_oracle_matches_numpy():
    for sid, (oh, ow) in [(3, (24, 20)), (8, (224, 224)), (11, (300, 7)), (5, (1, 1))]:
        H, W = oracle.sample_hw(42, sid)
        assert 128 <= H <= 512 and 128 <= W <= 512
        src = oracle.gen_sample(42, sid, H * W * 3).reshape(H, W, 3)
        prm = oracle.aug_params(42, 0, sid, H, W, oh, ow, oracle.AUG_RESIZE)
        got = oracle.augment(src, sid, 42, 0, oh, ow, oracle.AUG_RESIZE)
        assert np.array_equal(got, _np_resize(src, prm, oh, ow))


# ---- live reference cross-checks (build container / wherever oracle/_ref exists)
def test_oracle_vs_live_reference_random(ref_lib):
    rng = np.random.default_rng(7)
    for _ in range(200):
        d = int(rng.integers(1, 4000))
        s, e = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, 100))
        assert np.array_equal(oracle.permute_epoch(s, e, d), oracle.ref_permute_epoch(s, e, d))
    for _ in range(300):
        p = int(rng.integers(1, 17))
        d = int(rng.integers(64, 4000))
        B = int(rng.integers(1, min(d, 400)))
        batch = rng.choice(d, B, replace=False).astype(np.uint64)
        r = oracle.assign_step(batch, p, d, oracle.MODE_LOCALITY_BALANCED)
        lists, off, mv = oracle.ref_assign_balanced(batch, d, p)
        assert np.array_equal(r["final_ids"], lists)
        assert r["final_off"].tolist() == off.tolist()
        assert [m[:3] for m in r["moves"]] == mv
        if B % p == 0:
            for j in range(p):
                assert np.array_equal(oracle.ref_reg_slice(batch, p, j),
                                      batch[j * B // p:(j + 1) * B // p])


@pytest.mark.parametrize("bf16", [False, True])
def test_cpu_baseline_step_equals_spec(bf16):
    """The threaded table-driven CPU baseline computes exactly lo_augment_one."""
    pool = np.stack([oracle.gen_sample(42, i, 256 * 256 * 3) for i in range(16)])
    ids = np.array([3, 17, 100, 5, 2 ** 40 + 1], np.uint64)
    per = 3 * 224 * 224
    out = np.empty(len(ids) * per, np.uint16 if bf16 else np.float32)
    oracle.cpu_crop_step(pool, ids, 256, 256, 42, 2, out, bf16, 3)
    for k, sid in enumerate(ids):
        want = oracle.augment(pool[int(sid) % 16].reshape(256, 256, 3), int(sid), 42, 2, bf16=bf16)
        assert np.array_equal(out[k * per:(k + 1) * per].reshape(3, 224, 224), want)
