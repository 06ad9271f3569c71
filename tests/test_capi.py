"""The C-ABI library: builds, loads, exports every symbol include/locload_b200.h
declares, fails loudly without a GPU, and its pure-host exchange planning is
right.  CPU only (no compute call reaches a device)."""
import ctypes as C
import re
import os

import numpy as np
import pytest

import oracle
from paper_1910_01196_b200 import _capi

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                   "locload_b200.h")


def declared_symbols():
    return sorted(set(re.findall(r"\b(ll_[a-z0-9_]+)\s*\(", open(HDR).read())))


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    names = declared_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_capi.PROTOTYPES)
    assert lib.ll_version() == 1


def test_library_is_sm100a_only():
    so = _capi.LIB_PATH
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_gpu_means_loud_failure():
    lib = _capi.lib()
    n = C.c_int(-1)
    lib.ll_device_count(C.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    rc = lib.ll_ctx_create(C.byref(h), 0)
    assert rc == _capi.LL_ERR_CUDA
    with pytest.raises(_capi.LoaderError):
        from paper_1910_01196_b200 import permute_epoch
        permute_epoch(1, 0, 10)


def exchange_plan(moves, off, p, me):
    mv = (_capi.Move * max(len(moves), 1))()
    for i, m in enumerate(moves):
        mv[i].sender, mv[i].receiver, mv[i].count = m[0], m[1], m[2]
        mv[i].src_off, mv[i].dst_off = m[3], m[4]
    o = np.ascontiguousarray(off, dtype=np.uint64)
    out = (_capi.Xfer * max(2 * len(moves), 1))()
    n = C.c_uint32()
    _capi.check(_capi.lib().ll_exchange_plan(mv, len(moves), _capi.ptr(o, C.c_uint64), p, me,
                                             out, C.byref(n)))
    return [(x.peer, x.is_send, x.count, x.buf_first, x.list_first) for x in out[:n.value]]


def test_exchange_plan_delivers_the_tail_moves():
    """For random steps, applying every learner's planned sends/recvs to the
    oracle's pre-balance lists reproduces the oracle's final lists."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        p = int(rng.integers(2, 9))
        d = int(rng.integers(200, 5000))
        B = int(rng.integers(p, min(d, 600)))
        batch = rng.choice(d, B, replace=False).astype(np.uint64)
        r = oracle.assign_step(batch, p, d, oracle.MODE_LOCALITY_BALANCED)
        final, off, kept = r["final_ids"], r["final_off"], r["kept"]
        sendbufs = {}
        for me in range(p):
            buf = []
            for peer, is_send, cnt, bf, lf in exchange_plan(r["moves"], off, p, me):
                if is_send:
                    assert bf == len(buf)
                    buf.extend(final[lf:lf + cnt].tolist())
                    assert all(oracle.lib().lo_owner(int(s), p, d) == me
                               for s in final[lf:lf + cnt])
            sendbufs[me] = buf
        for me in range(p):
            recv = []
            sent_so_far = {j: 0 for j in range(p)}
            for peer, is_send, cnt, bf, lf in exchange_plan(r["moves"], off, p, me):
                if not is_send:
                    # the peer's sends to `me` appear in its buffer in schedule order
                    peer_plan = [x for x in exchange_plan(r["moves"], off, p, peer)
                                 if x[1] and x[0] == me]
                    x = peer_plan[sent_so_far[peer]]
                    sent_so_far[peer] += 1
                    assert bf == len(recv) and lf == off[me] + kept[me] + bf
                    recv.extend(sendbufs[peer][x[3]:x[3] + x[2]])
            lst = final[off[me]:off[me + 1]].tolist()
            assert lst[int(kept[me]):] == recv


def test_exchange_plan_rejects_bad_rank():
    with pytest.raises(_capi.InvalidArgument):
        exchange_plan([], [0, 1], 1, 3)


def test_toy_synthesize_matches_reference():
    """ll_toy_synthesize (host-only) reproduces ToyObjective::synthesize
    (equivalence.cpp:12-37): the reference's sample gradients and losses
    recomputed from our data agree bit for bit."""
    import oracle
    from paper_1910_01196_b200 import locload as ll
    n, dims, seed = 200, 8, 5
    obj = ll.ToyObjective.synthesize(n, dims, seed)
    rng = np.random.default_rng(0)
    for i in [0, 1, 99, 199]:
        w = rng.standard_normal(dims)
        g, loss = oracle.ref_sample_gradient(n, dims, seed, w, i)
        x = obj.xs[i]
        dot = 0.0
        for k in range(dims):
            dot = dot + w[k] * x[k]
        r = dot - obj.ys[i]
        assert np.array_equal(np.array([r * x[k] for k in range(dims)]), g)
        assert 0.5 * r * r == loss
    with pytest.raises(ValueError, match="need n >= 1"):
        ll.ToyObjective.synthesize(0, 8, 1)
