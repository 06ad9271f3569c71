"""Python access to the CPU checkers.  TEST INFRASTRUCTURE ONLY.

  lib()  -- oracle/_build/liblocload_oracle.so, the C restatement
            (locload_oracle.c; every function cites the reference file:line)
  ref()  -- oracle/_ref/liblocload_ref.so, the unmodified reference sources
            compiled in place by oracle/Makefile (+ ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this package; the product (paper_1910_01196_b200)
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liblocload_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblocload_ref.so")
REF_SRC = "/root/reference/proj"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
f32p = C.POINTER(C.c_float)

MODE_REGULAR, MODE_LOCALITY, MODE_LOCALITY_BALANCED = 0, 1, 2
AUG_CROP, AUG_RESIZE = 0, 1
IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


class LoMove(C.Structure):
    _fields_ = [("sender", C.c_uint32), ("receiver", C.c_uint32), ("count", C.c_uint64),
                ("src_off", C.c_uint64), ("dst_off", C.c_uint64)]


class LoAugParams(C.Structure):
    _fields_ = [("y0", C.c_uint32), ("x0", C.c_uint32), ("ch", C.c_uint32), ("cw", C.c_uint32),
                ("flip", C.c_uint32)]


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle); the reference part only where the
    reference sources exist (the build container)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_lib = None
_ref = None


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO) or (
                os.path.getmtime(os.path.join(HERE, "locload_oracle.c")) > os.path.getmtime(ORACLE_SO)):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.lo_mix64.restype = C.c_uint64
        L.lo_mix64.argtypes = [C.c_uint64]
        L.lo_derive_seed.restype = C.c_uint64
        L.lo_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.lo_derive_seed3.restype = C.c_uint64
        L.lo_derive_seed3.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.lo_permute_epoch.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.lo_permute_epoch_forced.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p,
                                              C.c_uint64]
        L.lo_cached_count.restype = C.c_uint64
        L.lo_cached_count.argtypes = [C.c_uint64, C.c_double]
        L.lo_owner.restype = C.c_uint32
        L.lo_owner.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        L.lo_owned_begin.restype = C.c_uint64
        L.lo_owned_begin.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64]
        L.lo_targets.argtypes = [C.c_uint64, C.c_uint32, i64p]
        L.lo_balance.argtypes = [i64p, i64p, C.c_uint32, C.POINTER(LoMove)]
        L.lo_assign_step.argtypes = [u64p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, u64p,
                                     u64p, u64p, u64p, C.POINTER(LoMove), u32p]
        L.lo_gen_sample.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u8p]
        L.lo_sample_hw.argtypes = [C.c_uint64, C.c_uint64, u32p, u32p]
        L.lo_aug_params_for.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                        C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                        C.POINTER(LoAugParams)]
        L.lo_norm_constants.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), f32p,
                                        f32p]
        L.lo_bf16_rne.restype = C.c_uint16
        L.lo_bf16_rne.argtypes = [C.c_float]
        L.lo_augment_one.argtypes = [u8p, C.c_uint32, C.c_uint32, C.POINTER(LoAugParams),
                                     C.c_uint32, C.c_uint32, C.c_int, f32p, f32p, C.c_int,
                                     C.c_void_p]
        L.lo_augment_batch_mt.argtypes = [C.POINTER(u8p), u32p, u32p, C.POINTER(LoAugParams),
                                          C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, f32p,
                                          f32p, C.c_int, C.c_void_p, C.c_int]
        L.lo_cpu_crop_step.argtypes = [u8p, C.c_uint64, u64p, C.c_uint64, C.c_uint32,
                                       C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32,
                                       C.c_uint32, f32p, f32p, C.c_int, C.c_void_p, C.c_int]
        L.lo_cpu_resize_step.argtypes = [C.POINTER(u8p), u32p, u32p, C.c_uint64, u64p,
                                         C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                         C.c_uint32, f32p, f32p, C.c_int, C.c_void_p, C.c_int]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_derive_seed3.restype = C.c_uint64
        L.ref_derive_seed3.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_splitmix_draws.argtypes = [C.c_uint64, C.c_uint64, u64p]
        L.ref_splitmix_bounded.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.ref_permute_epoch.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.ref_permutation_prefix.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.ref_batches_count.restype = C.c_int64
        L.ref_batches_count.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_cache_directory.argtypes = [C.c_uint64, C.c_uint32, C.c_double, u64p, u64p]
        L.ref_owner.argtypes = [C.c_uint64, C.c_uint32, C.c_double, u64p, C.c_uint64, u32p]
        L.ref_reg_slice.argtypes = [u64p, C.c_uint64, C.c_uint32, C.c_uint32, u64p]
        L.ref_loc_distribution.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double,
                                           u64p, u64p, u64p, u64p, u64p, u64p]
        L.ref_targets.argtypes = [C.c_int64, C.c_uint32, i64p]
        L.ref_balance.argtypes = [i64p, i64p, C.c_uint32, i64p, C.POINTER(C.c_int)]
        L.ref_optimal_message_count.argtypes = [i64p, i64p, C.c_uint32, C.POINTER(C.c_int)]
        L.ref_deficit_fraction.argtypes = [i64p, i64p, C.c_uint32, C.POINTER(C.c_double)]
        L.ref_assign_balanced.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint32, u64p, u64p,
                                          i64p, C.POINTER(C.c_int)]
        L.ref_generate_dataset.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_sample_path.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64]
        L.ref_loader_epoch.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, C.c_uint64,
                                       C.c_uint64, C.POINTER(C.c_double), u64p, u64p]
        f64p = C.POINTER(C.c_double)
        L.ref_run_training.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.c_uint32,
                                       C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_int,
                                       f64p, f64p]
        L.ref_full_batch_gradient.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, f64p, u64p,
                                              C.c_uint64, f64p]
        L.ref_sample_gradient.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, f64p, C.c_uint64,
                                          f64p, f64p]
        L.ref_simulate_imbalance.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                             C.c_uint64, C.c_double, f64p, f64p]
        _ref = L
    return _ref


class RefError(Exception):
    pass


def _ref_check(rc: int) -> None:
    if rc != 0:
        msg = ref().ref_last_error().decode()
        raise (ValueError if rc == -1 else RuntimeError)(msg)


# ---------------------------------------------------------------- oracle (C)
def permute_epoch(seed: int, epoch: int, d: int, forced=None) -> np.ndarray:
    out = np.empty(max(d, 1), np.uint64)
    if forced is None:
        rc = lib().lo_permute_epoch(seed, epoch, d, _p(out, C.c_uint64))
    else:
        f = np.ascontiguousarray(sorted(forced), dtype=np.uint64)
        rc = lib().lo_permute_epoch_forced(seed, epoch, d, _p(out, C.c_uint64),
                                           _p(f, C.c_uint64), len(f))
    if rc != 0:
        raise ValueError("permute_epoch: dataset must contain at least one sample")
    return out[:d]


def cached_count(d: int, alpha: float) -> int:
    return int(lib().lo_cached_count(d, alpha))


def owned_begin(j: int, p: int, cached: int) -> int:
    return int(lib().lo_owned_begin(j, p, cached))


def assign_step(batch, p: int, cached: int, mode: int) -> dict:
    b = np.ascontiguousarray(batch, dtype=np.uint64)
    B = len(b)
    ids = np.empty(max(B, 1), np.uint64)
    off = np.empty(p + 1, np.uint64)
    kept = np.empty(p, np.uint64)
    counts = np.empty(p, np.uint64)
    moves = (LoMove * max(p, 1))()
    nm = C.c_uint32()
    rc = lib().lo_assign_step(_p(b, C.c_uint64), B, p, cached, mode, _p(ids, C.c_uint64),
                              _p(off, C.c_uint64), _p(kept, C.c_uint64),
                              _p(counts, C.c_uint64), moves, C.byref(nm))
    if rc != 0:
        raise ValueError("assign: invalid arguments")
    return {"final_ids": ids[:B], "final_off": off, "kept": kept, "counts": counts,
            "moves": [(m.sender, m.receiver, m.count, m.src_off, m.dst_off)
                      for m in moves[:nm.value]]}


def targets(b: int, p: int) -> list:
    out = np.empty(p, np.int64)
    lib().lo_targets(b, p, _p(out, C.c_int64))
    return out.tolist()


def balance(counts, tgts) -> list:
    p = len(counts)
    c = np.ascontiguousarray(counts, dtype=np.int64)
    t = np.ascontiguousarray(tgts, dtype=np.int64)
    moves = (LoMove * max(p, 1))()
    n = lib().lo_balance(_p(c, C.c_int64), _p(t, C.c_int64), p, moves)
    if n < 0:
        raise ValueError("balance: counts and targets must sum to the same total")
    return [(m.sender, m.receiver, m.count) for m in moves[:n]]


def gen_sample(data_seed: int, sid: int, nbytes: int) -> np.ndarray:
    out = np.empty(nbytes, np.uint8)
    lib().lo_gen_sample(data_seed, sid, nbytes, _p(out, C.c_uint8))
    return out


def gen_samples(data_seed: int, ids, nbytes: int) -> np.ndarray:
    return np.stack([gen_sample(data_seed, int(i), nbytes) for i in ids]) if len(ids) else \
        np.zeros((0, nbytes), np.uint8)


def sample_hw(data_seed: int, sid: int):
    h, w = C.c_uint32(), C.c_uint32()
    lib().lo_sample_hw(data_seed, sid, C.byref(h), C.byref(w))
    return h.value, w.value


def aug_params(seed, epoch, sid, H, W, out_h=224, out_w=224, mode=AUG_CROP) -> tuple:
    prm = LoAugParams()
    lib().lo_aug_params_for(seed, epoch, sid, H, W, out_h, out_w, mode, C.byref(prm))
    return prm.y0, prm.x0, prm.ch, prm.cw, prm.flip


def norm_constants(mean=IMAGENET_MEAN, std=IMAGENET_STD):
    m = (C.c_double * 3)(*mean)
    s = (C.c_double * 3)(*std)
    m255 = np.empty(3, np.float32)
    inv = np.empty(3, np.float32)
    lib().lo_norm_constants(m, s, _p(m255, C.c_float), _p(inv, C.c_float))
    return m255, inv


def augment(src_hwc: np.ndarray, sid: int, seed: int, epoch: int, out_h=224, out_w=224,
            mode=AUG_CROP, bf16=False, mean=IMAGENET_MEAN, std=IMAGENET_STD) -> np.ndarray:
    """One sample, HWC u8 -> CHW fp32 (or bf16 bits as uint16)."""
    H, W, _ = src_hwc.shape
    src = np.ascontiguousarray(src_hwc, dtype=np.uint8)
    prm = LoAugParams()
    lib().lo_aug_params_for(seed, epoch, sid, H, W, out_h, out_w, mode, C.byref(prm))
    m255, inv = norm_constants(mean, std)
    out = np.empty((3, out_h, out_w), np.uint16 if bf16 else np.float32)
    lib().lo_augment_one(_p(src, C.c_uint8), H, W, C.byref(prm), out_h, out_w, mode,
                         _p(m255, C.c_float), _p(inv, C.c_float), int(bf16),
                         out.ctypes.data_as(C.c_void_p))
    return out


def augment_batch_mt(srcs, Hs, Ws, prms, out_h, out_w, mode, bf16, out, threads,
                     mean=IMAGENET_MEAN, std=IMAGENET_STD) -> None:
    """Multi-threaded CPU augment of n samples (baseline timing)."""
    n = len(srcs)
    ptrs = (u8p * n)(*[s.ctypes.data_as(u8p) for s in srcs])
    H = np.ascontiguousarray(Hs, dtype=np.uint32)
    W = np.ascontiguousarray(Ws, dtype=np.uint32)
    P = (LoAugParams * n)(*[LoAugParams(*p) for p in prms])
    m255, inv = norm_constants(mean, std)
    lib().lo_augment_batch_mt(ptrs, _p(H, C.c_uint32), _p(W, C.c_uint32), P, n, out_h, out_w,
                              mode, _p(m255, C.c_float), _p(inv, C.c_float), int(bf16),
                              out.ctypes.data_as(C.c_void_p), threads)


def cpu_crop_step(pool: np.ndarray, ids: np.ndarray, H: int, W: int, seed: int, epoch: int,
                  out: np.ndarray, bf16: bool, threads: int, out_h=224, out_w=224,
                  mean=IMAGENET_MEAN, std=IMAGENET_STD) -> None:
    """Threaded CPU crop+flip+normalise of one step (CPU baseline)."""
    m255, inv = norm_constants(mean, std)
    i = np.ascontiguousarray(ids, dtype=np.uint64)
    lib().lo_cpu_crop_step(_p(pool, C.c_uint8), pool.shape[0], _p(i, C.c_uint64), len(i), H, W,
                           seed, epoch, out_h, out_w, _p(m255, C.c_float), _p(inv, C.c_float),
                           int(bf16), out.ctypes.data_as(C.c_void_p), threads)


class VarPool:
    """Warm host cache of `n` variable-size samples (ids 0..n-1, true geometry)."""

    def __init__(self, data_seed: int, n: int):
        self.n = n
        self.H = np.empty(n, np.uint32)
        self.W = np.empty(n, np.uint32)
        self.samples = []
        for i in range(n):
            h, w = sample_hw(data_seed, i)
            self.H[i], self.W[i] = h, w
            self.samples.append(gen_sample(data_seed, i, h * w * 3))
        self.ptrs = (u8p * n)(*[a.ctypes.data_as(u8p) for a in self.samples])


def cpu_resize_step(pool: VarPool, ids, seed: int, epoch: int, out: np.ndarray, bf16: bool,
                    threads: int, out_h=224, out_w=224, mean=IMAGENET_MEAN,
                    std=IMAGENET_STD) -> None:
    m255, inv = norm_constants(mean, std)
    i = np.ascontiguousarray(ids, dtype=np.uint64)
    lib().lo_cpu_resize_step(pool.ptrs, _p(pool.H, C.c_uint32), _p(pool.W, C.c_uint32), pool.n,
                             _p(i, C.c_uint64), len(i), seed, epoch, out_h, out_w,
                             _p(m255, C.c_float), _p(inv, C.c_float), int(bf16),
                             out.ctypes.data_as(C.c_void_p), threads)


# ------------------------------------------------------------- reference (C++)
def ref_permute_epoch(seed: int, epoch: int, d: int) -> np.ndarray:
    out = np.empty(max(d, 1), np.uint64)
    _ref_check(ref().ref_permute_epoch(seed, epoch, d, _p(out, C.c_uint64)))
    return out[:d]


def ref_assign_balanced(batch, d: int, p: int):
    b = np.ascontiguousarray(batch, dtype=np.uint64)
    lists = np.empty(max(len(b), 1), np.uint64)
    off = np.empty(p + 1, np.uint64)
    moves = np.empty(3 * max(p, 1), np.int64)
    n = C.c_int()
    _ref_check(ref().ref_assign_balanced(_p(b, C.c_uint64), len(b), d, p, _p(lists, C.c_uint64),
                                         _p(off, C.c_uint64), _p(moves, C.c_int64), C.byref(n)))
    mv = [tuple(int(x) for x in moves[3 * k:3 * k + 3]) for k in range(n.value)]
    return lists[:len(b)], off, mv


def ref_simulate_imbalance(d: int, p: int, local_batch: int, steps: int, seed: int,
                           alpha: float = 1.0):
    """simulate_imbalance (simulate.cpp:42-79): per-step betas and the summary
    {median, q1, q3, whisker_lo, whisker_hi}."""
    betas = np.empty(max(steps, 1), np.float64)
    summ = np.empty(5, np.float64)
    f64p = C.POINTER(C.c_double)
    _ref_check(ref().ref_simulate_imbalance(d, p, local_batch, steps, seed, alpha,
                                            _p(betas, C.c_double), _p(summ, C.c_double)))
    return betas[:steps], summ


def eq8_beta_median(d: int, p: int, local_batch: int, seed: int = 42, steps: int = 500,
                    alpha: float = 1.0) -> float:
    """The predicted beta of Eq. 8 (model.hpp:72-74) the way the reference's
    `locload imbalance` subcommand draws it: simulate_imbalance with `steps`
    (default 500, locload.cpp:152) fresh batches and the per-cell seed
    derive_seed(seed, p, local_batch) (locload.cpp:170); the summary median."""
    s = int(ref().ref_derive_seed3(seed, p, local_batch))
    return float(ref_simulate_imbalance(d, p, local_batch, steps, s, alpha)[1][0])


def ref_loc_distribution(batch, d: int, p: int, alpha: float):
    b = np.ascontiguousarray(batch, dtype=np.uint64)
    B = len(b)
    lists = np.empty(max(B, 1), np.uint64)
    off = np.empty(p + 1, np.uint64)
    unc = np.empty(max(B, 1), np.uint64)
    nunc = C.c_uint64()
    counts = np.empty(p, np.uint64)
    cwu = np.empty(p, np.uint64)
    _ref_check(ref().ref_loc_distribution(_p(b, C.c_uint64), B, d, p, alpha,
                                          _p(lists, C.c_uint64), _p(off, C.c_uint64),
                                          _p(unc, C.c_uint64), C.byref(nunc),
                                          _p(counts, C.c_uint64), _p(cwu, C.c_uint64)))
    return {"lists": [lists[off[j]:off[j + 1]] for j in range(p)],
            "uncached": unc[:nunc.value], "counts": counts, "cwu": cwu}


def ref_balance(counts, tgts) -> list:
    p = len(counts)
    c = np.ascontiguousarray(counts, dtype=np.int64)
    t = np.ascontiguousarray(tgts, dtype=np.int64)
    moves = np.empty(3 * max(p, 1), np.int64)
    n = C.c_int()
    _ref_check(ref().ref_balance(_p(c, C.c_int64), _p(t, C.c_int64), p, _p(moves, C.c_int64),
                                 C.byref(n)))
    return [tuple(int(x) for x in moves[3 * k:3 * k + 3]) for k in range(n.value)]


def ref_targets(b: int, p: int) -> list:
    out = np.empty(max(p, 1), np.int64)
    _ref_check(ref().ref_targets(b, p, _p(out, C.c_int64)))
    return out[:p].tolist()


def ref_reg_slice(batch, p: int, j: int) -> np.ndarray:
    b = np.ascontiguousarray(batch, dtype=np.uint64)
    out = np.empty(max(len(b), 1), np.uint64)
    _ref_check(ref().ref_reg_slice(_p(b, C.c_uint64), len(b), p, j, _p(out, C.c_uint64)))
    return out[:len(b) // p]


def ref_gen_sample(data_seed: int, sid: int, nbytes: int, tmpdir: str) -> np.ndarray:
    """generate_dataset (n = sid + 1 files) then read sample sid back."""
    root = os.path.join(tmpdir, f"ref_{data_seed}_{sid}_{nbytes}")
    _ref_check(ref().ref_generate_dataset(root.encode(), sid + 1, nbytes, data_seed))
    buf = C.create_string_buffer(4096)
    _ref_check(ref().ref_sample_path(root.encode(), sid, buf, 4096))
    with open(buf.value.decode(), "rb") as f:
        return np.frombuffer(f.read(), np.uint8)


# ------------------------------------------------- equivalence (reference)
_SCHEMES = {"regular": 0, "locality": 1, "locality_balanced": 2}


def ref_run_training(n: int, dims: int, obj_seed: int, scheme: str, p: int, b: int, steps: int,
                     seed: int, lr: float, agg: str = "canonical"):
    """The compiled reference's run_training on ToyObjective::synthesize(n, dims,
    obj_seed): (final_weights[dims], step_gradients[steps][dims])."""
    w = np.empty(dims, np.float64)
    g = np.empty((max(steps, 1), dims), np.float64)
    _ref_check(ref().ref_run_training(n, dims, obj_seed, _SCHEMES[scheme], p, b, steps, seed, lr,
                                      0 if agg == "canonical" else 1, _p(w, C.c_double),
                                      _p(g, C.c_double)))
    return w, g[:steps]


def ref_full_batch_gradient(n: int, dims: int, obj_seed: int, w, batch) -> np.ndarray:
    w = np.ascontiguousarray(w, np.float64)
    b = np.ascontiguousarray(batch, np.uint64)
    out = np.empty(dims, np.float64)
    _ref_check(ref().ref_full_batch_gradient(n, dims, obj_seed, _p(w, C.c_double),
                                             _p(b, C.c_uint64), len(b), _p(out, C.c_double)))
    return out


def ref_sample_gradient(n: int, dims: int, obj_seed: int, w, i: int):
    w = np.ascontiguousarray(w, np.float64)
    out = np.empty(dims, np.float64)
    loss = C.c_double()
    _ref_check(ref().ref_sample_gradient(n, dims, obj_seed, _p(w, C.c_double), i,
                                         _p(out, C.c_double), C.byref(loss)))
    return out, loss.value
