"""ctypes binding of include/locload_b200.h (the C-ABI of liblocload_b200.so).

Loading fails loudly when the CUDA extension is missing: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LL_LIB", os.path.join(HERE, "liblocload_b200.so"))

LL_OK, LL_ERR_INVALID, LL_ERR_RUNTIME, LL_ERR_CUDA, LL_ERR_NCCL, LL_ERR_UNSUPPORTED = range(6)
SCHEME_REGULAR, SCHEME_LOCALITY, SCHEME_LOCALITY_BALANCED = 0, 1, 2
AGG_CANONICAL, AGG_LEARNER_ORDER = 0, 1
EXCHANGE_NONE, EXCHANGE_NCCL, EXCHANGE_P2P = 0, 1, 2
OUT_F32, OUT_BF16 = 0, 1
AUG_CROP, AUG_RESIZE = 0, 1
GEOM_FIXED, GEOM_VARIABLE = 0, 1

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class Move(C.Structure):
    _fields_ = [("sender", C.c_uint32), ("receiver", C.c_uint32), ("count", C.c_uint32),
                ("src_off", C.c_uint32), ("dst_off", C.c_uint32), ("nvlink", C.c_uint32),
                ("reserved", C.c_uint32 * 2)]


class AugmentSpec(C.Structure):
    _fields_ = [("mode", C.c_int32), ("out_dtype", C.c_int32), ("out_h", C.c_uint32),
                ("out_w", C.c_uint32), ("mean", C.c_double * 3), ("std", C.c_double * 3)]


class LoaderConfig(C.Structure):
    _fields_ = [("d", C.c_uint64), ("height", C.c_uint32), ("width", C.c_uint32),
                ("learners", C.c_uint32), ("rank", C.c_uint32), ("batch_size", C.c_uint64),
                ("alpha", C.c_double), ("seed", C.c_uint64), ("data_seed", C.c_uint64),
                ("scheme", C.c_int32), ("exchange", C.c_int32), ("prefetch_depth", C.c_uint32),
                ("geometry", C.c_uint32), ("augment", AugmentSpec)]


class StepInfo(C.Structure):
    _fields_ = [("epoch", C.c_uint64), ("step", C.c_uint64), ("n_local", C.c_uint64),
                ("kept", C.c_uint64), ("received", C.c_uint64), ("moved_total", C.c_uint64),
                ("nvlink_bytes", C.c_uint64), ("uncached", C.c_uint64),
                ("reg_remote", C.c_uint64), ("device_out", C.c_size_t),
                ("device_ids", C.c_size_t), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64)]


class Xfer(C.Structure):
    _fields_ = [("peer", C.c_uint32), ("is_send", C.c_uint32), ("count", C.c_uint64),
                ("buf_first", C.c_uint64), ("list_first", C.c_uint64)]


class LoaderError(RuntimeError):
    """CUDA / NCCL / unsupported failures of the device path."""


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference."""


# name -> (restype, argtypes)
PROTOTYPES = {
    "ll_version": (C.c_int, []),
    "ll_last_error": (C.c_char_p, []),
    "ll_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ll_ctx_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "ll_ctx_destroy": (C.c_int, [C.c_void_p]),
    "ll_ctx_sync": (C.c_int, [C.c_void_p]),
    "ll_ctx_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "ll_ctx_launch_count": (C.c_int, [C.c_void_p, u64p]),
    "ll_ctx_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "ll_ctx_kernel_stats": (C.c_int, [C.c_void_p, C.c_char_p, u64p, C.POINTER(C.c_double)]),
    "ll_ctx_reset_stats": (C.c_int, [C.c_void_p]),
    "ll_ctx_copy_to_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64]),
    "ll_permute_epoch": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    "ll_permutation_prefix": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_uint64, u64p]),
    "ll_permute_epoch_forced": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, u64p,
                                          C.c_uint64, u64p]),
    "ll_last_permute_rounds": (C.c_int, [C.c_void_p, u32p]),
    "ll_last_permute_profile": (C.c_int, [C.c_void_p, u64p]),
    "ll_assign": (C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double,
                            C.c_int, u64p, u64p, u64p, u64p, C.POINTER(Move), u32p, u64p]),
    "ll_plan_epoch": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                C.c_uint64, C.c_double, C.c_int, u64p, u64p, u64p, u64p, u64p,
                                C.POINTER(Move), u32p, u64p]),
    "ll_balance_batch": (C.c_int, [C.c_void_p, i64p, i64p, C.c_uint32, C.c_uint64,
                                   C.POINTER(Move), u32p]),
    "ll_exchange_plan": (C.c_int, [C.POINTER(Move), C.c_uint32, u64p, C.c_uint32, C.c_uint32,
                                   C.POINTER(Xfer), u32p]),
    "ll_train_run": (C.c_int, [C.c_void_p, f64p, f64p, C.c_uint64, C.c_uint32, C.c_int,
                               C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_int,
                               f64p, f64p]),
    "ll_toy_synthesize": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, f64p, f64p]),
    "ll_full_batch_gradient": (C.c_int, [C.c_void_p, f64p, f64p, C.c_uint64, C.c_uint32, f64p,
                                         u64p, C.c_uint64, f64p]),
    "ll_loader_link_peers": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32]),
    "ll_generate_samples": (C.c_int, [C.c_void_p, C.c_uint64, u64p, C.c_uint64, C.c_uint64,
                                      u8p]),
    "ll_augment": (C.c_int, [C.c_void_p, C.POINTER(AugmentSpec), C.c_uint64, C.c_uint64, u8p,
                             u64p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]),
    "ll_augment_device": (C.c_int, [C.c_void_p, C.POINTER(AugmentSpec), C.c_uint64, C.c_uint64,
                                    C.c_size_t, C.c_size_t, C.c_uint64, C.c_uint32, C.c_uint32,
                                    C.c_size_t]),
    "ll_ctx_enable_peer": (C.c_int, [C.c_void_p, C.c_int]),
    "ll_augment_params": (C.c_int, [C.c_void_p, C.POINTER(AugmentSpec), C.c_uint64, C.c_uint64,
                                    u64p, C.c_uint64, C.c_uint32, C.c_uint32, u32p]),
    "ll_loader_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_void_p,
                                   C.POINTER(LoaderConfig)]),
    "ll_loader_destroy": (C.c_int, [C.c_void_p]),
    "ll_nccl_unique_id": (C.c_int, [u8p]),
    "ll_loader_comm_init": (C.c_int, [C.c_void_p, u8p]),
    "ll_loader_ipc_handle": (C.c_int, [C.c_void_p, u8p]),
    "ll_loader_open_peers": (C.c_int, [C.c_void_p, u8p]),
    "ll_loader_populate": (C.c_int, [C.c_void_p]),
    "ll_loader_populate_from_host": (C.c_int, [C.c_void_p, u8p]),
    "ll_loader_populate_from_files": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint32]),
    "ll_loader_shard_range": (C.c_int, [C.c_void_p, u64p, u64p]),
    "ll_loader_steps_per_epoch": (C.c_int, [C.c_void_p, u64p]),
    "ll_loader_plan_epoch": (C.c_int, [C.c_void_p, C.c_uint64]),
    "ll_loader_step": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(StepInfo)]),
    "ll_loader_step_host": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, u64p, u64p,
                                      C.POINTER(StepInfo)]),
    "ll_loader_submit_host": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, u64p]),
    "ll_loader_wait_host": (C.c_int, [C.c_void_p, u64p, C.POINTER(StepInfo)]),
    "ll_loader_plan_step": (C.c_int, [C.c_void_p, C.c_uint64, u64p, u64p, u64p, u64p,
                                      C.POINTER(Move), u32p]),
    "ll_loader_epoch_totals": (C.c_int, [C.c_void_p, u64p]),
    "ll_loader_batch_dlpack": (C.c_int, [C.c_void_p, C.POINTER(StepInfo), C.POINTER(C.c_void_p)]),
    "ll_loader_exchange_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int]),
    "ll_toy_grads_device": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t, C.c_uint32,
                                      C.c_size_t, C.c_size_t, C.c_uint64, C.c_size_t]),
    "ll_ordered_sum_device": (C.c_int, [C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint32,
                                        C.c_size_t, C.c_size_t]),
    "ll_sgd_apply_device": (C.c_int, [C.c_void_p, C.c_size_t, C.c_uint32, C.c_double,
                                      C.c_double, C.c_size_t, C.c_size_t]),
    "ll_store_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_uint64]),
    "ll_store_destroy": (C.c_int, [C.c_void_p]),
    "ll_store_size": (C.c_int, [C.c_void_p, u64p]),
    "ll_store_sample_bytes": (C.c_int, [C.c_void_p, u64p]),
    "ll_store_lookup": (C.c_int, [C.c_void_p, u64p, C.c_uint64, C.POINTER(C.c_uint8)]),
    "ll_store_insert": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_uint64, C.c_uint64,
                                  C.POINTER(C.c_void_p), C.POINTER(C.c_uint8)]),
    "ll_store_gather": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_uint64,
                                  C.POINTER(C.c_uint8)]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded extension; raises ImportError when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == LL_OK:
        return
    msg = lib().ll_last_error().decode()
    if status == LL_ERR_INVALID:
        raise InvalidArgument(msg)
    if status == LL_ERR_RUNTIME:
        raise RuntimeError(msg)
    raise LoaderError(f"status {status}: {msg}")


def ptr(a, ctype):
    """ctypes pointer to a numpy array's data."""
    return a.ctypes.data_as(C.POINTER(ctype))
