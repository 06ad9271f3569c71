"""DeviceLoader: one learner of the locality-aware loader on one GPU.

Mirrors Loader / LoaderConfig / ThroughputReport (proj/include/locload/
pipeline.hpp:46-123) for a device-resident consumer: the learner's shard of
the dataset lives in HBM (its CacheDirectory block, sampling.cpp:19-25), the
epoch plan is computed on the device, and every step delivers this learner's
augmented NCHW batch in HBM.  All work runs through include/locload_b200.h.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _capi
from ._capi import InvalidArgument, check, ptr
from .locload import context

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


@dataclass
class AugmentConfig:
    mode: str = "crop"          # "crop" (cfg1/2) | "resize" (cfg5)
    out_dtype: str = "fp32"     # "fp32" | "bf16"
    out_h: int = 224
    out_w: int = 224
    mean: tuple = IMAGENET_MEAN
    std: tuple = IMAGENET_STD

    def to_c(self) -> _capi.AugmentSpec:
        s = _capi.AugmentSpec()
        s.mode = {"crop": _capi.AUG_CROP, "resize": _capi.AUG_RESIZE}[self.mode]
        s.out_dtype = {"fp32": _capi.OUT_F32, "bf16": _capi.OUT_BF16}[self.out_dtype]
        s.out_h, s.out_w = self.out_h, self.out_w
        for c in range(3):
            s.mean[c] = self.mean[c]
            s.std[c] = self.std[c]
        return s


@dataclass
class LoaderConfig:
    """pipeline.hpp:46-53 plus the device fields."""
    d: int = 10000
    height: int = 256
    width: int = 256
    learners: int = 1
    rank: int = 0
    batch_size: int = 256          # GLOBAL batch (pipeline.hpp:50)
    alpha: float = 1.0
    seed: int = 42
    data_seed: int = 42
    scheme: str = "locality_balanced"
    exchange: str = "none"         # "none" | "nccl" | "p2p"
    prefetch_depth: int = 2
    geometry: str = "fixed"        # "fixed" (height x width) | "variable" (cfg5, 128-512 px)
    augment: AugmentConfig = field(default_factory=AugmentConfig)

    def to_c(self) -> _capi.LoaderConfig:
        c = _capi.LoaderConfig()
        c.d, c.height, c.width = self.d, self.height, self.width
        c.learners, c.rank, c.batch_size = self.learners, self.rank, self.batch_size
        c.alpha, c.seed, c.data_seed = self.alpha, self.seed, self.data_seed
        c.scheme = {"regular": 0, "locality": 1, "locality_balanced": 2}[self.scheme]
        c.exchange = {"none": 0, "nccl": 1, "p2p": 2}[self.exchange]
        c.prefetch_depth = self.prefetch_depth
        c.geometry = {"fixed": 0, "variable": 1}[self.geometry]
        c.augment = self.augment.to_c()
        return c

    @property
    def sample_bytes(self) -> int:
        return self.height * self.width * 3


@dataclass
class ThroughputReport:  # pipeline.hpp:55-64
    epoch: int = 0
    batches: int = 0
    samples: int = 0
    wall_s: float = 0.0
    samples_per_second: float = 0.0
    cache_hits: int = 0            # samples served from this learner's shard
    cache_misses: int = 0          # samples received from other learners
    batch_latency_s: List[float] = field(default_factory=list)


class DeviceLoader:
    def __init__(self, cfg: LoaderConfig, device: int = 0):
        self.cfg = cfg
        self.device = device
        self.ctx = context(device)
        self._h = C.c_void_p()
        self._c = cfg.to_c()
        check(_capi.lib().ll_loader_create(C.byref(self._h), self.ctx, C.byref(self._c)))

    def close(self) -> None:
        if self._h:
            _capi.lib().ll_loader_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- bootstrap -----------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(_capi.lib().ll_nccl_unique_id(buf))
        return bytes(buf)

    def comm_init(self, uid: bytes) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(_capi.lib().ll_loader_comm_init(self._h, buf))

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        check(_capi.lib().ll_loader_ipc_handle(self._h, buf))
        return bytes(buf)

    def open_peers(self, handles: List[bytes]) -> None:
        raw = b"".join(handles)
        buf = (C.c_uint8 * len(raw)).from_buffer_copy(raw)
        check(_capi.lib().ll_loader_open_peers(self._h, buf))

    @staticmethod
    def link_peers(loaders: List["DeviceLoader"]) -> None:
        """Same-process learners: share shard pointers for exchange="p2p"."""
        arr = (C.c_void_p * len(loaders))(*[ld._h.value for ld in loaders])
        check(_capi.lib().ll_loader_link_peers(arr, len(loaders)))

    def populate(self) -> None:
        check(_capi.lib().ll_loader_populate(self._h))

    def populate_from_files(self, root: str, threads: int = 0) -> None:
        """Cache population from the reference's on-disk dataset
        (<root>/%08llu.bin, generate_dataset); errors name the sample."""
        check(_capi.lib().ll_loader_populate_from_files(self._h, root.encode(), threads))

    def populate_from_host(self, samples: np.ndarray) -> None:
        a = np.ascontiguousarray(samples, dtype=np.uint8)
        check(_capi.lib().ll_loader_populate_from_host(self._h, ptr(a, C.c_uint8)))

    def shard_range(self):
        f, n = C.c_uint64(), C.c_uint64()
        check(_capi.lib().ll_loader_shard_range(self._h, C.byref(f), C.byref(n)))
        return f.value, n.value

    @property
    def steps_per_epoch(self) -> int:
        n = C.c_uint64()
        check(_capi.lib().ll_loader_steps_per_epoch(self._h, C.byref(n)))
        return n.value

    # -- epoch / step --------------------------------------------------------
    def plan_epoch(self, epoch: int) -> None:
        check(_capi.lib().ll_loader_plan_epoch(self._h, epoch))

    def step(self, epoch: int, step: int) -> _capi.StepInfo:
        info = _capi.StepInfo()
        check(_capi.lib().ll_loader_step(self._h, epoch, step, C.byref(info)))
        return info

    def _host_batch(self, batch) -> np.ndarray:
        b = np.ascontiguousarray(batch, dtype=np.uint64)
        if b.ndim != 1 or b.size != self.cfg.batch_size:
            raise InvalidArgument(f"Loader: a global batch holds batch_size = "
                                  f"{self.cfg.batch_size} ids (got {b.size})")
        return b

    def _out_ids(self, out_ids: np.ndarray) -> np.ndarray:
        # the library writes up to batch_size u64 ids
        if (not isinstance(out_ids, np.ndarray) or out_ids.dtype != np.uint64 or
                not out_ids.flags.c_contiguous or out_ids.size < self.cfg.batch_size):
            raise InvalidArgument("Loader: out_ids must be a contiguous uint64 array of at "
                                  f"least batch_size = {self.cfg.batch_size} elements")
        return out_ids

    def step_host(self, epoch: int, step: int, batch: np.ndarray, out_ids: np.ndarray):
        b, o = self._host_batch(batch), self._out_ids(out_ids)
        info = _capi.StepInfo()
        check(_capi.lib().ll_loader_step_host(self._h, epoch, step, ptr(b, C.c_uint64),
                                              ptr(o, C.c_uint64), C.byref(info)))
        return info

    def submit_host(self, epoch: int, step: int, batch: np.ndarray) -> None:
        """Queue one host-driven step (at most prefetch_depth outstanding)."""
        b = self._host_batch(batch)
        check(_capi.lib().ll_loader_submit_host(self._h, epoch, step, ptr(b, C.c_uint64)))

    def wait_host(self, out_ids: np.ndarray):
        """Deliver the oldest outstanding host step: (info) with out_ids filled."""
        o = self._out_ids(out_ids)
        info = _capi.StepInfo()
        check(_capi.lib().ll_loader_wait_host(self._h, ptr(o, C.c_uint64), C.byref(info)))
        return info

    def plan_step(self, step: int):
        B, p = self.cfg.batch_size, self.cfg.learners
        ids = np.empty(B, np.uint64)
        off = np.empty(p + 1, np.uint64)
        kept = np.empty(p, np.uint64)
        counts = np.empty(p, np.uint64)
        moves = (_capi.Move * max(p, 1))()
        nm = C.c_uint32()
        check(_capi.lib().ll_loader_plan_step(self._h, step, ptr(ids, C.c_uint64),
                                              ptr(off, C.c_uint64), ptr(kept, C.c_uint64),
                                              ptr(counts, C.c_uint64), moves, C.byref(nm)))
        mv = [(m.sender, m.receiver, m.count, m.src_off, m.dst_off, m.nvlink)
              for m in moves[:nm.value]]
        return ids, off, kept, counts, mv

    def epoch_totals(self) -> dict:
        out = np.zeros(4, np.uint64)
        check(_capi.lib().ll_loader_epoch_totals(self._h, ptr(out, C.c_uint64)))
        return {"moved": int(out[0]), "moved_nvlink": int(out[1]), "uncached": int(out[2]),
                "reg_remote": int(out[3])}

    def exchange_stats(self, reset: bool = False) -> dict:
        """NCCL exchange accounting (ll_loader_exchange_stats)."""
        out = (C.c_double * 8)()
        check(_capi.lib().ll_loader_exchange_stats(self._h, out, 1 if reset else 0))
        r = {"steps": int(out[0]), "bytes_sent": int(out[1]), "bytes_recv": int(out[2]),
             "timed_steps": int(out[3]), "timed_bytes_recv": int(out[4]), "ms_pack": out[5],
             "ms_wire": out[6]}
        r["wire_gbs"] = (r["timed_bytes_recv"] / (r["ms_wire"] / 1e3) / 1e9
                         if r["ms_wire"] > 0 else None)
        return r

    def fetch(self, info: _capi.StepInfo) -> np.ndarray:
        """Host copy of a step's augmented batch [n_local, 3, out_h, out_w]
        (bf16 comes back as raw uint16 bits)."""
        a = self.cfg.augment
        dt = np.float32 if a.out_dtype == "fp32" else np.uint16
        out = np.empty((info.n_local, 3, a.out_h, a.out_w), dt)
        if info.n_local:
            check(_capi.lib().ll_ctx_copy_to_host(self.ctx, out.ctypes.data_as(C.c_void_p),
                                                  info.device_out, out.nbytes))
        return out

    def stream_ptr(self) -> int:
        sp = C.c_size_t()
        check(_capi.lib().ll_ctx_stream(self.ctx, C.byref(sp)))
        return sp.value

    def torch_batch(self, info: _capi.StepInfo):
        """Zero-copy torch view of a step's augmented batch ([n, 3, H, W] on this
        GPU; float32 or bfloat16) -- the trainer hand-off.  torch's current
        stream is made to wait for the loader stream, so the tensor can be used
        right away; it stays valid until prefetch_depth later steps."""
        import torch
        a = self.cfg.augment
        shape = (int(info.n_local), 3, a.out_h, a.out_w)

        class _View:  # __cuda_array_interface__ (v3) over the library's buffer
            __cuda_array_interface__ = {
                "shape": shape, "typestr": "<f4" if a.out_dtype == "fp32" else "<u2",
                "data": (int(info.device_out), False), "version": 3, "strides": None}

        dev = torch.device("cuda", self.device)
        t = torch.as_tensor(_View(), device=dev)
        if a.out_dtype == "bf16":
            t = t.view(torch.bfloat16)
        loader_stream = torch.cuda.ExternalStream(self.stream_ptr(), device=dev)
        torch.cuda.current_stream(dev).wait_stream(loader_stream)
        return t

    def dlpack_batch(self, info: _capi.StepInfo):
        """The same batch through the C-ABI's DLPack export
        (ll_loader_batch_dlpack): a "dltensor" PyCapsule any DLPack consumer
        takes, e.g. torch.utils.dlpack.from_dlpack(capsule).  Order the
        consumer's stream after stream_ptr() before reading."""
        out = C.c_void_p()
        check(_capi.lib().ll_loader_batch_dlpack(self._h, C.byref(info), C.byref(out)))
        new_capsule = C.pythonapi.PyCapsule_New
        new_capsule.restype = C.py_object
        new_capsule.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        return new_capsule(out, b"dltensor", None)

    def fetch_ids(self, info: _capi.StepInfo) -> np.ndarray:
        out = np.empty(info.n_local, np.uint32)
        if info.n_local:
            check(_capi.lib().ll_ctx_copy_to_host(self.ctx, out.ctypes.data_as(C.c_void_p),
                                                  info.device_ids, out.nbytes))
        return out.astype(np.uint64)

    def sync(self) -> None:
        check(_capi.lib().ll_ctx_sync(self.ctx))

    def run_epoch(self, epoch: int,
                  consumer: Optional[Callable[[_capi.StepInfo], None]] = None
                  ) -> ThroughputReport:
        """Loader::run_epoch (pipeline.cpp:247-336) for a device consumer: every
        step of the epoch in order; the consumer sees each step's StepInfo
        (device_out / device_ids point at this learner's batch in HBM)."""
        rep = ThroughputReport(epoch=epoch, batches=self.steps_per_epoch)
        t0 = time.perf_counter()
        for s in range(rep.batches):
            ts = time.perf_counter()
            info = self.step(epoch, s)
            if consumer is not None:
                self.sync()
                consumer(info)
            rep.samples += info.n_local
            rep.cache_hits += info.kept
            rep.cache_misses += info.received
            rep.batch_latency_s.append(time.perf_counter() - ts)
        self.sync()
        rep.wall_s = time.perf_counter() - t0
        rep.samples_per_second = rep.samples / rep.wall_s if rep.wall_s > 0 else 0.0
        return rep
