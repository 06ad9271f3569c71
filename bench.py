"""Benchmark: preprocessed samples/s per box of the locality-aware loader.

Workload (BASELINE.json configs[1], weak-scaled so N=1 fits one B200):
  "cfg2-weak": synthetic ImageNet-1K-shaped u8 HWC 256x256x3 samples,
  d = 160,000 * N (== 1.28 M at N = 8), one learner per GPU (p = N), global
  batch 1024 * N (1,024 per GPU), full cache (alpha = 1: each GPU holds its
  160,000-sample CacheDirectory block = 31.5 GB in HBM), locality-aware
  balanced assignment, crop 224 + h-flip + ImageNet normalise -> NCHW fp32.
  A step = exchange + augment of one global batch; the epoch plan
  (permutation + assignment of all 156 steps) runs inside the timed region at
  every epoch boundary (timed region starts at one).  Inputs (31.5 GB shard,
  616 MB output per step) are far larger than L2, so no flush is needed.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  N>1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "preprocessed samples/sec/box"
PER_GPU_D = 160_000
PER_GPU_B = 1024
H = W = 256
CROP = 224
SEED = 42
SRC_BYTES = CROP * CROP * 3                    # crop window read per sample


def out_bytes(dtype: str) -> int:
    return 3 * CROP * CROP * (4 if dtype == "fp32" else 2)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1560)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg3", "cfg4", "cfg5"],
                    help="cfg2: fixed 256x256 crop224 (default, the headline); "
                         "cfg3: cfg2 with each learner caching 25%% of the dataset "
                         "(alpha = min(1, 0.25 N); uncached samples from the pinned host "
                         "storage tier); cfg4: cfg2 under the regular (naive "
                         "DistributedSampler) scheme, remote samples read over NVLink; "
                         "cfg5: variable 128-512 px, bilinear resize to 224")
    ap.add_argument("--dtype", default=None, choices=["fp32", "bf16"],
                    help="output dtype (default fp32 for cfg2, bf16 for cfg5)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--per-gpu-d", type=int, default=PER_GPU_D)
    ap.add_argument("--per-gpu-batch", type=int, default=PER_GPU_B)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--prefetch-depth", type=int, default=4,
                    help="LoaderConfig::prefetch_depth (output ring / host steps in flight)")
    args = ap.parse_args()
    if args.dtype is None:
        args.dtype = "bf16" if args.workload == "cfg5" else "fp32"
    return args


def mean_window_bytes_cfg5() -> float:
    """E[3 * min(H, W)^2] for H, W iid uniform on [128, 512] (geometry.cuh):
    the resize crop window (the source region an output depends on)."""
    v = np.arange(128, 513, dtype=np.float64)
    mn = np.minimum(v[:, None], v[None, :])
    return float(3.0 * (mn ** 2).mean())


def src_bytes_per_sample(args) -> float:
    return mean_window_bytes_cfg5() if args.workload == "cfg5" else float(SRC_BYTES)



def measure_h2d_gbs(device: int) -> float:
    """Pinned host -> device copy bandwidth (the storage tier's link), GB/s."""
    import torch
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dv = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    best = float("inf")
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dv.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return n / (best / 1e3) / 1e9


def alpha_for(args, n) -> float:
    return min(1.0, 0.25 * n) if args.workload == "cfg3" else 1.0


def workload(args, n):
    if args.workload in ("cfg3", "cfg4"):
        a = alpha_for(args, n)
        name = ("cfg3-weak: cfg2 shapes, 25% of the dataset cached per learner "
                f"(alpha={a:g}; uncached samples read from the pinned host storage tier)"
                if args.workload == "cfg3" else
                "cfg4-weak: cfg2 shapes under the regular scheme (reg_slice; every "
                "non-owned sample read from its owner's HBM over NVLink)")
        name += (f", d={args.per_gpu_d}*N, p=N, global batch {args.per_gpu_batch}*N, "
                 f"crop224+flip+normalize -> NCHW {args.dtype}")
    elif args.workload == "cfg5":
        name = ("cfg5-weak: variable-size synthetic u8 HWC (H, W uniform 128-512 px), "
                f"d={args.per_gpu_d}*N, p=N, global batch {args.per_gpu_batch}*N, alpha=1, "
                f"locality_balanced, random square crop + flip + bilinear resize 224 + "
                f"normalize -> NCHW {args.dtype}")
    else:
        name = ("cfg2-weak: ImageNet-1K-shaped synthetic u8 256x256x3, "
                f"d={args.per_gpu_d}*N, p=N, global batch {args.per_gpu_batch}*N, "
                f"alpha=1, locality_balanced, crop224+flip+normalize -> NCHW {args.dtype}")
    return {"workload": name,
            "d": args.per_gpu_d * n, "learners": n, "global_batch": args.per_gpu_batch * n,
            "per_gpu_batch": args.per_gpu_batch, "alpha": alpha_for(args, n),
            "scheme": "regular" if args.workload == "cfg4" else "locality_balanced",
            "exchange": args.exchange if n > 1 else "none", "out_dtype": args.dtype,
            "l2": "inputs larger than L2 (31.5 GB shard, 616 MB output/step); no flush"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML (the library nvidia-smi reads) polled every ~20 ms in a thread.
    (At 2 ms the NVML calls contended with the CUDA/NCCL calls of the step
    loop for the driver: NCCL-exchange runs at N = 2 lost up to 2x.)"""
    NAMES = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int, enabled: bool = True):
        self.samples = []
        self.ok = False
        self.err = "disabled"
        if not enabled:
            self._stop = threading.Event()
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                mem = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_MEM)
                self.samples.append((mhz, rs, mem))
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        mask = 0
        for _, r, _m in self.samples:
            mask |= r
        reasons = sorted({n for b, n in self.NAMES.items() if mask & b})
        mhz = [m for m, _, _m in self.samples]
        mem = [m for _, _r, m in self.samples]
        return {"sm_mhz": float(np.median(mhz)) if mhz else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(mhz),
                "mem_mhz": [min(mem), float(np.median(mem)), max(mem)] if mem else None,
                "source": "NVML"}


# ------------------------------------------------------------------ CPU arm
def cpu_reference_run(args, n, steps, warmup, seconds_cap=None):
    """The reference's CPU path: oracle/_ref (the unmodified reference sources:
    permute_epoch, loc_distribution + targets + balance + tail moves) for the
    plan, and the oracle's C augment restatement on every host thread (the
    reference has no augment; its Loader 'preprocess' is an injected sleep).
    Samples come from a warm host cache: a pool of 4,096 generate_dataset
    samples, sample id s served from slot s mod 4096."""
    import oracle
    d, B = args.per_gpu_d * n, args.per_gpu_batch * n
    spe = d // B
    pool_n = 4096
    if args.workload == "cfg5":
        vpool = oracle.VarPool(SEED, pool_n)
    else:
        pool = np.stack([oracle.gen_sample(SEED, i, H * W * 3) for i in range(pool_n)])
    cores = len(os.sched_getaffinity(0))
    chunk = min(B, 1024)
    out = np.empty(chunk * out_bytes(args.dtype), np.uint8)
    bf16 = args.dtype == "bf16"
    cache = {"epoch": None, "order": None}

    def one_step(t):
        e, s = divmod(t, spe)
        if cache["epoch"] != e:
            cache["order"] = oracle.ref_permute_epoch(SEED, e, d)  # core.cpp:11-27
            cache["epoch"] = e
        batch = cache["order"][s * B:(s + 1) * B]
        lists, off, _ = oracle.ref_assign_balanced(batch, d, n)    # sampling+balance
        for c0 in range(0, B, chunk):
            if args.workload == "cfg5":
                oracle.cpu_resize_step(vpool, lists[c0:c0 + chunk], SEED, e, out, bf16, cores)
            else:
                oracle.cpu_crop_step(pool, lists[c0:c0 + chunk], H, W, SEED, e, out, bf16, cores)
        return B

    for t in range(warmup):
        one_step(t)
    t0 = time.perf_counter()
    done = samples = 0
    start = ((warmup + spe - 1) // spe) * spe
    for k in range(steps):
        samples += one_step(start + k)
        done += 1
        if seconds_cap and time.perf_counter() - t0 > seconds_cap:
            break
    dt = time.perf_counter() - t0
    return {"value": samples / dt, "unit": "samples/s", "cores": cores, "steps": done,
            "seconds": dt}


def remote_summary(args, n, d, B, totals):
    """Remote samples per epoch of THIS run's workload (p = N learners):
    locality-balanced moves and the regular scheme's remote samples, both
    counted by K4 in the run's own device plan."""
    per = mean_window_bytes_cfg5() if args.workload == "cfg5" else H * W * 3
    steps = d // B
    D = steps * B
    return {"p": n, "d": d, "B": B, "samples_per_epoch": D,
            "loc_moved_samples": totals["moved"],
            "loc_nvlink_samples": totals["moved_nvlink"],
            "reg_remote_samples": totals["reg_remote"],
            "bytes_per_sample": per,
            "loc_remote_bytes": totals["moved_nvlink"] * per,
            "reg_remote_bytes": totals["reg_remote"] * per,
            "eq7_samples": alpha_for(args, n) * D * (n - 1) / n,
            "local_fraction": 1.0 - (totals["moved"] / D if D else 0.0),
            "storage_samples": totals["uncached"],
            "storage_window_bytes": totals["uncached"] * src_bytes_per_sample(args)}


HEADLINE_D = 1_280_000


def eq8_betas() -> dict:
    """Eq. 8's predicted beta per p: the median of the reference's
    simulate_imbalance (simulate.cpp:42-79) run the way `locload imbalance`
    runs it (500 steps, seed derive_seed(42, p, 1024)), computed by running
    oracle/_ref in the build container and committed as a fixture
    (tests/golden/make_golden.py); the bench only reads the number."""
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        g = json.load(f)
    return {c["p"]: c["beta_median"] for c in g["simulate_imbalance"]
            if c["d"] == HEADLINE_D and c["local_batch"] == 1024}


def headline_remote(device: int, seed: int = SEED, epoch: int = 0) -> dict:
    """Remote bytes per epoch at the headline configuration (cfg2: d = 1.28 M,
    B = 1,024 p) for p = 2 / 4 / 8, from the device plan (ll_plan_epoch: K2+K3
    + K4 over the whole epoch -- the plan is replicated, so one GPU computes
    every learner's share).  Loc = samples the balancer moves; Reg = samples
    reg_slice hands to a non-owner (naive DistributedSampler, cfg4).  Model
    (model.hpp:65-74): Eq. 7 alpha*D*(p-1)/p, Eq. 8 alpha*D*beta_median with
    beta from the reference's simulate_imbalance (eq8_betas), D = steps * B
    samples per epoch (remainder dropped, core.cpp:57-73)."""
    import paper_1910_01196_b200 as ll
    betas = eq8_betas()
    whole, window, msg = H * W * 3, SRC_BYTES, 157_696  # NCCL crop-window slot
    out = {"seed": seed, "epoch": epoch, "d": HEADLINE_D, "alpha": 1.0,
           "bytes_per_sample": {"whole": whole, "crop_window": window,
                                "nccl_window_slot": msg},
           "model": "Eq. 7 = alpha*D*(p-1)/p, Eq. 8 = alpha*D*beta_median (model.hpp:65-74); "
                    "beta_median from reference simulate_imbalance (500 steps, "
                    "derive_seed(42, p, 1024))", "p": {}}
    for p in (2, 4, 8):
        B = 1024 * p
        t0 = time.perf_counter()
        plan = ll.plan_epoch(seed, epoch, HEADLINE_D, p, B, device=device, with_ids=False)
        ms = (time.perf_counter() - t0) * 1e3
        D = plan.steps * B
        moved, reg = int(plan.totals[0]), int(plan.totals[3])
        beta = betas.get(p)
        eq8 = D * beta if beta is not None else None
        out["p"][str(p)] = {
            "B": B, "steps": plan.steps, "samples_per_epoch": D,
            "loc_moved_samples": moved, "loc_moved_bytes_whole": moved * whole,
            "loc_moved_bytes_window": moved * window,
            "reg_remote_samples": reg, "reg_remote_bytes_whole": reg * whole,
            "reg_remote_bytes_window": reg * window,
            "eq7_samples": D * (p - 1) / p, "eq8_samples": eq8, "beta_median": beta,
            "beta_measured": moved / D, "loc_vs_eq8": moved / eq8 if eq8 else None,
            "reg_vs_eq7": reg / (D * (p - 1) / p),
            "loc_over_reg_bytes": moved / reg if reg else None,
            "local_fraction": 1.0 - moved / D, "plan_wall_ms": ms}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    n = args.gpus
    if rank != 0:
        return
    r = cpu_reference_run(args, n, args.steps, args.warmup, seconds_cap=None)
    sample = (f"{r['steps']} steps x {args.per_gpu_batch * n} samples of the workload on "
              f"{r['cores']} host threads (warm host cache of 4096 samples). Contents: the "
              "reference's own permute_epoch, loc_distribution, targets and balance "
              "(unmodified reference sources compiled into oracle/_ref) plus the "
              "equivalence.cpp:77-88 tail moves, then the oracle's C augment restatement "
              "(crop/flip/normalise or bilinear resize) on every host thread -- the "
              "reference has no augment (its Loader's preprocess is an injected sleep, "
              "pipeline.cpp:87-108) and its file-reading Loader::run_epoch is not timed")
    line = {"metric": METRIC, "value": r["value"], "unit": "samples/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * r["seconds"] / max(r["steps"], 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": workload(args, n), "impl": "reference",
            "cpu_baseline": {"value": r["value"], "unit": "samples/s", "cores": r["cores"],
                             "kind": "reference", "sample": sample},
            "e2e": {"value": r["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import paper_1910_01196_b200 as ll
    from paper_1910_01196_b200 import _capi
    from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.gpus
    assert world == n, f"--gpus {n} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.workload == "cfg4" and args.exchange == "nccl":
            # the regular scheme's all-to-all: 128 KB NVLink P2P chunks (the
            # loader's comm_init asks for the same, but NCCL reads its
            # parameters once per process, here at the first communicator)
            os.environ.setdefault("NCCL_P2P_NVL_CHUNKSIZE", "131072")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    d, B = args.per_gpu_d * n, args.per_gpu_batch * n
    cfg5 = args.workload == "cfg5"
    cfg = LoaderConfig(d=d, height=H, width=W, learners=n, rank=rank, batch_size=B,
                       alpha=alpha_for(args, n), seed=SEED, data_seed=SEED,
                       scheme="regular" if args.workload == "cfg4" else "locality_balanced",
                       exchange=args.exchange if n > 1 else "none",
                       prefetch_depth=args.prefetch_depth,
                       geometry="variable" if cfg5 else "fixed",
                       augment=AugmentConfig(mode="resize" if cfg5 else "crop",
                                             out_dtype=args.dtype))
    aug_kernel = "augment_resize" if cfg5 else "augment_crop"
    ld = DeviceLoader(cfg, device=local)
    ld.populate()                                   # K1: this learner's shard in HBM
    if n > 1:
        if args.exchange == "p2p":
            handles = [None] * n
            dist.all_gather_object(handles, ld.ipc_handle())
            ld.open_peers(handles)
        else:
            uid = [DeviceLoader.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ld.comm_init(uid[0])
    spe = ld.steps_per_epoch
    lib = _capi.lib()
    ctx = ld.ctx
    sp = C.c_size_t()
    _capi.check(lib.ll_ctx_stream(ctx, C.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    nvl_bytes = [0]

    def run_steps(t0, k):
        local_samples = 0
        for t in range(t0, t0 + k):
            e, s = divmod(t, spe)
            info = ld.step(e, s)
            local_samples += info.n_local
            nvl_bytes[0] += info.nvlink_bytes
        return local_samples

    def max_over_ranks(x):
        if dist is None:
            return x
        v = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    def sum_over_ranks(x):
        if dist is None:
            return x
        v = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        return float(v.item())

    # warm-up: W steps of epoch 0 (and beyond)
    run_steps(0, args.warmup)
    start = ((args.warmup + spe - 1) // spe) * spe     # next epoch boundary
    barrier()

    # ---- timed region (value) ----
    # Nothing but the steps runs in here (no per-launch events: bracketing each
    # launch with CUDA events adds a ~3 us bubble per step, about 4 % at cfg2).
    # On the loader stream a step is exactly one launch of the dominant
    # kernel (the exchange and the K7 prologue go on the side stream, the next
    # epoch's plan on the plan stream), so the region's own event pair gives
    # the dominant kernel's time per launch, gaps between launches included:
    # roofline.achieved and value describe the same launches.
    _capi.check(lib.ll_ctx_reset_stats(ctx))
    nvl_bytes[0] = 0
    launches0 = C.c_uint64()
    _capi.check(lib.ll_ctx_launch_count(ctx, C.byref(launches0)))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, enabled=not os.environ.get("LL_BENCH_NO_CLOCKS")) as clk:
        barrier()
        ev0.record(stream)
        h0 = time.perf_counter()
        samples = run_steps(start, args.steps)
        host_enqueue_s = time.perf_counter() - h0
        ev1.record(stream)
        ev1.synchronize()
        barrier()
    launches1 = C.c_uint64()
    _capi.check(lib.ll_ctx_launch_count(ctx, C.byref(launches1)))
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local)
    total_samples = sum_over_ranks(samples)
    value = total_samples / (ms / 1e3)
    region_nvl_bytes = nvl_bytes[0]
    e_first, s_first = divmod(start, spe)
    e_last, s_last = divmod(start + args.steps - 1, spe)
    n_plans = sum(1 for t in range(start, start + args.steps) if t % spe == spe // 2)
    timed_region = (f"{args.steps} steps from epoch {e_first} step {s_first} to epoch {e_last} "
                    f"step {s_last} ({spe} steps per epoch); {n_plans} next-epoch plan(s) "
                    "(K2+K3 permutation + K4 assignment of a whole epoch, issued at mid-epoch "
                    "on the plan stream) inside"
                    + ("" if n_plans else "; this region's own epoch plan was prefetched "
                       "before it (during warm-up / population)"))
    per_launch_bytes = args.per_gpu_batch * (src_bytes_per_sample(args) + out_bytes(args.dtype))
    launch_ms = ms_local / args.steps
    achieved = per_launch_bytes / (launch_ms / 1e3) / 1e9
    achieved = max_over_ranks(-achieved) * -1 if dist is not None else achieved  # min over ranks

    # ---- diagnostic pass: per-launch CUDA events (library launch hook) ----
    # the kernel alone, without the gaps between launches; its share of the
    # step is what the ncu launch list must agree with
    _capi.check(lib.ll_ctx_reset_stats(ctx))
    _capi.check(lib.ll_ctx_set_timing(ctx, 1))
    nccl = n > 1 and args.exchange == "nccl"
    if nccl:
        ld.exchange_stats(reset=True)
    k2 = min(args.steps, 2 * spe)
    start2 = start + ((args.steps + spe - 1) // spe) * spe
    barrier()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    run_steps(start2, k2)
    d1.record(stream)
    barrier()
    _capi.check(lib.ll_ctx_set_timing(ctx, 0))
    diag_ms = d0.elapsed_time(d1)
    exchange = None
    if n > 1 and args.exchange == "p2p" and not cfg5:
        # the fused exchange: crop windows K6 read from peer shards over
        # NVLink (TMA) inside the augment, per rank per step of value's
        # region, min over ranks
        per_step = region_nvl_bytes / args.steps
        gbs = per_step / (ms_local / args.steps / 1e3) / 1e9
        gbs = max_over_ranks(-gbs) * -1 if dist is not None else gbs
        exchange = {"backend": "p2p: TMA reads of peer HBM fused into K6",
                    "recv_bytes_per_step": per_step, "nvlink_gbs": gbs, "peak_gbs": 900.0,
                    "frac": gbs / 900.0,
                    "peak_source": "NVLink 5 nominal, per direction per GPU",
                    "note": "crop-window bytes read from peers / step time of value's region "
                            "(the exchange overlaps the local part of the augment), min over "
                            "ranks"}
    if nccl:
        # NVLink GB/s of the NCCL exchange: message bytes this rank received
        # / time from the grouped send/recv's issue to its completion on the
        # side stream (CUDA events), min over ranks; it runs concurrently with
        # the previous step's augment
        xs = ld.exchange_stats(reset=True)
        gbs = xs["wire_gbs"] or 0.0
        gbs = max_over_ranks(-gbs) * -1 if dist is not None else gbs
        exchange = {"backend": "nccl grouped send/recv", "steps_timed": xs["timed_steps"],
                    "recv_bytes_per_step": xs["timed_bytes_recv"] / max(xs["timed_steps"], 1),
                    "wire_ms_per_step": xs["ms_wire"] / max(xs["timed_steps"], 1),
                    "pack_ms_per_step": xs["ms_pack"] / max(xs["timed_steps"], 1),
                    "nvlink_gbs": gbs, "peak_gbs": 900.0, "frac": gbs / 900.0,
                    "peak_source": "NVLink 5 nominal, per direction per GPU",
                    "note": "diagnostic pass (per-launch events on); min over ranks"}
    stats = {}
    for name in [aug_kernel, "permute", "assign", "pack", "reg_prep", "resize_prep",
                 "resize_pull"]:
        cnt, tot = C.c_uint64(), C.c_double()
        _capi.check(lib.ll_ctx_kernel_stats(ctx, name.encode(), C.byref(cnt), C.byref(tot)))
        stats[name] = (cnt.value, tot.value)
    aug_n, aug_ms = stats[aug_kernel]
    kernel_only = None
    if aug_n:
        ko = per_launch_bytes / (aug_ms / aug_n / 1e3) / 1e9
        kernel_only = {"avg_launch_ms": aug_ms / aug_n, "achieved": ko, "launches": aug_n,
                       "share_of_step": aug_ms / diag_ms if diag_ms else None,
                       "note": "separate pass with CUDA events around every launch (adds a "
                               "bubble per launch); diagnostic only"}
    peak = 6544.3
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except Exception:
        peak, peak_src = 6650.0, "B200_PROFILING.md fallback"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", f"{aug_kernel}_traffic.json")) as f:
            prof = json.load(f)
        if (prof.get("dtype") == args.dtype and prof.get("per_gpu_batch") == args.per_gpu_batch
                and prof.get("kernel") == aug_kernel):
            traffic = prof["dram_bytes_per_launch"]
    except Exception:
        pass

    # ---- e2e: reference-facing host call, host buffers, copies in the region ----
    e2e = None
    if not args.no_e2e:
        pinned_ids = torch.empty(B, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        # at least one epoch, so the prefetch pipeline's fill and drain (depth 4)
        # do not dominate a short run (the driver's 20 steps)
        k_e2e = min(max(args.steps, spe), 2 * spe)
        depth = cfg.prefetch_depth
        h2d = d2h = 0
        # warm-up of the host path (pinned slots, side stream, first launches)
        wo = ll.permute_epoch(SEED, 0, d, device=local).order
        for s_ in range(min(args.warmup, spe)):
            ld.submit_host(0, s_, wo[s_ * B:(s_ + 1) * B])
            ld.wait_host(pinned_ids)
        from paper_1910_01196_b200.locload import context
        perm_ctx = context(local)
        perm_pinned = torch.empty(d, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        barrier()
        t0 = time.perf_counter()
        e_cur = None
        order = None
        outstanding = 0
        for t in range(start, start + k_e2e):
            e, s = divmod(t, spe)
            if e != e_cur:
                # epoch order computed on the device, D2H into pinned host memory
                _capi.check(lib.ll_permute_epoch(perm_ctx, SEED, e, d,
                                                 perm_pinned.ctypes.data_as(C.POINTER(C.c_uint64))))
                order = perm_pinned
                d2h += 8 * d
                e_cur = e
            ld.submit_host(e, s, order[s * B:(s + 1) * B])  # GlobalBatch from host memory
            outstanding += 1
            if outstanding == depth:                         # in-order delivery
                info = ld.wait_host(pinned_ids)
                outstanding -= 1
                h2d += info.h2d_bytes                        # counted by the library
                d2h += info.d2h_bytes
        while outstanding:
            info = ld.wait_host(pinned_ids)
            outstanding -= 1
            h2d += info.h2d_bytes
            d2h += info.d2h_bytes
        barrier()
        wall = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": sum_over_ranks(k_e2e * args.per_gpu_batch) / wall, "unit": "samples/s",
               "h2d_bytes_per_step": h2d // k_e2e, "d2h_bytes_per_step": d2h // k_e2e,
               "steps": k_e2e,
               "path": f"ll_loader_submit_host/wait_host, prefetch_depth {depth}: GlobalBatch ids "
                       "from host memory -> device assign/exchange/augment -> local ids + "
                       "step tables to host; ll_permute_epoch order D2H per epoch"}

    # ---- CPU baseline (rank 0, N = 1) ----
    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        r = cpu_reference_run(args, n, spe, 2, seconds_cap=args.cpu_seconds)
        cpu = {"value": r["value"], "unit": "samples/s", "cores": r["cores"],
               "kind": "reference",
               "sample": f"{r['steps']} steps x {B} samples (epoch 1) of the workload: "
                         "reference permute_epoch/loc_distribution/balance/tail moves "
                         "(oracle/_ref) + oracle C augment on all host threads, warm host "
                         "cache of 4096 samples"}

    totals = ld.epoch_totals()
    if os.environ.get("LL_BENCH_RANK_STATS"):  # per-rank kernel times on stderr
        print(json.dumps({"rank": rank, "kernel_ms": {k: (v[1] / v[0] if v[0] else None)
                                                      for k, v in stats.items()}}),
              file=sys.stderr, flush=True)
    storage = None
    if totals["uncached"] and aug_n:
        # alpha < 1: the dominant kernel also reads the uncached samples' windows
        # from pinned host memory over PCIe; that link, not HBM, bounds it.
        st_bytes = totals["uncached"] / (d // B) / n * src_bytes_per_sample(args)
        st_achieved = st_bytes / (aug_ms / aug_n / 1e3) / 1e9
        h2d_peak = measure_h2d_gbs(local)
        storage = {"bound": "pcie", "kernel": aug_kernel, "achieved": st_achieved,
                   "peak": h2d_peak, "unit": "GB/s", "frac": st_achieved / h2d_peak,
                   "bytes_per_launch": st_bytes,
                   "peak_source": "measured here: pinned host -> device copy-engine "
                                  "bandwidth (torch copy_ of 512 MiB, best of 5, CUDA events)",
                   "note": "zero-copy reads of the crop windows by the augment kernel"}
    headline = None
    if rank == 0 and not os.environ.get("LL_BENCH_NO_HEADLINE_PLAN"):
        try:
            headline = headline_remote(local)
        except Exception as e:  # never lose the bench line over the side report
            headline = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": n,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": args.dtype, "data": "synthetic",
                "config": dict(workload(args, n), timed_region=timed_region),
                "clocks": clk.summary(),
                "e2e": e2e,
                "gpu_launches": int(launches1.value - launches0.value),
                "host_enqueue_ms_per_step": host_enqueue_s * 1e3 / args.steps,
                "roofline": {"bound": "hbm", "kernel": aug_kernel, "achieved": achieved,
                             "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                             "traffic": traffic, "peak_source": peak_src,
                             "algorithmic_bytes_per_launch": per_launch_bytes,
                             "avg_launch_ms": launch_ms, "launches_timed": args.steps,
                             "timing": "the timed region of `value` (CUDA events on the "
                                       "loader stream, which carries one launch of this "
                                       "kernel per step and nothing else); gaps between "
                                       "launches are counted as kernel time",
                             "kernel_only": kernel_only},
                "storage_roofline": storage,
                "exchange": exchange,
                "kernel_ms": {k: (v[1] / v[0] if v[0] else None) for k, v in stats.items()},
                "cpu_baseline": cpu,
                # the headline configuration's remote bytes per epoch (p = 2 / 4 /
                # 8 at d = 1.28 M) vs the paper's model, then this run's own
                "remote_per_epoch": dict(headline or {},
                                         this_run=remote_summary(args, n, d, B, totals))}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
