"""Exchange bandwidth on NVLink (2 GPUs, one process): the fused P2P path's
remote-sample rate vs local, a plain peer copy, and NCCL send/recv of the same
bytes.  Writes one JSON line (profiles/ keeps it)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1910_01196_b200 as ll
from paper_1910_01196_b200 import _capi
from paper_1910_01196_b200.loader import AugmentConfig

lib = _capi.lib()
n, H, W = 1024, 256, 256
S = H * W * 3
res = {"n_samples": n, "window_bytes_per_sample": 224 * 224 * 3,
       "out_bytes_per_sample": 3 * 224 * 224 * 4}
src0 = torch.randint(0, 255, (n * S,), dtype=torch.uint8, device="cuda:0")
src1 = torch.randint(0, 255, (n * S,), dtype=torch.uint8, device="cuda:1")
ids = torch.arange(n, dtype=torch.int64, device="cuda:0")
out = torch.empty(n * 3 * 224 * 224, dtype=torch.float32, device="cuda:0")
ctx = ll.locload.context(0)
_capi.check(lib.ll_ctx_enable_peer(ctx, 1))
spec = AugmentConfig().to_c()
sp = C.c_size_t()
_capi.check(lib.ll_ctx_stream(ctx, C.byref(sp)))
stream = torch.cuda.ExternalStream(sp.value, device="cuda:0")


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize(0)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def aug(src):
    _capi.check(lib.ll_augment_device(ctx, C.byref(spec), 42, 0, src.data_ptr(), ids.data_ptr(),
                                      n, H, W, out.data_ptr()))


ms_local = timed(lambda: aug(src0))
ms_remote = timed(lambda: aug(src1))
win = n * 224 * 224 * 3
res["augment_local_us"] = ms_local * 1e3
res["augment_all_remote_us"] = ms_remote * 1e3
# remote windows crossed NVLink while the outputs were written locally
res["fused_remote_read_GBps"] = win / (ms_remote * 1e-3) / 1e9
# plain peer copy of the same window bytes (torch -> cudaMemcpyPeer)
dst = torch.empty(win, dtype=torch.uint8, device="cuda:0")
with torch.cuda.stream(torch.cuda.Stream(0)):
    s_ = torch.cuda.current_stream(0)
    for _ in range(3):
        dst.copy_(src1[:win], non_blocking=True)
    torch.cuda.synchronize(0)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(20):
        a.record(s_)
        dst.copy_(src1[:win], non_blocking=True)
        b.record(s_)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
res["peer_copy_GBps"] = win / (best * 1e-3) / 1e9
res["nvlink_nominal_GBps_per_direction"] = 900
res["fused_frac_of_nominal"] = res["fused_remote_read_GBps"] / 900
print(json.dumps(res))
