"""Where does augment_crop's time go?  Kernel times (CUDA events via the
library's per-kernel timing) under varied source locality / output dtype."""
import ctypes as C
import json
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1910_01196_b200 as ll
from paper_1910_01196_b200 import _capi
from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig

lib = _capi.lib()
ctx = ll.locload.context(0)


def kstat(name="augment_crop"):
    n, t = C.c_uint64(), C.c_double()
    _capi.check(lib.ll_ctx_kernel_stats(ctx, name.encode(), C.byref(n), C.byref(t)))
    return t.value / max(n.value, 1) * 1e3, n.value


res = {}
for d, B in [(160000, 1024), (16384, 1024), (2048, 1024), (1024, 1024), (512, 512)]:
    for dt in ["fp32", "bf16"]:
        ld = DeviceLoader(LoaderConfig(d=d, batch_size=B, augment=AugmentConfig(out_dtype=dt)))
        ld.populate()
        spe = ld.steps_per_epoch
        for t in range(4):
            ld.step(0, t % spe)
        ld.sync()
        _capi.check(lib.ll_ctx_reset_stats(ctx))
        _capi.check(lib.ll_ctx_set_timing(ctx, 1))
        for t in range(40):
            ld.step(1 + t // spe, t % spe)
        _capi.check(lib.ll_ctx_set_timing(ctx, 0))
        us, n = kstat()
        per = B * (150528 + 3 * 224 * 224 * (4 if dt == "fp32" else 2))
        res[f"d={d},B={B},{dt}"] = {"us": round(us, 2), "GBps": round(per / us / 1e3, 1)}
        ld.close()
        print(json.dumps(res), flush=True)
