"""Host cost of one device-planned step (ll_loader_step through the Python
binding): a tiny batch keeps the GPU far ahead of the host, so the loop's wall
time per step is the host's.  Measurement aid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

from paper_1910_01196_b200 import _capi  # noqa: E402
from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig  # noqa: E402

for mode, geom, dt in [("crop", "fixed", "fp32"), ("crop", "fixed", "bf16"),
                       ("resize", "variable", "bf16")]:
    ld = DeviceLoader(LoaderConfig(d=64 * 1000, batch_size=64, seed=1, data_seed=1, geometry=geom,
                                   augment=AugmentConfig(mode=mode, out_dtype=dt)))
    ld.populate()
    spe = ld.steps_per_epoch
    for t in range(50):
        ld.step(1 + t // spe, t % spe)
    ld.synchronize() if hasattr(ld, "synchronize") else _capi.lib().ll_ctx_sync(ld.ctx)
    n = 800
    t0 = time.perf_counter()
    for t in range(n):
        ld.step(2 + t // spe, t % spe)
    host = (time.perf_counter() - t0) / n
    _capi.lib().ll_ctx_sync(ld.ctx)
    # the C call alone (no Python StepInfo wrapper): raw ctypes
    info = _capi.StepInfo()
    f = _capi.lib().ll_loader_step
    t0 = time.perf_counter()
    for t in range(n):
        f(ld._h, 20 + t // spe, t % spe, C.byref(info))
    raw = (time.perf_counter() - t0) / n
    _capi.lib().ll_ctx_sync(ld.ctx)
    print(f"{mode}/{dt}: host us per step: python wrapper {host * 1e6:.1f}, raw ctypes {raw * 1e6:.1f}",
          flush=True)
    ld.close()
