"""Host-path probe (1 GPU, cfg2 shapes): per-call host time of submit_host /
wait_host and the e2e rate at prefetch depth 1/2/4, beside the device-planned
rate.  Measurement aid only."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_01196_b200 as ll  # noqa: E402
from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig  # noqa: E402

d, B, seed = 160_000, 1024, 42
for depth in (1, 2, 4):
    ld = DeviceLoader(LoaderConfig(d=d, batch_size=B, seed=seed, data_seed=seed, prefetch_depth=depth,
                                   augment=AugmentConfig(out_dtype="fp32")))
    ld.populate()
    spe = ld.steps_per_epoch
    order = ll.permute_epoch(seed, 1, d).order
    ids = np.empty(B, np.uint64)
    for s in range(8):
        ld.submit_host(1, s, order[s * B:(s + 1) * B])
        ld.wait_host(ids)
    n = 150
    ts, tw = [], []
    t0 = time.perf_counter()
    out = 0
    for s in range(n):
        a = time.perf_counter()
        ld.submit_host(1, s, order[s * B:(s + 1) * B])
        ts.append(time.perf_counter() - a)
        out += 1
        if out == depth:
            a = time.perf_counter()
            ld.wait_host(ids)
            tw.append(time.perf_counter() - a)
            out -= 1
    while out:
        ld.wait_host(ids)
        out -= 1
    wall = time.perf_counter() - t0
    # device-planned steps for comparison
    for s in range(4):
        ld.step(2, s)
    ld.sync() if hasattr(ld, "sync") else None
    t1 = time.perf_counter()
    for s in range(n):
        info = ld.step(2, s)
    ld.fetch_ids(info)
    wall2 = time.perf_counter() - t1
    print(f"depth {depth}: e2e {n * B / wall / 1e6:.2f} M/s ({wall / n * 1e6:.1f} us/step), "
          f"submit {np.mean(ts) * 1e6:.1f} us, wait {np.mean(tw) * 1e6:.1f} us; "
          f"device-planned {n * B / wall2 / 1e6:.2f} M/s", flush=True)
    ld.close()
