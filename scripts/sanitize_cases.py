"""Small invocations of every hot kernel for compute-sanitizer runs
(scripts/sanitize.sh): K1 shard generation, K2+K3 permutation (with forced
Lemire rejections), K4 assignment (balanced, regular, alpha < 1), K5 pack +
K6 crop augment over the P2P and storage paths, K7 resize (variable
geometry), the HBM sample store and the consumer kernels."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_01196_b200 as ll  # noqa: E402
from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "all"
if case in ("permute", "all"):
    ll.permute_epoch(42, 0, 100_003)
    ll.permute_epoch(7, 1, 4_097)
    ll.permutation_prefix(3, 2, 50_000, 1000)
if case in ("assign", "all"):
    ll.plan_epoch(42, 0, 40_000, 4, 4096)
    ll.plan_epoch(42, 1, 40_000, 8, 4096, scheme="regular")
    ll.plan_epoch(9, 0, 30_000, 3, 999, alpha=0.4)
if case in ("augment", "all"):
    for dtype in ("fp32", "bf16"):
        lds = []
        for j in range(2):
            ld = DeviceLoader(LoaderConfig(d=4096, learners=2, rank=j, batch_size=128, seed=42,
                                           data_seed=42, exchange="p2p",
                                           augment=AugmentConfig(out_dtype=dtype)))
            ld.populate()
            lds.append(ld)
        DeviceLoader.link_peers(lds)
        for t in range(3):
            for ld in lds:
                ld.step(1, t)
        for ld in lds:
            ld.close()
    ld = DeviceLoader(LoaderConfig(d=3000, learners=1, rank=0, batch_size=120, alpha=0.25,
                                   seed=42, data_seed=42))
    ld.populate()
    for t in range(2):
        ld.step(1, t)
    ld.close()
if case in ("resize", "all"):
    ld = DeviceLoader(LoaderConfig(d=512, learners=1, rank=0, batch_size=64, seed=42,
                                   data_seed=42, geometry="variable",
                                   augment=AugmentConfig(mode="resize", out_dtype="bf16")))
    ld.populate()
    for t in range(2):
        ld.step(1, t)
    ld.close()
print("sanitize cases done:", case)
