import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1910_01196_b200.loader import AugmentConfig, DeviceLoader, LoaderConfig
for H, W, p in [(250, 250, 1), (250, 250, 2), (256, 256, 1), (240, 320, 1), (224, 224, 1), (232, 224, 1)]:
    d, B, seed = 2000, 96, 42
    lds = []
    for j in range(p):
        ld = DeviceLoader(LoaderConfig(d=d, height=H, width=W, learners=p, rank=j, batch_size=B,
                                       seed=seed, data_seed=seed, exchange="p2p" if p > 1 else "none",
                                       augment=AugmentConfig(out_dtype="fp32")))
        ld.populate(); lds.append(ld)
    if p > 1: DeviceLoader.link_peers(lds)
    order = oracle.permute_epoch(seed, 1, d)
    r = oracle.assign_step(order[0:B], p, d, oracle.MODE_LOCALITY_BALANCED)
    info = lds[0].step(1, 0)
    lst = r["final_ids"][r["final_off"][0]:r["final_off"][1]]
    got = lds[0].fetch(info)
    src = oracle.gen_samples(seed, lst, H * W * 3)
    ok = [bool(np.array_equal(got[k], oracle.augment(src[k].reshape(H, W, 3), int(s), seed, 1))) for k, s in enumerate(lst)]
    # explicit path on the same samples
    print(H, W, p, "loader ok", sum(ok), "/", len(ok), "kept", info.kept, flush=True)
    if not all(ok):
        k = ok.index(False)
        want = oracle.augment(src[k].reshape(H, W, 3), int(lst[k]), seed, 1)
        g = got[k]
        print("  first bad k", k, "max diff", float(np.abs(g - want).max()), "rows equal:", [bool(np.array_equal(g[0, y], want[0, y])) for y in range(0, 224, 16)])
        for e in [0, 2]:
            w2 = oracle.augment(src[k].reshape(H, W, 3), int(lst[k]), seed, e)
            print("  epoch", e, np.array_equal(g, w2))
    for ld in lds: ld.close()
