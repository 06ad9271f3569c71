"""Phase breakdown of the permutation kernel at the bench sizes."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1910_01196_b200 as ll
from paper_1910_01196_b200 import _capi
lib = _capi.lib(); ctx = ll.locload.context(0)
out = {}
for d in [10000, 160000, 320000, 640000, 1280000]:
    ll.permute_epoch(42, 0, d)
    best = None
    for e in range(1, 6):
        ll.permute_epoch(42, e, d)
        p = np.zeros(6, np.uint64)
        _capi.check(lib.ll_last_permute_profile(ctx, _capi.ptr(p, C.c_uint64)))
        if best is None or p[5] < best[5]:
            best = p.copy()
    out[d] = {"rounds": int(best[0]), "grid_rounds": int(best[1]), "us_draws": best[2] / 1e3,
              "us_grid": best[3] / 1e3, "us_cta": best[4] / 1e3, "us_total": best[5] / 1e3}
    print(json.dumps({d: out[d]}), flush=True)
