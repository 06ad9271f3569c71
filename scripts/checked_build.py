"""Build the checked variant library variants/liblocload_checked.so
(-DLL_CHECKED: device-side bounds / invariant checks, LL_DCHECK in
csrc/ll_internal.h).  compute-sanitizer is closed on the GPU pool, so the GPU
test suite is run against this build as the out-of-bounds check:

    python scripts/checked_build.py
    LL_LIB=variants/liblocload_checked.so python -m pytest tests -m gpu -x -q
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_01196_b200 import build as b  # noqa: E402

os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
print(b.build(extra=["-DLL_CHECKED"], lib=os.path.join(ROOT, "variants", "liblocload_checked.so")))
