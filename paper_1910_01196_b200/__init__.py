"""B200-native locality-aware data loader (arXiv 1910.01196 hot path).

The product is liblocload_b200.so (CUDA sm_100a kernels + C-ABI, see
include/locload_b200.h); this package holds its ctypes binding and a Python
mirror of the reference's locload API.  Importing this package does not need
a GPU; calling any compute entry point without one raises LoaderError.
"""
import os as _os

# NCCL exchange: 128 KB NVLink P2P chunks. With the registered exchange buffers
# (loader_comm_init) the grouped send/recv shares HBM and SMs with the augment,
# and small chunks keep it moving: cfg4 over NCCL at N = 2 8.56 -> 10.17 M
# samples/s (fp32), 9.97 -> 12.23 M (bf16); cfg2 / cfg5 unchanged
# (profiles/r2_nccl_exchange.md).  Set before any NCCL communicator exists
# (NCCL reads its parameters once per process); a user's own value wins.
_os.environ.setdefault("NCCL_P2P_NVL_CHUNKSIZE", "131072")

from . import _capi  # noqa: F401
from .locload import (CacheDirectory, EpochPermutation, GlobalBatch, ImbalanceVector,  # noqa: F401
                      LocalAssignment, LocDistribution, Move, TransferSchedule, assign,
                      assign_batch, balance, balance_many, batches, counts_with_uncached,
                      EpochPlan, deficit_fraction, loc_distribution, permutation_prefix,
                      permute_epoch, plan_epoch,
                      reg_slice, targets)
from .loader import AugmentConfig, DeviceLoader, LoaderConfig, ThroughputReport  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
