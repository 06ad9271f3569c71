"""B200-native locality-aware data loader (arXiv 1910.01196 hot path).

The product is liblocload_b200.so (CUDA sm_100a kernels + C-ABI, see
include/locload_b200.h); this package holds its ctypes binding and a Python
mirror of the reference's locload API.  Importing this package does not need
a GPU; calling any compute entry point without one raises LoaderError.
"""
from . import _capi  # noqa: F401
from .locload import (CacheDirectory, EpochPermutation, GlobalBatch, ImbalanceVector,  # noqa: F401
                      LocalAssignment, LocDistribution, Move, TransferSchedule, assign,
                      assign_batch, balance, balance_many, batches, counts_with_uncached,
                      EpochPlan, deficit_fraction, loc_distribution, permutation_prefix,
                      permute_epoch, plan_epoch,
                      reg_slice, targets)
from .loader import AugmentConfig, DeviceLoader, LoaderConfig, ThroughputReport  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
