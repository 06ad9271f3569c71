"""Consumer side (equivalence.hpp): synchronous SGD on the
device fed by the loader's epoch plan, against the compiled reference's own
run_training / full_batch_gradient (oracle/_ref, equivalence.cpp:95-205).

Bar: bit-exact fp64 (final weights and every step gradient), for all three
schemes under both aggregations; Theorem 1 (canonical aggregation makes the
schemes identical) then holds on the GPU by construction and is asserted too.
"""
import numpy as np
import pytest

import oracle
from paper_1910_01196_b200 import locload as ll
from paper_1910_01196_b200._capi import InvalidArgument

pytestmark = pytest.mark.gpu

CASES = [  # n, dims, obj_seed, p, B, steps, seed, lr
    (120, 8, 5, 3, 12, 50, 6, 0.01),     # test_equivalence.cpp:64-76 shape
    (64, 8, 9, 2, 2, 30, 1, 0.02),       # two-sample batches
    (512, 8, 21, 4, 64, 100, 2, 0.01),   # several epochs
    (1000, 17, 3, 5, 60, 40, 11, 0.005),  # B does not divide n (remainder dropped)
    (4096, 32, 7, 8, 512, 25, 4, 0.001),  # wider, many learners
    (50, 3, 1, 1, 50, 10, 0, 0.1),       # one learner, full batch
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("agg", ["canonical", "learner_order"])
def test_run_training_bit_exact_vs_reference(case, agg):
    n, dims, os_, p, B, steps, seed, lr = case
    obj = ll.ToyObjective.synthesize(n, dims, os_)
    runs = {}
    for scheme in ["regular", "locality", "locality_balanced"]:
        if scheme == "regular" and B % p:
            continue
        got = ll.run_training(obj, scheme, p, B, steps, seed, lr, agg)
        w, g = oracle.ref_run_training(n, dims, os_, scheme, p, B, steps, seed, lr, agg)
        assert np.array_equal(got.final_weights, w), (scheme, np.abs(got.final_weights - w).max())
        assert np.array_equal(got.step_gradients, g), scheme
        runs[scheme] = got
    if agg == "canonical":  # Theorem 1, bit for bit
        ref_w = runs["locality"].final_weights
        for r in runs.values():
            assert np.array_equal(r.final_weights, ref_w)


def test_imbalanced_vs_balanced_pair():
    obj = ll.ToyObjective.synthesize(512, 8, 21)
    loc, bal = ll.run_training_imbalanced_vs_balanced(obj, 4, 64, 100, 2, 0.01)
    assert np.array_equal(loc.final_weights, bal.final_weights)
    assert np.array_equal(loc.step_gradients, bal.step_gradients)


def test_full_batch_gradient_vs_reference():
    n, dims, os_ = 640, 8, 13
    obj = ll.ToyObjective.synthesize(n, dims, os_)
    rng = np.random.default_rng(3)
    for b in [1, 7, 64, 640]:
        batch = ll.GlobalBatch(step=0, samples=rng.permutation(n)[:b].astype(np.uint64))
        w = rng.standard_normal(dims)
        got = ll.full_batch_gradient(obj, w, batch)
        assert np.array_equal(got, oracle.ref_full_batch_gradient(n, dims, os_, w, batch.samples))


def test_errors_match_reference():
    obj = ll.ToyObjective.synthesize(120, 8, 5)
    with pytest.raises(InvalidArgument, match="need at least one learner"):
        ll.run_training(obj, "regular", 0, 12, 10, 6, 0.01)
    with pytest.raises(InvalidArgument, match=r"batch size must be in \[1, n\]"):
        ll.run_training(obj, "locality", 3, 0, 10, 6, 0.01)
    with pytest.raises(InvalidArgument, match=r"batch size must be in \[1, n\]"):
        ll.run_training(obj, "locality", 3, 121, 10, 6, 0.01)
    with pytest.raises(InvalidArgument, match="learner count must divide the batch size"):
        ll.run_training(obj, "regular", 5, 12, 10, 6, 0.01)
    with pytest.raises(ValueError):
        oracle.ref_run_training(120, 8, 5, "regular", 5, 12, 10, 6, 0.01)


@pytest.mark.parametrize("agg", ["canonical", "learner_order", "allreduce"])
@pytest.mark.parametrize("scheme", ["regular", "locality", "locality_balanced"])
def test_distributed_trainer_device_ops_bit_exact(scheme, agg):
    """train_dist.DistributedTrainer on one process (all learners local): lists
    from ll_plan_epoch, per-sample gradients (ll_toy_grads_device), ordered
    sums (ll_ordered_sum_device) and the update (ll_sgd_apply_device) on the
    GPU.  With one process the all-reduce is the learner-order sum, so every
    aggregation must equal the reference bit for bit."""
    from paper_1910_01196_b200.train_dist import DistributedTrainer
    n, dims, os_, p, B, steps, seed, lr = 512, 8, 21, 4, 64, 20, 2, 0.01
    obj = ll.ToyObjective.synthesize(n, dims, os_)
    run = DistributedTrainer(obj, scheme, p, B, seed, lr, aggregation=agg).run(steps)
    ref_agg = "canonical" if agg == "canonical" else "learner_order"
    w, g = oracle.ref_run_training(n, dims, os_, scheme, p, B, steps, seed, lr, ref_agg)
    assert np.array_equal(run.final_weights, w), (scheme, agg)
    assert np.array_equal(run.step_gradients, g), (scheme, agg)
