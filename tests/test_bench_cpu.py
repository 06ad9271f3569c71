"""bench.py host logic on CPU: the Eq. 8 comparator fixture, the cfg5 window
accounting, the workload labels.  (The GPU arm itself runs on the B200.)"""
import importlib.util
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_eq8_betas_come_from_the_reference_fixture(golden):
    b = _bench()
    betas = b.eq8_betas()
    assert sorted(betas) == [2, 4, 8]
    for c in golden["simulate_imbalance"]:
        assert betas[c["p"]] == c["beta_median"]
    # Eq. 8 at p = 8: alpha * D * beta with D = 156 * 8192 samples per epoch
    assert round(156 * 8192 * betas[8]) == 14820


def test_eq8_beta_fixture_equals_a_live_reference_run(ref_lib):
    """The committed beta equals simulate_imbalance run now through oracle/_ref
    (the way `locload imbalance` seeds it)."""
    import oracle
    b = _bench()
    for p, beta in b.eq8_betas().items():
        assert oracle.eq8_beta_median(b.HEADLINE_D, p, 1024, 42) == beta


def test_cfg5_window_accounting():
    b = _bench()
    # E[3 min(H, W)^2] for H, W uniform on [128, 512]
    v = np.arange(128, 513)
    want = 3.0 * np.mean(np.minimum(v[:, None], v[None, :]) ** 2)
    assert abs(b.mean_window_bytes_cfg5() - want) < 1e-6
    assert 220_000 < want < 222_000


def test_workload_labels():
    b = _bench()

    class A:
        workload, per_gpu_d, per_gpu_batch, dtype, exchange = "cfg2", 160000, 1024, "fp32", "p2p"
    w = b.workload(A, 8)
    assert w["d"] == 1_280_000 and w["global_batch"] == 8192 and w["learners"] == 8
    assert "cfg2" in w["workload"]
