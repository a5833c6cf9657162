"""Long-series regime (the paper's GPU-speedup experiment runs 1,000 series at
up to 40,000 time steps): parity of the padded-global-series kNN variant (chosen
automatically once a shared-memory copy of the series would cut the resident CTAs per SM, and
forced here at small sizes through CCM_KNN_SERIES=global) and of the full path at L = 40,000
on sampled rows."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2011_11082_b200 import libccm, synth
from tests.test_gpu_parity import assert_rho_close, dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2011_11082_b200 import build
    build.build()
    libccm.load()
    yield
    libccm.release_workspaces()


@pytest.fixture
def global_series():
    os.environ["CCM_KNN_SERIES"] = "global"
    yield
    del os.environ["CCM_KNN_SERIES"]


def test_global_series_variant_parity(global_series):
    data = synth.random_dataset(30, 300, 71)
    d = dev(data)
    for tau in (1, 2):
        optE = libccm.simplex_optimal_E(d, 12, tau).cpu().numpy()
        ref_E, _ = O.simplex_all(data, 12, tau)
        np.testing.assert_array_equal(optE, ref_E)
        for mode in ("target", "library"):
            for Tp in (0, 1):
                g = libccm.ccm_all_pairs(d, dev(optE, torch.int32), tau, Tp, mode).cpu().numpy()
                assert_rho_close(g, O.ccm_rows(data, optE, tau, Tp, 0 if mode == "target" else 1))
    E = np.random.default_rng(72).integers(1, 9, 30).astype(np.int32)
    g = libccm.ccm_lagged(d, dev(E, torch.int32), 1, -2, 3).cpu().numpy()
    assert_rho_close(g, O.ccm_lagged_rows(data, E, 1, -2, 3))


def test_global_series_equals_shared_series():
    data = synth.make_config("c2", N=300)
    d = dev(data)
    E = libccm.simplex_optimal_E(d, 20)
    a = libccm.ccm_all_pairs(d, E).cpu().numpy()
    os.environ["CCM_KNN_SERIES"] = "global"
    try:
        E2 = libccm.simplex_optimal_E(d, 20)
        b = libccm.ccm_all_pairs(d, E2).cpu().numpy()
    finally:
        del os.environ["CCM_KNN_SERIES"]
    assert torch.equal(E, E2)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_L40000_sampled():
    # the paper's longest series: phase 1 on 3 series (E_max 5 keeps the oracle in seconds) and
    # phase 2 rows of 2 libraries against every target, E forced to {2, 3}
    L = 40000
    data = synth.make_config("c5", N=3, L=L)
    d = dev(data)
    optE = libccm.simplex_optimal_E(d, 5).cpu().numpy()
    ref_E, _ = O.simplex_all(data, 5)
    np.testing.assert_array_equal(optE, ref_E)
    E = np.array([2, 3, 2], np.int32)
    g = libccm.ccm_all_pairs(d, dev(E, torch.int32), 1, 1, "target", True, 0, 2).cpu().numpy()
    assert_rho_close(g, O.ccm_rows(data, E, 1, 1, 0, True, 0, 2))
