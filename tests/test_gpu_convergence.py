"""GPU parity of the CCM convergence test (edm_ccm_convergence, reading R16)
with the fp64 oracle: every sample rho within 1e-4 with NaN exactly where the oracle has NaN,
the sample means likewise, the full-library case byte-identical to edm_ccm_all_pairs, and the
convergence property on the coupled logistic pair."""
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


def check(data, E, sizes, orders, tau=1, Tp=1, mode="target", excl=True, lb=0, le=None):
    g_mean, g_smp = libccm.ccm_convergence(dev(data), dev(E, torch.int32), sizes, orders, tau, Tp, mode, excl, lb, le,
                                           samples=True)
    o_mean, o_smp = O.ccm_convergence_rows(data, E, sizes, orders, tau, Tp, 0 if mode == "target" else 1, excl, lb,
                                           le, samples=True)
    assert_rho_close(g_smp.cpu().numpy(), o_smp)
    assert_rho_close(g_mean.cpu().numpy(), o_mean)
    return g_mean.cpu().numpy()


@pytest.mark.parametrize("mode", ["target", "library"])
@pytest.mark.parametrize("Tp", [0, 1])
def test_convergence_small(mode, Tp):
    data = synth.random_dataset(12, 200, 31)
    rng = np.random.default_rng(32)
    E = rng.integers(1, 9, 12).astype(np.int32)
    orders = synth.library_orders(3, 200, 33)
    orders[0] = np.arange(200)  # contiguous prefix library
    check(data, E, [5, 12, 30, 80, 200], orders, 1, Tp, mode)


def test_convergence_sparse_sets_all_E():
    # every E = 1..20, sizes at and around the minimum E + 2 (partial prefill lists), tau = 2,
    # sizes unsorted, a size with no defined E at all
    N, L = 40, 300
    data = synth.random_dataset(N, L, 41)
    E = (1 + np.arange(N) % 20).astype(np.int32)
    orders = synth.library_orders(2, L, 42)
    for mode in ("target", "library"):
        check(data, E, [22, 3, 1, 9, 60], orders, 2, 1, mode, True, 3, 29)
    check(data, E, [21, 4], orders, 1, 1, "target", False, 0, 8)


def test_full_library_is_the_phase2_map():
    """A library set covering every row set gives the phase-2 map: identical kNN indices (both
    paths are bit-exact), rho within 1e-6 -- the map's E-sequential kNN (every E in 1..Etop
    selected) forms the fused weights from its certified fp32 sweep distances, the
    convergence test's sweep kernel from the exact fp64 keys; both are within 1e-6 of the
    oracle's weights. With a gap in the E values both use the sweep kernel: byte-identical."""
    data = synth.random_dataset(50, 260, 51)
    E = np.random.default_rng(52).integers(1, 12, 50).astype(np.int32)   # every E in 1..11
    E_gap = np.where(E == 5, 6, E).astype(np.int32)                       # E = 5 never selected
    orders = synth.library_orders(2, 260, 53)
    d = dev(data)
    for Ev, exact in ((E, False), (E_gap, True)):
        Ed = dev(Ev, torch.int32)
        for mode in ("target", "library"):
            m, smp = libccm.ccm_convergence(d, Ed, [260], orders, 1, 1, mode, samples=True)
            full = libccm.ccm_all_pairs(d, Ed, 1, 1, mode).cpu().numpy()
            for r in range(2):
                s = smp.cpu().numpy()[:, 0, r]
                if exact or mode == "library":
                    assert np.array_equal(s.view(np.uint32), full.view(np.uint32))
                else:
                    assert np.array_equal(np.isnan(s), np.isnan(full))
                    assert np.nanmax(np.abs(s - full)) <= 1e-6


def test_convergence_c2_shape_sampled_rows():
    # c2 shape (N = L = 1000, optimal E from phase 1); 6 sampled library rows vs the oracle
    data = synth.make_config("c2")
    d = dev(data)
    optE = libccm.simplex_optimal_E(d, 20).cpu().numpy()
    sizes, orders = [40, 200, 999], synth.library_orders(2, 1000, 61)
    g = libccm.ccm_convergence(d, dev(optE, torch.int32), sizes, orders, 1, 1, "target", True, 0, 300).cpu().numpy()
    pick = [0, 137, 299]
    ref = np.concatenate([O.ccm_convergence_rows(data, optE, sizes, orders, 1, 1, 0, True, p, p + 1) for p in pick])
    assert_rho_close(g[pick], ref)


def test_convergence_property_on_gpu():
    data = synth.sugihara_pair(400, beta_yx=0.1)
    sizes = [10, 25, 50, 100, 200, 398]
    m = libccm.ccm_convergence(dev(data), dev(np.array([2, 2]), torch.int32), sizes,
                               synth.library_orders(8, 400, 7)).cpu().numpy()
    assert np.all(np.diff(m[1, :, 0]) > 0) and m[1, -1, 0] > 0.8


def test_convergence_errors():
    data = synth.random_dataset(4, 50, 1)
    d, Ed = dev(data), dev(np.array([2, 2, 2, 2]), torch.int32)
    bad = np.tile(np.arange(50, dtype=np.int32), (1, 1))
    bad[0, 0] = 1
    with pytest.raises(libccm.EdmError):
        libccm.ccm_convergence(d, Ed, [10], bad)
    with pytest.raises(libccm.EdmError):
        libccm.ccm_convergence(d, dev(np.array([2, 2, 2, 45]), torch.int32), [10], synth.library_orders(1, 50, 0))
