"""Bit-exact parity of the hot path's phase-2 kNN tables (Alg. 2 line 5 "kNN(ts[i], ts[i], E)",
PAPER.md:430; partialSort selection) read back through edm_ccm_tables, which
runs the same table build as edm_ccm_all_pairs / edm_ccm_lagged / edm_ccm_convergence (same
kernels, specialisations, library blocks and launch configuration) and copies the tables out
instead of running the lookup.

Bars (BASELINE.json north_star): idx bit-exact (lowest index on exact ties), dist equal to
fp32(sqrt(oracle fp64 d2)) exactly, weights within 1e-6. Covered: the c3 bench configuration
(53,053 x 1,450, all 20 E selected, 256-library blocks), the padded-global-series variant, the
convergence-test library sets, library mode, lagged tables, quantised ties and tau = 2; plus
the input domain of reading R17 (rescaled extreme magnitudes, non-finite input rejected).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2011_11082_b200 import libccm, synth
from tests.test_gpu_parity import assert_rho_close, dev

pytestmark = pytest.mark.gpu
W_TOL = 1e-6


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2011_11082_b200 import build
    build.build()
    libccm.load()
    yield
    libccm.release_workspaces()


def _pool():
    return ThreadPoolExecutor(max_workers=os.cpu_count() or 4)  # ctypes releases the GIL


def check_tables(data, E, Eq, libs, tau=1, lag_min=1, lag_max=None, mode="target", excl=True, lib_begin=0,
                 lib_end=None, order=None, lib_size=0, d=None):
    """Read back the tables at Eq of rows [lib_begin, lib_end) and compare the sampled library
    rows `libs` with the oracle's table of that library series."""
    lag_max = lag_min if lag_max is None else lag_max
    L, N = data.shape
    lib_end = N if lib_end is None else lib_end
    d = dev(data) if d is None else d
    idx, dist, w = libccm.ccm_tables(d, dev(E, torch.int32), Eq, tau, lag_min, lag_max, mode, excl, lib_begin, lib_end,
                                     lib_size, order)
    idx, dist, w = idx.cpu().numpy(), dist.cpu().numpy(), w.cpu().numpy()
    m_lo, m_hi = max(0, -lag_min), max(0, lag_max)
    lo, hi = (Eq - 1) * tau + m_lo, L - 1 - m_hi

    def ref(i):
        x = data[:, i].astype(np.float64)
        if order is not None:
            return O.ccm_subset_table(x, Eq, order, lib_size, tau, lag_min, excl)
        return O.knn(x, lo, hi, x, lo, hi, Eq, tau, excl)

    checked = 0
    with _pool() as ex:
        refs = list(ex.map(ref, libs))
    for i, (ri, rd2) in zip(libs, refs):
        r = i - lib_begin
        if mode == "library" and E[i] != Eq:
            assert np.all(idx[r] == -1)  # not built at Eq: untouched
            continue
        np.testing.assert_array_equal(idx[r], ri, err_msg=f"library {i} E={Eq}")
        np.testing.assert_array_equal(dist[r], np.sqrt(rd2).astype(np.float32), err_msg=f"library {i} E={Eq}")
        rw = np.stack([O.weights(row) for row in rd2])
        np.testing.assert_allclose(w[r], rw, atol=W_TOL, rtol=0, err_msg=f"library {i} E={Eq}")
        checked += 1
    return checked


def test_tables_c3_bench_configuration():
    """c3 at full size in the bench's launch configuration: a whole 256-library block, every E
    1..20 selected (FULLMASK, shared-memory series); sampled libraries of the block at every E."""
    data = synth.make_config("c3")
    L, N = data.shape
    d = dev(data)
    E = (1 + np.arange(N) % 20).astype(np.int32)  # every E in S, as in the bench's optE mix
    rng = np.random.default_rng(17)
    for r0 in (0, 26_368, N - 256):
        libs = np.sort(rng.choice(np.arange(r0, r0 + 256), 3, replace=False))
        for Eq in range(1, 21):
            assert check_tables(data, E, Eq, libs, lib_begin=r0, lib_end=r0 + 256, d=d) == 3


@pytest.mark.parametrize("case", range(4))
def test_tables_small_variants(case):
    """Ragged N, quantised (exact ties), tau = 2, Tp in {0, 1, 2}, exclusion on/off."""
    rng = np.random.default_rng(40 + case)
    N, L = [45, 70, 33, 90][case], [300, 257, 400, 180][case]
    data = synth.random_dataset(N, L, case)
    if case == 1:
        data = synth.quantise8(data)
    tau, Tp, excl = 1 + case % 2, case % 3, case != 3
    E = rng.integers(1, 9, N).astype(np.int32)
    libs = np.arange(N)
    for Eq in np.unique(E):
        check_tables(data, E, int(Eq), libs, tau, Tp, excl=excl)


def test_tables_global_series_variant():
    """The padded-global-series kNN (long series) forced at c2 size: identical tables."""
    data = synth.make_config("c2", N=300)
    E = (1 + np.arange(300) % 20).astype(np.int32)
    os.environ["CCM_KNN_SERIES"] = "global"
    try:
        for Eq in (1, 2, 3, 7, 20):
            check_tables(data, E, Eq, np.arange(0, 300, 23))
    finally:
        del os.environ["CCM_KNN_SERIES"]


def test_tables_library_mode():
    data = synth.make_config("c2", N=260, L=600)
    E = np.random.default_rng(3).integers(1, 21, 260).astype(np.int32)
    libs = np.arange(0, 260, 7)
    for Eq in (1, 2, 3, 11, 20):
        check_tables(data, E, Eq, libs, mode="library")


def test_tables_lagged():
    data = synth.random_dataset(40, 220, 9)
    E = np.random.default_rng(9).integers(1, 7, 40).astype(np.int32)
    for lags in ((-3, 2), (-1, 0), (0, 3)):
        for Eq in np.unique(E):
            check_tables(data, E, int(Eq), np.arange(0, 40, 3), 1, lags[0], lags[1])


def test_tables_convergence_library_sets():
    data = synth.make_config("c2", N=64, L=500)
    E = (1 + np.arange(64) % 12).astype(np.int32)
    orders = synth.library_orders(2, 500, 5)
    for r, size in ((0, 30), (1, 120), (0, 499)):
        for Eq in (1, 3, 8, 12):
            if size - 1 < Eq + 1:
                continue
            check_tables(data, E, Eq, np.arange(0, 64, 5), order=orders[r], lib_size=size)


def test_tables_target_mode_requires_built_E():
    data = synth.make_config("c2", N=20, L=200)
    E = np.full(20, 3, np.int32)
    with pytest.raises(libccm.EdmError) as e:
        libccm.ccm_tables(dev(data), dev(E, torch.int32), 4)
    assert e.value.status == libccm.EDM_EINVAL


# ---------------------------------------------------------------- input domain (reading R17)
@pytest.mark.parametrize("scale", [2.0 ** 70, 2.0 ** -70, 1e25, 2.0 ** -120])
def test_extreme_magnitudes_exact(scale):
    """Series scaled by an exact power of two (or 1e25, inexactly) keep bit-exact kNN indices
    and distances (the sweep rescales them into its safe range), optE and rho."""
    base = synth.random_dataset(24, 200, 33)
    data = (base.astype(np.float64) * scale).astype(np.float32)
    assert np.all(np.isfinite(data))
    d = dev(data)
    E = np.random.default_rng(4).integers(1, 6, 24).astype(np.int32)
    for Eq in np.unique(E):
        check_tables(data, E, int(Eq), np.arange(24), d=d)
    idx, dist, w = libccm.embed_knn(d[:, 5].contiguous(), 3, 1, 1, True)
    ri, rd2, rw = O.ccm_table(data[:, 5].astype(np.float64), 3, 1, 1, True)
    np.testing.assert_array_equal(idx.cpu().numpy(), ri)
    np.testing.assert_array_equal(dist.cpu().numpy(), np.sqrt(rd2).astype(np.float32))
    optE, rhoE = libccm.simplex_optimal_E(d, 8, return_rho=True)
    rE, rrho = O.simplex_all(data, 8)
    np.testing.assert_array_equal(optE.cpu().numpy(), rE)
    g = libccm.ccm_all_pairs(d, dev(E, torch.int32)).cpu().numpy()
    assert_rho_close(g, O.ccm_rows(data, E))


def test_mixed_magnitudes_in_one_dataset():
    base = synth.random_dataset(16, 160, 34)
    scales = 2.0 ** np.array([0, 80, -80, 40, -30, 100, -100, 10] * 2)
    data = (base.astype(np.float64) * scales[None, :]).astype(np.float32)
    d = dev(data)
    E = np.full(16, 3, np.int32)
    check_tables(data, E, 3, np.arange(16), d=d)
    assert_rho_close(libccm.ccm_all_pairs(d, dev(E, torch.int32)).cpu().numpy(), O.ccm_rows(data, E))


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_input_rejected(bad):
    data = synth.random_dataset(10, 120, 35)
    data[57, 4] = bad
    d = dev(data)
    E = dev(np.full(10, 2, np.int32), torch.int32)
    for call in (lambda: libccm.simplex_optimal_E(d, 5),
                 lambda: libccm.ccm_all_pairs(d, E),
                 lambda: libccm.ccm_lagged(d, E, 1, -1, 1),
                 lambda: libccm.ccm_tables(d, E, 2),
                 lambda: libccm.embed_knn(d[:, 4].contiguous(), 2)):
        with pytest.raises(libccm.EdmError) as e:
            call()
        assert e.value.status == libccm.EDM_EINVAL, e.value
    # the other series alone are fine
    ok = np.delete(data, 4, axis=1)
    libccm.simplex_optimal_E(dev(ok), 5)


def test_unrescalable_series_unsupported():
    data = synth.random_dataset(4, 100, 36)
    data[:, 2] = 1.0
    data[10, 2] = 2.0 ** 100    # max |x| >= 2^60 -> rescaled down by 2^-41 ...
    data[11, 2] = 1.2345e-30     # ... which this value cannot follow exactly (subnormal)
    with pytest.raises(libccm.EdmError) as e:
        libccm.simplex_optimal_E(dev(data), 4)
    assert e.value.status == libccm.EDM_EUNSUPPORTED


def test_eseq_and_sweep_kernels_build_identical_tables():
    """The E-sequential kNN (default when every E in 1..Etop is selected) and the round-1 sweep
    kernel (CCM_KNN_ALGO=sweep) are two schedules of the same selection: identical labels and
    distances, weights within 1e-6, on c2 with every E = 1..20 and on quantised data (ties)."""
    for data in (synth.make_config("c2", N=300), synth.quantise8(synth.make_config("c2", N=120, L=500))):
        N = data.shape[1]
        d = dev(data)
        E = dev((1 + np.arange(N) % 20).astype(np.int32), torch.int32)
        for Eq in (1, 2, 3, 9, 20):
            a = libccm.ccm_tables(d, E, Eq)
            os.environ["CCM_KNN_ALGO"] = "sweep"
            try:
                b = libccm.ccm_tables(d, E, Eq)
            finally:
                del os.environ["CCM_KNN_ALGO"]
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), Eq
            assert float((a[2] - b[2]).abs().max()) <= 1e-6
        sa = libccm.simplex_optimal_E(d, 20, return_rho=True)
        os.environ["CCM_KNN_ALGO"] = "sweep"
        try:
            sb = libccm.simplex_optimal_E(d, 20, return_rho=True)
        finally:
            del os.environ["CCM_KNN_ALGO"]
        assert torch.equal(sa[0], sb[0]) and torch.equal(sa[1].view(torch.int32), sb[1].view(torch.int32))


def test_tables_long_series_kernel():
    """Series longer than the register chunks (1,536 < candidates <= 16,384: knn_long_kernel,
    super-chunks of 1,536 with exact per-E lists): tables bit-exact against the oracle, identical
    to the sweep kernel's, and phase 1 equal to the oracle's; L = 3,000 (two super-chunks) and an
    odd length with a ragged last super-chunk."""
    for L, N in ((3000, 24), (4711, 12)):
        data = synth.make_config("c5", N=N, L=L)
        d = dev(data)
        E = (1 + np.arange(N) % 20).astype(np.int32)
        for Eq in (1, 2, 5, min(20, N)):
            check_tables(data, E, Eq, np.arange(0, N, 5), d=d)
            a = libccm.ccm_tables(d, dev(E, torch.int32), Eq)
            os.environ["CCM_KNN_ALGO"] = "sweep"
            try:
                b = libccm.ccm_tables(d, dev(E, torch.int32), Eq)
            finally:
                del os.environ["CCM_KNN_ALGO"]
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), (L, Eq)
        optE, rhoE = libccm.simplex_optimal_E(d, 20, 1, 0, 4, return_rho=True)
        rE, rrho = O.simplex_all(data, 20, 1, 0, 4)
        np.testing.assert_array_equal(optE.cpu().numpy(), rE)
