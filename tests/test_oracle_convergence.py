"""Pins of the CCM convergence-test oracle (reading R16):
a numpy brute force on tiny inputs (library sets built by masking, full lexsort, corrcoef), the
full-library special case (= the plain phase-2 map), the undefined small sizes, and the property
the test exists for -- skill of the causal direction grows with the library size (Sugihara et
al. 2012, the coupled logistic pair of SPEC.md:457)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2011_11082_b200 import synth
from tests.test_oracle_bruteforce import corr, embed, nn_weights


def micro_convergence(data, E, tau, Tp, mode, sizes, perms, excl=True):
    L, N = data.shape
    R = len(perms)
    out = np.full((N, len(sizes), R, N), np.nan)
    for i in range(N):
        x = data[:, i].astype(float)
        for q, l in enumerate(sizes):
            for r, perm in enumerate(perms):
                for j in range(N):
                    e = E[j] if mode == 0 else E[i]
                    P = np.arange((e - 1) * tau, L - Tp)
                    inP = perm[(perm >= P[0]) & (perm <= P[-1])]
                    C = np.sort(inP[:l])  # membership only: the order inside C is irrelevant
                    if len(C) - (1 if excl else 0) < e + 1:
                        continue
                    idx, W = nn_weights(embed(x, e, tau, P), embed(x, e, tau, C), C, e + 1,
                                        excl_times=P if excl else None)
                    y = data[:, j].astype(float)
                    out[i, q, r, j] = corr((W * y[idx + Tp]).sum(axis=1), y[P + Tp])
    return out


@pytest.mark.parametrize("seed", range(3))
def test_convergence_matches_micro(seed):
    rng = np.random.default_rng(300 + seed)
    N, L = 4, int(rng.integers(40, 70))
    data = synth.random_dataset(N, L, seed)
    E = rng.integers(1, 5, N).astype(np.int32)
    tau = 1 + seed % 2
    perms = synth.library_orders(3, L, seed)
    perms[0] = np.arange(L)  # contiguous library prefix
    sizes = [3, 7, 15, L]
    for mode in (0, 1):
        for Tp in (0, 1):
            mean, smp = O.ccm_convergence_rows(data, E, sizes, perms, tau, Tp, mode, samples=True)
            ref = micro_convergence(data, E, tau, Tp, mode, sizes, perms)
            np.testing.assert_allclose(smp, ref, atol=1e-12, rtol=0)
            cnt = np.sum(~np.isnan(ref), axis=2)
            ref_mean = np.where(cnt > 0, np.nansum(ref, axis=2) / np.maximum(cnt, 1), np.nan)
            np.testing.assert_allclose(mean, ref_mean, atol=1e-12, rtol=0)


def test_full_library_equals_phase2_map():
    data = synth.make_config("c1")
    E = np.array([2, 2, 3, 1, 4, 2, 5, 3], np.int32)
    perms = synth.library_orders(2, data.shape[0], 1)
    for mode in (0, 1):
        mean, smp = O.ccm_convergence_rows(data, E, [data.shape[0]], perms, mode=mode, samples=True)
        full = O.ccm_rows(data, E, mode=mode)
        for r in range(2):
            np.testing.assert_array_equal(smp[:, 0, r, :], full)
        np.testing.assert_array_equal(mean[:, 0, :], full)


def test_small_library_is_undefined():
    data = synth.random_dataset(3, 80, 5)
    E = np.array([3, 3, 3], np.int32)
    perms = synth.library_orders(2, 80, 2)
    # exclude_self: a library point has |C| - 1 candidates, so |C| = E + 1 is one short
    mean = O.ccm_convergence_rows(data, E, [E[0] + 1, E[0] + 2], perms)
    assert np.all(np.isnan(mean[:, 0, :]))
    assert np.all(np.isfinite(mean[:, 1, :]))
    mean = O.ccm_convergence_rows(data, E, [E[0] + 1], perms, exclude_self=False)
    assert np.all(np.isfinite(mean))


def test_skill_converges_with_library_size():
    # y is driven by x (beta_yx > 0, beta_xy = 0): x's state is recoverable from y's manifold,
    # so "library y -> target x" is the causal direction and its skill grows with the library;
    # the reverse map has no information to converge to.
    L = 400
    data = synth.sugihara_pair(L, beta_yx=0.1)
    E = np.array([2, 2], np.int32)
    sizes = [10, 25, 50, 100, 200, 398]
    perms = synth.library_orders(8, L, 7)
    mean = O.ccm_convergence_rows(data, E, sizes, perms)
    causal, reverse = mean[1, :, 0], mean[0, :, 1]
    assert np.all(np.diff(causal) > 0), causal
    assert causal[-1] > 0.8 and causal[-1] - causal[0] > 0.5
    assert reverse[-1] - reverse[0] < 0.1 and np.all(np.abs(reverse) < 0.2), reverse


def test_bad_orders_rejected():
    data = synth.random_dataset(2, 40, 1)
    E = np.array([2, 2], np.int32)
    bad = np.arange(40, dtype=np.int32)[None, :].copy()
    bad[0, 5] = 6  # duplicate label
    with pytest.raises(ValueError):
        O.ccm_convergence_rows(data, E, [10], bad)
    with pytest.raises(ValueError):
        O.ccm_convergence_rows(data, E, [0], synth.library_orders(1, 40, 0))


@pytest.mark.parametrize("seed", range(4))
def test_subset_table_matches_bruteforce(seed):
    # oracle_ccm_subset_table (the per-(l, r, E) table of reading R16, exposed for the GPU table
    # readback parity) against the numpy brute force: library set by masking, full lexsort
    rng = np.random.default_rng(700 + seed)
    L = int(rng.integers(50, 90))
    x = synth.random_dataset(4, L, seed)[:, seed % 4].astype(float)  # column 0 is quantised (ties)
    perm = synth.library_orders(1, L, seed)[0]
    tau, Tp = 1 + seed % 2, seed % 3
    for E in (1, 2, 4):
        for l in (E + 3, 20, L):
            for excl in (True, False):
                P = np.arange((E - 1) * tau, L - Tp)
                C = np.sort(perm[(perm >= P[0]) & (perm <= P[-1])][:l])
                idx, d2 = O.ccm_subset_table(x, E, perm, l, tau, Tp, excl)
                ridx, _ = nn_weights(embed(x, E, tau, P), embed(x, E, tau, C), C, E + 1,
                                     excl_times=P if excl else None)
                np.testing.assert_array_equal(idx, ridx)
                # the distances are the plain fp64 sums of C3 (brute force in the same order)
                Q, Cm = embed(x, E, tau, P), embed(x, E, tau, idx.ravel())
                ref = np.zeros(idx.size)
                for m in range(E):
                    diff = np.repeat(Q[:, m], E + 1) - Cm[:, m]
                    ref = ref + diff * diff
                np.testing.assert_array_equal(d2.ravel(), ref)
    with pytest.raises(ValueError):  # |C| - 1 < E + 1
        O.ccm_subset_table(x, 3, perm, 4, 1, 1, True)
