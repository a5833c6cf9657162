"""Pins of the oracle's time-delay cross mapping ("The adjacency in the
network is determined by time delay cross mapping"): consistency with the single-horizon map
(a pinned function), a numpy brute-force micro-oracle, and the causal-lag signature of Ye et
al. 2015 (cited by the paper as [ye2015distinguishing]): when x drives y with a delay d, the
skill of cross-mapping x from y's manifold peaks at lag -(d+1) (y(t+1) carries x(t-d))."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2011_11082_b200 import synth
from tests.test_oracle_bruteforce import corr, embed, nn_weights


def micro_lagged(data, E, tau, lmin, lmax, mode):
    L, N = data.shape
    mlo, mhi = max(0, -lmin), max(0, lmax)
    R = np.zeros((N, lmax - lmin + 1, N))
    for i in range(N):
        x = data[:, i].astype(float)
        for j in range(N):
            e = E[j] if mode == 0 else E[i]
            P = np.arange((e - 1) * tau + mlo, L - mhi)
            idx, W = nn_weights(embed(x, e, tau, P), embed(x, e, tau, P), P, e + 1, excl_times=P)
            y = data[:, j].astype(float)
            for a, l in enumerate(range(lmin, lmax + 1)):
                R[i, a, j] = corr((W * y[idx + l]).sum(axis=1), y[P + l])
    return R


def test_single_lag_equals_single_horizon_map():
    data = synth.random_dataset(10, 90, 4)
    E, _ = O.simplex_all(data, 5)
    for Tp in (0, 1, 2):
        for mode in (0, 1):
            a = O.ccm_lagged_rows(data, E, 1, Tp, Tp, mode)[:, 0, :]
            b = O.ccm_rows(data, E, 1, Tp, mode)
            assert np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("seed", range(3))
def test_lagged_matches_micro(seed):
    rng = np.random.default_rng(seed)
    data = synth.random_dataset(4, 60, 30 + seed)
    E = rng.integers(1, 4, 4).astype(np.int32)
    lmin, lmax = [(-3, 2), (-1, 0), (0, 3)][seed]
    for mode in (0, 1):
        a = O.ccm_lagged_rows(data, E, 1 + seed % 2, lmin, lmax, mode)
        b = micro_lagged(data, E, 1 + seed % 2, lmin, lmax, mode)
        np.testing.assert_allclose(a, b, atol=1e-12, rtol=0)


def delayed_pair(L, delay, burn=300):
    """x drives y with a delay: y(t+1) = y(t)(3.5 - 3.5 y(t) - 0.1 x(t - delay))."""
    x, y = 0.4, 0.2
    hist = [x] * (delay + 1)
    out = []
    for t in range(burn + L):
        xd = hist[-1 - delay]
        x, y = x * (3.8 - 3.8 * x), y * (3.5 - 3.5 * y - 0.1 * xd)
        hist.append(x)
        if t >= burn:
            out.append((x, y))
    return np.array(out, np.float32)


@pytest.mark.parametrize("delay", [0, 3])
def test_causal_lag_signature(delay):
    data = delayed_pair(1000, delay)
    lmin, lmax = -6, 3
    R = O.ccm_lagged_rows(data, np.array([2, 2]), 1, lmin, lmax)
    y_to_x = R[1, :, 0]
    assert lmin + int(np.argmax(y_to_x)) == -(delay + 1)
    assert y_to_x.max() > 0.95
    assert np.abs(R[0, :, 1]).max() < 0.2  # x's manifold does not encode y at any lag
