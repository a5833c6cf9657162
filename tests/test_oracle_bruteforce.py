"""Brute-force micro-oracle (numpy, full distance matrices + full stable sort) on tiny
inputs, pinning the C oracle's indexing: the library/target split, the
one-step-ahead alignment of phase 1, the phase-2 row set P_E and horizon Tp
 and the target/library E conventions (P:434 / north_star).

The micro-oracle is structured differently from ccm_oracle.c on purpose: embeddings are
materialised as matrices, neighbours come from np.lexsort over the whole row, and Pearson
comes from numpy.corrcoef, so a dropped term, a wrong sign/lag/offset or a transposed
operand in the C code would show up here.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2011_11082_b200 import synth


def embed(x, E, tau, times):
    """Rows = delay vectors (x[t], x[t-tau], ..., x[t-(E-1)tau]) for the given times."""
    return np.stack([x[times - m * tau] for m in range(E)], axis=1)


def nn_weights(Q, C, cand_times, k, excl_times=None):
    D = np.zeros((len(Q), len(C)))
    for m in range(Q.shape[1]):
        diff = Q[:, m][:, None] - C[:, m][None, :]
        D = D + diff * diff
    idx = np.zeros((len(Q), k), int)
    W = np.zeros((len(Q), k))
    for r in range(len(Q)):
        keep = np.ones(len(C), bool) if excl_times is None else cand_times != excl_times[r]
        ct, dr = cand_times[keep], D[r, keep]
        order = np.lexsort((ct, dr))[:k]
        idx[r] = ct[order]
        d = np.sqrt(dr[order])
        if d[0] > 0:
            u = np.exp(-d / d[0])
        else:
            u = (d == 0).astype(float)
        u = np.maximum(u, 1e-6)
        W[r] = u / u.sum()
    return idx, W


def corr(a, b):
    if np.all(a == a[0]) or np.all(b == b[0]):
        return np.nan
    return np.corrcoef(a, b)[0, 1]


def micro_simplex_rho(x, E, tau):
    L = len(x)
    Llib = -(-L // 2)
    lib, tgt = x[:Llib], x[Llib:]
    q = np.arange((E - 1) * tau, len(tgt) - 1)
    c = np.arange((E - 1) * tau, Llib - 1)
    if len(c) < E + 1 or len(q) < 2:
        return np.nan
    idx, W = nn_weights(embed(tgt, E, tau, q), embed(lib, E, tau, c), c, E + 1)
    yhat = (W * lib[idx + 1]).sum(axis=1)
    return corr(yhat, tgt[q + 1])


def micro_ccm(data, E, tau, Tp, mode):
    L, N = data.shape
    R = np.zeros((N, N))
    for i in range(N):
        x = data[:, i].astype(float)
        for j in range(N):
            e = E[j] if mode == 0 else E[i]
            P = np.arange((e - 1) * tau, L - Tp)
            idx, W = nn_weights(embed(x, e, tau, P), embed(x, e, tau, P), P, e + 1, excl_times=P)
            y = data[:, j].astype(float)
            R[i, j] = corr((W * y[idx + Tp]).sum(axis=1), y[P + Tp])
    return R


@pytest.mark.parametrize("seed", range(6))
def test_simplex_matches_micro(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(24, 120))
    x = synth.coupled_network(2, L, seed)[:, 0].astype(float) if seed % 2 else rng.standard_normal(L)
    tau = 1 + seed % 2
    for E in range(1, 7):
        a = O.simplex_rho_E(x, E, tau)
        b = micro_simplex_rho(x, E, tau)
        assert (np.isnan(a) and np.isnan(b)) or a == pytest.approx(b, abs=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_ccm_matches_micro(seed):
    rng = np.random.default_rng(50 + seed)
    N, L = 5, int(rng.integers(30, 70))
    data = synth.random_dataset(N, L, seed)
    E = rng.integers(1, 5, N).astype(np.int32)
    tau = 1 + seed % 2
    for mode in (0, 1):
        for Tp in (0, 1, 2):
            a = O.ccm_rows(data, E, tau, Tp, mode, True)
            b = micro_ccm(data, E, tau, Tp, mode)
            np.testing.assert_allclose(a, b, atol=1e-12, rtol=0)


def test_simplex_all_matches_per_series():
    data = synth.random_dataset(6, 100, 8)
    optE, rhoE = O.simplex_all(data, 7)
    for j in range(6):
        e, r, _ = O.simplex(data[:, j].astype(float), 7)
        assert e == optE[j]
        np.testing.assert_array_equal(r, rhoE[j])
        ref = [micro_simplex_rho(data[:, j].astype(float), E, 1) for E in range(1, 8)]
        np.testing.assert_allclose(r, ref, atol=1e-12)
