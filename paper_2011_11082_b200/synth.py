"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds NO arithmetic of the method (no embedding, kNN, weights, lookup or
Pearson): it only generates time series. Both sides of every parity test draw their
inputs from here, nothing else is shared.

Every dataset is returned as float32, time-major, shape [L, N] (``data[t, j]``), the
layout of the paper's "L x N array ts" (Alg. 1 input) and of SPEC.md:30.

Generators
----------
* :func:`sugihara_pair`     -- two-species coupled logistic map, the standard CCM test system
  (SPEC.md:457 formula; the system of the paper's cited CCM paper, PAPER.md:134-135
  [sugihara2012detecting]).
* :func:`noise`             -- i.i.d. N(0,1) null series.
* :func:`sine`              -- noiseless sine, 25 points per cycle.
* :func:`coupled_network`   -- a network of coupled chaotic maps observed through a
  calcium-like AR(1) filter: stands in for the whole-brain firing-rate recordings of
  PAPER.md:205-208 / Table ``table:dataset`` (recipe: SURVEY.md 8(d)).
* :func:`quantise8`         -- 8-bit quantised copy (exact in fp32; creates exact
  distance ties that exercise lowest-index tie-breaking).
* :func:`make_config`       -- BASELINE.json configs c1..c5.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2011_11082

# BASELINE.json "configs" (index 0..4 -> c1..c5): (N, L, E_max, tau, Tp)
CONFIGS = {
    "c1": dict(N=8, L=200, E_max=10, tau=1, Tp=1),
    "c2": dict(N=1000, L=1000, E_max=20, tau=1, Tp=1),
    "c3": dict(N=53053, L=1450, E_max=20, tau=1, Tp=1),
    "c4": dict(N=101729, L=1450, E_max=20, tau=1, Tp=1),
    "c5": dict(N=10000, L=10000, E_max=20, tau=1, Tp=1),
}


def sugihara_pair(L: int, rx: float = 3.8, ry: float = 3.5, beta_xy: float = 0.0,
                  beta_yx: float = 0.1, x0: float = 0.4, y0: float = 0.2,
                  burn: int = 300) -> np.ndarray:
    """Coupled logistic map, SPEC.md:457:
    x(t+1) = x(t)(r_x - r_x x(t) - beta_xy y(t)),  y(t+1) = y(t)(r_y - r_y y(t) - beta_yx x(t)).
    x drives y when beta_yx > 0 and beta_xy = 0. r_y = 3.5 (SURVEY.md 2.6 synth row). Returns [L, 2] float32."""
    x, y = float(x0), float(y0)
    out = np.empty((L, 2), dtype=np.float64)
    for t in range(burn + L):
        x, y = x * (rx - rx * x - beta_xy * y), y * (ry - ry * y - beta_yx * x)
        if t >= burn:
            out[t - burn, 0] = x
            out[t - burn, 1] = y
    return out.astype(np.float32)


def noise(N: int, L: int, seed: int) -> np.ndarray:
    """i.i.d. standard normal series, [L, N] float32."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((L, N)).astype(np.float32)


def sine(L: int, period: float = 25.0, phase: float = 0.0) -> np.ndarray:
    """sin(2 pi t / period + phase), [L, 1] float32 (25 points per cycle)."""
    t = np.arange(L, dtype=np.float64)
    return np.sin(2.0 * np.pi * t / period + phase).astype(np.float32)[:, None]


def coupled_network(N: int, L: int, seed: int, burn: int = 300, n_parents: int = 2,
                    noise_frac: float = 0.05, n_const: int = 2) -> np.ndarray:
    """Network of coupled logistic maps seen through a calcium-like filter.

    x_i(t+1) = (1-eps_i) f_i(x_i(t)) + eps_i * mean_{p in P_i} f_p(x_p(t)),  f_i(x) = r_i x (1-x),
    r_i ~ U(3.7, 3.95), eps_i ~ U(0, 0.3), |P_i| = n_parents random parents.
    Observation c_i(t) = alpha_i c_i(t-1) + x_i(t), alpha_i ~ U(0, 0.8), plus N(0, (s_i sd_i)^2)
    noise with s_i ~ U(0.01, 0.05). A fraction noise_frac of the series are replaced by pure
    N(0,1) noise and n_const series are constant (the undefined-rho / NaN path).
    Returns [L, N] float32, time-major.
    """
    rng = np.random.default_rng(seed)
    r = rng.uniform(3.7, 3.95, N)
    eps = rng.uniform(0.0, 0.3, N)
    parents = rng.integers(0, N, size=(N, n_parents))
    alpha = rng.uniform(0.0, 0.8, N)
    x = rng.uniform(0.05, 0.95, N)
    c = np.zeros(N)
    out = np.empty((L, N), dtype=np.float64)
    for t in range(burn + L):
        f = r * x * (1.0 - x)
        x = (1.0 - eps) * f + eps * f[parents].mean(axis=1)
        c = alpha * c + x
        if t >= burn:
            out[t - burn] = c
    sd = out.std(axis=0)
    s = rng.uniform(0.01, 0.05, N)
    out += rng.standard_normal((L, N)) * (s * sd)[None, :]
    n_noise = int(round(noise_frac * N))
    if n_noise > 0 and N > n_const + 1:
        cols = rng.choice(N, size=n_noise, replace=False)
        out[:, cols] = rng.standard_normal((L, n_noise))
    if n_const > 0 and N > n_const + 1:
        cols = rng.choice(N, size=n_const, replace=False)
        out[:, cols] = rng.uniform(-1.0, 1.0, n_const)[None, :]
    return out.astype(np.float32)


def quantise8(data: np.ndarray) -> np.ndarray:
    """Per-series 8-bit quantisation onto 256 levels (integers 0..255 stored as float32:
    exact in fp32 and fp64, so many embedded distances tie exactly)."""
    d = data.astype(np.float64)
    lo = d.min(axis=0, keepdims=True)
    hi = d.max(axis=0, keepdims=True)
    span = np.where(hi > lo, hi - lo, 1.0)
    q = np.floor((d - lo) / span * 255.0 + 0.5)
    return q.astype(np.float32)


def make_config(name: str, N: int | None = None, L: int | None = None) -> np.ndarray:
    """Dataset for BASELINE.json config ``name`` (c1..c5), optionally with N/L overridden
    (smaller parity cases of the same recipe). Seed = 2011_11082 + config number."""
    cfg = CONFIGS[name]
    N = cfg["N"] if N is None else N
    L = cfg["L"] if L is None else L
    seed = SEED_BASE + int(name[1:])
    if name == "c1":
        pair = sugihara_pair(L)
        rest = noise(max(N - 2, 0), L, seed)
        return np.ascontiguousarray(np.concatenate([pair, rest], axis=1)[:, :N])
    return coupled_network(N, L, seed)


def random_dataset(N: int, L: int, seed: int) -> np.ndarray:
    """Small random datasets for equivalence/parity tests: a mix of coupled-network,
    noise and (every 4th column) a quantised column."""
    d = coupled_network(N, L, seed, n_const=0, noise_frac=0.2)
    q = quantise8(d)
    d[:, ::4] = q[:, ::4]
    return np.ascontiguousarray(d)


def library_orders(R: int, L: int, seed: int) -> np.ndarray:
    """R seeded random orders of the time labels 0..L-1, int32 [R, L]: the random draws of the
    CCM convergence test (R16). Sample r's library set of size l is the first l labels
    of row r inside the row set P_E."""
    rng = np.random.default_rng(seed)
    return np.stack([rng.permutation(L) for _ in range(R)]).astype(np.int32)
