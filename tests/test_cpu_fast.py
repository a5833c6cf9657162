"""The fast host implementation (cpu_baseline/) against the oracle: it is built
to reach the oracle's numbers exactly (same fp64 operation order for every distance, weight,
prediction and Pearson sum; only the work is organised differently: incremental distances over
E, table reuse, seeded selection, 4-target SIMD lookup), so optimal E, rho(E) and the causal map
must be bit-identical, NaNs included."""
import numpy as np
import pytest

from cpu_baseline import cpu
from oracle import oracle as O
from paper_2011_11082_b200 import synth


def same(a, b):
    assert np.array_equal(np.isnan(a), np.isnan(b))
    assert np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])


@pytest.mark.parametrize("seed", range(4))
def test_simplex_identical(seed):
    data = synth.random_dataset(24, [120, 201, 300, 77][seed], seed)
    tau = 1 + seed % 2
    e1, r1 = cpu.simplex_all(data, 12, tau, nthreads=4)
    e2, r2 = O.simplex_all(data, 12, tau)
    np.testing.assert_array_equal(e1, e2)
    same(r1, r2)


@pytest.mark.parametrize("seed", range(4))
def test_ccm_identical(seed):
    rng = np.random.default_rng(90 + seed)
    N, L = 23, [150, 260, 333, 90][seed]
    data = synth.random_dataset(N, L, 40 + seed)
    data[:, 3] = 1.5                                   # a constant series: NaN paths
    data[:, 7] = synth.quantise8(data[:, 7:8])[:, 0]   # exact ties
    E = rng.integers(1, 11, N).astype(np.int32)
    tau = 1 + seed % 2
    for mode in (0, 1):
        for Tp in (0, 1, 2):
            for excl in (True, False):
                a = cpu.ccm_rows(data, E, tau, Tp, mode, excl, 2, 19, nthreads=3)
                b = O.ccm_rows(data, E, tau, Tp, mode, excl, 2, 19)
                same(a, b)


def test_c1_full_map_identical():
    data = synth.make_config("c1")
    E, _ = O.simplex_all(data, 10)
    same(cpu.ccm_rows(data, E), O.ccm_rows(data, E))


def test_errors():
    data = synth.random_dataset(4, 30, 1)
    with pytest.raises(ValueError):
        cpu.ccm_rows(data, np.array([1, 2, 25, 1], np.int32))
    with pytest.raises(ValueError):
        cpu.ccm_rows(data, np.array([1, 2, 20, 1], np.int32))   # too short for E = 20
