"""Parity of the CUDA path (through the C ABI) with the fp64 oracle, element by element.

Bars (BASELINE.json north_star):
  * kNN indices and optimal E: bit-exact (the kNN distances are fp64 with the oracle's
    operation order, so there is no tie exception);
  * kNN distances: fp32(sqrt(oracle d2)) exactly; weights within 1e-6;
  * rho: within 1e-4 absolute, NaN exactly where the oracle has NaN.
Inputs are the seeded generators of paper_2011_11082_b200.synth only.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2011_11082_b200 import libccm, synth

pytestmark = pytest.mark.gpu
RHO_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2011_11082_b200 import build
    build.build()
    libccm.load()
    yield
    libccm.release_workspaces()


def dev(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def assert_rho_close(gpu, ref, tol=RHO_TOL):
    gpu = np.asarray(gpu, np.float64)
    nan_g, nan_r = np.isnan(gpu), np.isnan(ref)
    assert np.array_equal(nan_g, nan_r), f"NaN mismatch at {np.argwhere(nan_g != nan_r)[:5]}"
    err = np.abs(gpu[~nan_g] - ref[~nan_r]).max(initial=0.0)
    assert err <= tol, f"max |rho_gpu - rho_oracle| = {err}"
    return err


# ---------------------------------------------------------------- edm_embed_knn
@pytest.mark.parametrize("case", range(10))
def test_embed_knn_bit_exact(case):
    rng = np.random.default_rng(1000 + case)
    L = [40, 77, 200, 333, 1000, 1450, 64, 65, 500, 257][case]
    E = [1, 2, 3, 5, 8, 20, 4, 10, 13, 6][case]
    tau = 1 + case % 3
    Tp = case % 2
    if case % 4 == 3:
        x = synth.quantise8(synth.coupled_network(2, L, case))[:, 0]   # exact ties
    elif case % 4 == 1:
        x = np.floor(rng.uniform(0, 4, L)).astype(np.float32)             # massive ties
    else:
        x = synth.coupled_network(2, L, case)[:, 1]
    for excl in (True, False):
        if L - (E - 1) * tau - Tp - excl < E + 1:
            continue
        idx, dist, w = libccm.embed_knn(dev(x), E, tau, Tp, excl)
        ri, rd2, rw = O.ccm_table(x.astype(np.float64), E, tau, Tp, excl)
        np.testing.assert_array_equal(idx.cpu().numpy(), ri)
        np.testing.assert_array_equal(dist.cpu().numpy(), np.sqrt(rd2).astype(np.float32))
        np.testing.assert_allclose(w.cpu().numpy(), rw, atol=1e-6, rtol=0)


def test_embed_knn_errors():
    x = dev(np.arange(10, dtype=np.float32))
    with pytest.raises(libccm.EdmError) as e:
        libccm.embed_knn(x, 5, 2, 1)
    assert e.value.status == libccm.EDM_ETOOSHORT
    with pytest.raises(libccm.EdmError) as e:
        libccm.embed_knn(x, 21, 1, 0)
    assert e.value.status == libccm.EDM_EINVAL


# ---------------------------------------------------------------- edm_simplex_optimal_E
def check_simplex(data, E_max, tau=1, s_begin=0, s_end=None):
    optE, rhoE = libccm.simplex_optimal_E(dev(data), E_max, tau, s_begin, s_end, return_rho=True)
    rE, rrho = O.simplex_all(data, E_max, tau, s_begin, s_end)
    np.testing.assert_array_equal(optE.cpu().numpy(), rE)
    g = rhoE.cpu().numpy().astype(np.float64)
    assert np.array_equal(np.isnan(g), np.isnan(rrho))
    np.testing.assert_allclose(g[~np.isnan(g)], rrho[~np.isnan(rrho)], atol=1e-6)
    return optE.cpu().numpy()


def test_simplex_c1_full():
    check_simplex(synth.make_config("c1"), 10)


def test_simplex_c2_sample():
    data = synth.make_config("c2", N=300)
    check_simplex(data, 20)


def test_simplex_quantised_and_ranges():
    data = synth.quantise8(synth.make_config("c2", N=150, L=400))
    check_simplex(data, 20, 1, 17, 131)
    check_simplex(synth.random_dataset(70, 301, 5), 12, 2)   # odd L, tau = 2


# ---------------------------------------------------------------- edm_ccm_all_pairs
def check_ccm(data, E, tau=1, Tp=1, mode="target", excl=True, lib_begin=0, lib_end=None):
    N = data.shape[1]
    lib_end = N if lib_end is None else lib_end
    g = libccm.ccm_all_pairs(dev(data), dev(E, torch.int32), tau, Tp, mode, excl, lib_begin, lib_end)
    torch.cuda.synchronize()
    ref = O.ccm_rows(data, E, tau, Tp, 0 if mode == "target" else 1, excl, lib_begin, lib_end)
    return assert_rho_close(g.cpu().numpy(), ref)


def test_ccm_c1_full_both_modes():
    data = synth.make_config("c1")
    E, _ = O.simplex_all(data, 10)
    for mode in ("target", "library"):
        for Tp in (0, 1):
            check_ccm(data, E, 1, Tp, mode)


def test_ccm_random_ragged():
    # N not a multiple of 32, several E segments, tau = 2, exclusion off as well
    rng = np.random.default_rng(3)
    data = synth.random_dataset(45, 150, 11)
    E = rng.integers(1, 8, 45).astype(np.int32)
    for mode in ("target", "library"):
        check_ccm(data, E, 2, 1, mode)
        check_ccm(data, E, 1, 0, mode, excl=False)
        check_ccm(data, E, 1, 2, mode, lib_begin=7, lib_end=40)


def test_ccm_c2_sample():
    data = synth.make_config("c2", N=400)
    optE = libccm.simplex_optimal_E(dev(data), 20).cpu().numpy()
    for mode in ("target", "library"):
        check_ccm(data, optE, 1, 1, mode, lib_begin=100, lib_end=140)


def test_ccm_all_twenty_E_and_constant_series():
    data = synth.make_config("c2", N=130, L=600)
    data[:, 77] = 0.25  # constant -> NaN column and NaN-free elsewhere
    E = (1 + np.arange(130) % 20).astype(np.int32)
    check_ccm(data, E, 1, 1, "target", lib_begin=60, lib_end=90)
    check_ccm(data, E, 1, 1, "library", lib_begin=60, lib_end=90)


def test_ccm_single_series_and_tiny():
    data = synth.make_config("c2", N=1, L=50)
    check_ccm(data, np.array([3], np.int32), 1, 1, "target")
    data = synth.random_dataset(3, 12, 1)
    check_ccm(data, np.array([1, 2, 3], np.int32), 1, 1, "target")


def test_ccm_long_series_gmem_path():
    # L > 1816: the target tile no longer fits shared memory -> L2/HBM gather variant
    data = synth.make_config("c5", N=40, L=2100)
    E = (1 + np.arange(40) % 6).astype(np.int32)
    check_ccm(data, E, 1, 1, "target", lib_begin=0, lib_end=4)


def test_ccm_deterministic_and_split_invariant():
    data = synth.make_config("c2", N=200, L=500)
    d = dev(data)
    E = libccm.simplex_optimal_E(d, 20)
    a = libccm.ccm_all_pairs(d, E).cpu().numpy()
    b = libccm.ccm_all_pairs(d, E).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    parts = [libccm.ccm_all_pairs(d, E, lib_begin=s, lib_end=min(s + 37, 200)).cpu().numpy() for s in range(0, 200, 37)]
    assert np.array_equal(np.concatenate(parts).view(np.uint32), a.view(np.uint32))


def test_ccm_errors():
    data = dev(synth.make_config("c2", N=10, L=30))
    with pytest.raises(libccm.EdmError) as e:
        libccm.ccm_all_pairs(data, dev(np.full(10, 21), torch.int32))
    assert e.value.status == libccm.EDM_EINVAL
    with pytest.raises(libccm.EdmError) as e:
        libccm.ccm_all_pairs(data, dev(np.full(10, 20), torch.int32))
    assert e.value.status == libccm.EDM_ETOOSHORT


def test_causal_map_host_end_to_end():
    data = synth.make_config("c1")
    optE, rho = libccm.causal_map_host(data, 10, 1, 1)
    rE, _ = O.simplex_all(data, 10)
    np.testing.assert_array_equal(optE, rE)
    assert_rho_close(rho, O.ccm_rows(data, rE, 1, 1, 0, True))


def test_causal_map_host_pinned_chunked_equals_pageable():
    # a page-locked rho buffer switches edm_causal_map_host to 8 row chunks whose copies overlap
    # the next chunk's compute; the map must be byte-identical to the one-shot (pageable) path
    data = synth.make_config("c2", N=2200, L=300)
    N = data.shape[1]
    E1, r1 = libccm.causal_map_host(data, 12, 1, 1)
    pinned = torch.empty((N, N), dtype=torch.float32).pin_memory().numpy()
    E2, r2 = libccm.causal_map_host(data, 12, 1, 1, rho_out=pinned)
    np.testing.assert_array_equal(E1, E2)
    assert np.array_equal(r1.view(np.uint32), r2.view(np.uint32))
    pick = [0, 700, 2199]
    assert_rho_close(r2[pick], np.concatenate([O.ccm_rows(data, E1, 1, 1, 0, True, p, p + 1) for p in pick]))


def test_sugihara_direction_on_gpu():
    data = synth.sugihara_pair(1000)
    rho = libccm.ccm_all_pairs(dev(data), dev(np.array([2, 2]), torch.int32)).cpu().numpy()
    assert rho[1, 0] > 0.9 and abs(rho[0, 1]) < 0.2


# ---------------------------------------------------------------- full BASELINE size, sampled
def test_c3_full_size_sampled():
    """c3 at full size (53,053 x 1,450, the bench workload) in the bench's launch
    configuration (whole 256-library blocks, all targets): optE bit-exact on sampled series (all
    series: tests/test_gpu_full_optE.py), rho within 1e-4 on every target of sampled library rows
    (the oracle computes them one by one)."""
    data = synth.make_config("c3")
    L, N = data.shape
    d = dev(data)
    optE = libccm.simplex_optimal_E(d, 20).cpu().numpy()
    rng = np.random.default_rng(7)
    ss = np.sort(rng.choice(N, 48, replace=False))
    for s in ss:
        e, _, _ = O.simplex(data[:, s].astype(np.float64), 20)
        assert e == optE[s], (s, e, optE[s])
    E_dev = dev(optE, torch.int32)
    for r0 in (0, 26368, N - 256):
        rows = libccm.ccm_all_pairs(d, E_dev, 1, 1, "target", True, r0, r0 + 256).cpu().numpy()
        pick = [0, 117, 255]
        ref = np.concatenate([O.ccm_rows(data, optE, 1, 1, 0, True, r0 + p, r0 + p + 1) for p in pick])
        assert_rho_close(rows[pick], ref)


def test_c4_full_size_sampled():
    """c4 (101,729 x 1,450, the north_star's 8-GPU target) at full size: optE on sampled
    series and rho on every target of sampled library rows (one 256-library block)."""
    data = synth.make_config("c4")
    L, N = data.shape
    d = dev(data)
    rng = np.random.default_rng(11)
    ss = np.sort(rng.choice(N, 24, replace=False))
    optE = libccm.simplex_optimal_E(d, 20).cpu().numpy()
    for s in ss:
        e, _, _ = O.simplex(data[:, s].astype(np.float64), 20)
        assert e == optE[s], (s, e, optE[s])
    r0 = 50_000
    rows = libccm.ccm_all_pairs(d, dev(optE, torch.int32), 1, 1, "target", True, r0, r0 + 256).cpu().numpy()
    pick = [5, 130, 255]
    ref = np.concatenate([O.ccm_rows(data, optE, 1, 1, 0, True, r0 + p, r0 + p + 1) for p in pick])
    assert_rho_close(rows[pick], ref)


def test_c5_long_series_sampled():
    """c5 shape (L = 10,000, E up to 20; kNN/distance-dominated regime): full-length series,
    a sample of 64 series x 64 sampled rows' worth of targets, incl. the forced-E variant
    E[j] = 1 + (j mod 20) that exercises all 20 tables."""
    data = synth.make_config("c5", N=64)
    L, N = data.shape
    d = dev(data)
    optE = libccm.simplex_optimal_E(d, 20, 1, 0, 8).cpu().numpy()
    for s in range(8):
        e, _, _ = O.simplex(data[:, s].astype(np.float64), 20)
        assert e == optE[s]
    forced = (1 + np.arange(N) % 20).astype(np.int32)
    rows = libccm.ccm_all_pairs(d, dev(forced, torch.int32), 1, 1, "target", True, 3, 5).cpu().numpy()
    ref = O.ccm_rows(data, forced, 1, 1, 0, True, 3, 5)
    assert_rho_close(rows, ref)


# ---------------------------------------------------------------- edm_ccm_lagged
def test_lagged_parity_and_single_lag_identity():
    data = synth.random_dataset(45, 160, 21)
    rng = np.random.default_rng(5)
    E = rng.integers(1, 7, 45).astype(np.int32)
    d, Ed = dev(data), dev(E, torch.int32)
    for mode in ("target", "library"):
        g = libccm.ccm_lagged(d, Ed, 1, -3, 2, mode, True, 4, 40).cpu().numpy()
        ref = O.ccm_lagged_rows(data, E, 1, -3, 2, 0 if mode == "target" else 1, True, 4, 40)
        assert_rho_close(g, ref)
        for Tp in (0, 1):
            a = libccm.ccm_lagged(d, Ed, 1, Tp, Tp, mode).cpu().numpy()[:, 0, :]
            b = libccm.ccm_all_pairs(d, Ed, 1, Tp, mode).cpu().numpy()
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_lagged_c3_shape_sampled_and_causal_lag():
    data = synth.make_config("c3", N=2048)
    d = dev(data)
    optE = libccm.simplex_optimal_E(d, 20).cpu().numpy()
    g = libccm.ccm_lagged(d, dev(optE, torch.int32), 1, -2, 2, "target", True, 256, 512).cpu().numpy()
    pick = [0, 101, 255]
    ref = np.concatenate([O.ccm_lagged_rows(data, optE, 1, -2, 2, 0, True, 256 + p, 257 + p) for p in pick])
    assert_rho_close(g[pick], ref)
    from tests.test_oracle_lagged import delayed_pair
    pair = delayed_pair(1000, 3)
    r = libccm.ccm_lagged(dev(pair), dev(np.array([2, 2]), torch.int32), 1, -6, 3).cpu().numpy()
    assert -6 + int(np.argmax(r[1, :, 0])) == -4


# ---------------------------------------------------------------- edm_ccm_rows (library lists, multi-GPU dealing)
def test_ccm_rows_list_equals_range_rows():
    """A library LIST gives exactly the rows of the range call (byte for byte), in list order,
    duplicates included; library mode deals rows this way across GPUs."""
    data = synth.make_config("c2", N=300, L=400)
    d = dev(data)
    E = libccm.simplex_optimal_E(d, 20)
    rng = np.random.default_rng(8)
    lst = np.concatenate([rng.permutation(300)[:270], [5, 5, 299]]).astype(np.int32)
    for mode in ("target", "library"):
        full = libccm.ccm_all_pairs(d, E, 1, 1, mode).cpu().numpy()
        rows = libccm.ccm_rows(d, E, lst, 1, 1, mode).cpu().numpy()
        assert np.array_equal(rows.view(np.uint32), full[lst].view(np.uint32))
    Eh = E.cpu().numpy()
    from paper_2011_11082_b200 import distributed as D
    parts = D.assign_rows(Eh, 3, "library")
    got = np.concatenate([libccm.ccm_rows(d, E, p, 1, 1, "library").cpu().numpy() for p in parts])
    order = np.concatenate(parts)
    full = libccm.ccm_all_pairs(d, E, 1, 1, "library").cpu().numpy()
    assert np.array_equal(got.view(np.uint32), full[order].view(np.uint32))
