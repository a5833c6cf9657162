"""The opt-in 16-bit lookup targets (EDM_LOOKUP_U16, include/libccm.h).

Not a paper step: the lookup of Alg. 5 with every target series mapped affinely
onto 16-bit codes. Pearson rho is invariant under the affine map, so the result is
the rho of the rounded series; the bar is the north_star's: within 1e-4 of the fp64 oracle,
NaN exactly where the oracle has NaN. 64-target tiles that the guard flags (a target whose
observed window has sd below range / 16, or whose codes are constant while its values are not)
run on the fp32 path and must equal the default lookup byte for byte; kNN tables and optE are
not touched by the option.
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


def same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32))


def pair(data, E, tau=1, Tp=1, mode="target", excl=True, lb=0, le=None):
    """(u16 rows, fp32 rows, oracle rows) of libraries [lb, le)."""
    N = data.shape[1]
    le = N if le is None else le
    d, Ed = dev(data), dev(E, torch.int32)
    q = libccm.ccm_all_pairs(d, Ed, tau, Tp, mode, excl, lb, le, lookup="u16").cpu().numpy()
    f = libccm.ccm_all_pairs(d, Ed, tau, Tp, mode, excl, lb, le).cpu().numpy()
    ref = O.ccm_rows(data, E, tau, Tp, 0 if mode == "target" else 1, excl, lb, le)
    return q, f, ref


def test_u16_small_maps_both_modes():
    data = synth.make_config("c1")
    E, _ = O.simplex_all(data, 10)
    for mode in ("target", "library"):
        for Tp in (0, 1):
            q, f, ref = pair(data, E, 1, Tp, mode)
            assert_rho_close(q, ref)
    rng = np.random.default_rng(3)
    data = synth.random_dataset(45, 150, 11)       # ragged N, several E segments
    E = rng.integers(1, 8, 45).astype(np.int32)
    for mode in ("target", "library"):
        assert_rho_close(pair(data, E, 2, 1, mode)[0], pair(data, E, 2, 1, mode)[2])
        q, f, ref = pair(data, E, 1, 0, mode, excl=False)
        assert_rho_close(q, ref)
        q, f, ref = pair(data, E, 1, 2, mode, lb=7, le=40)
        assert_rho_close(q, ref)


def test_u16_c2_all_twenty_E_and_constant_series():
    data = synth.make_config("c2", N=400)
    optE = libccm.simplex_optimal_E(dev(data), 20).cpu().numpy()
    for mode in ("target", "library"):
        q, f, ref = pair(data, optE, 1, 1, mode, lb=100, le=140)
        assert_rho_close(q, ref)
    data = synth.make_config("c2", N=130, L=600)
    data[:, 77] = 0.25
    E = (1 + np.arange(130) % 20).astype(np.int32)
    for mode in ("target", "library"):
        q, f, ref = pair(data, E, 1, 1, mode, lb=60, le=90)
        assert_rho_close(q, ref)
        assert np.isnan(q[:, 77]).all()


def test_u16_guard_heavy_tails_fall_back_to_fp32():
    """Every series with one outlier of 400 sd: range / sd > 16 everywhere -> every tile on the
    fp32 path -> byte-identical to the default lookup."""
    data = synth.make_config("c2", N=150, L=500).astype(np.float64)
    data[123, :] += 400.0 * data.std(axis=0)
    data = data.astype(np.float32)
    E = (1 + np.arange(150) % 6).astype(np.int32)
    for mode in ("target", "library"):
        q, f, ref = pair(data, E, 1, 1, mode)
        assert same_bits(q, f)
        assert_rho_close(q, ref)


def test_u16_guard_mixed_tiles():
    """Outliers in a few series only: their 64-target tiles run on fp32 (byte-identical columns),
    the others on the codes; everything within the bar."""
    data = synth.make_config("c2", N=300, L=700).astype(np.float64)
    bad = [5, 131, 299]
    for j in bad:
        data[321, j] += 500.0 * data[:, j].std()
    data = data.astype(np.float32)
    E = libccm.simplex_optimal_E(dev(data), 20).cpu().numpy()
    q, f, ref = pair(data, E, 1, 1, "library", lb=0, le=40)
    assert_rho_close(q, ref)
    assert same_bits(q[:, bad], f[:, bad])
    assert not same_bits(q, f)  # the unflagged tiles do use the codes


def test_u16_window_that_rounds_to_a_constant():
    """A series whose variation outside the first rows is far below one 16-bit step: its observed
    windows are not constant but their codes are -> guard -> fp32 path, byte-identical to the
    default lookup (not NaN). That column itself (variation 1e-7 under an offset of 4: range / sd
    = 4e7) is beyond the fp32 lookup's conditioning too (lookup conditioning), so
    the oracle bar is checked on the other columns."""
    data = synth.make_config("c2", N=70, L=400).astype(np.float64)
    j = 33
    data[:, j] = 1.0 + 1e-7 * np.sin(np.arange(400) * 0.7)
    data[0, j] = 5.0
    data = data.astype(np.float32)
    E = (1 + np.arange(70) % 4).astype(np.int32)
    E[j] = 3
    q, f, ref = pair(data, E, 1, 1, "target")
    assert same_bits(q[:, j], f[:, j]) and not np.isnan(q[:, j]).all()
    keep = np.arange(70) != j
    assert_rho_close(q[:, keep], ref[:, keep])


def test_u16_lagged_rows_and_long_series():
    data = synth.random_dataset(45, 160, 21)
    rng = np.random.default_rng(5)
    E = rng.integers(1, 7, 45).astype(np.int32)
    d, Ed = dev(data), dev(E, torch.int32)
    for mode in ("target", "library"):
        g = libccm.ccm_lagged(d, Ed, 1, -3, 2, mode, True, 4, 40, lookup="u16").cpu().numpy()
        ref = O.ccm_lagged_rows(data, E, 1, -3, 2, 0 if mode == "target" else 1, True, 4, 40)
        assert_rho_close(g, ref)
        lst = np.array([40, 3, 3, 17], np.int32)
        rows = libccm.ccm_rows(d, Ed, lst, 1, 1, mode, lookup="u16").cpu().numpy()
        full = libccm.ccm_all_pairs(d, Ed, 1, 1, mode, lookup="u16").cpu().numpy()
        assert same_bits(rows, full[lst])
    # L beyond the shared-memory tile: the option is ignored (the fp32 L2-gather lookup runs)
    data = synth.make_config("c5", N=40, L=2100)
    E = (1 + np.arange(40) % 6).astype(np.int32)
    d, Ed = dev(data), dev(E, torch.int32)
    q = libccm.ccm_all_pairs(d, Ed, 1, 1, "target", True, 0, 4, lookup="u16").cpu().numpy()
    f = libccm.ccm_all_pairs(d, Ed, 1, 1, "target", True, 0, 4).cpu().numpy()
    assert same_bits(q, f)


def test_u16_c3_full_size_sampled():
    """c3 at full size in the bench's launch configuration (whole 256-library blocks, all
    targets, --lookup u16): rho within 1e-4 of the oracle on every target of sampled rows, and
    the whole blocks within 1e-4 of the fp32 lookup."""
    data = synth.make_config("c3")
    L, N = data.shape
    d = dev(data)
    optE = libccm.simplex_optimal_E(d, 20)
    Eh = optE.cpu().numpy()
    worst = 0.0
    for r0 in (0, 26368, N - 256):
        q = libccm.ccm_all_pairs(d, optE, 1, 1, "target", True, r0, r0 + 256, lookup="u16").cpu().numpy()
        f = libccm.ccm_all_pairs(d, optE, 1, 1, "target", True, r0, r0 + 256).cpu().numpy()
        assert np.array_equal(np.isnan(q), np.isnan(f))
        ok = ~np.isnan(q)
        worst = max(worst, float(np.abs(q[ok].astype(np.float64) - f[ok]).max(initial=0.0)))
        pick = [0, 117, 255]
        ref = np.concatenate([O.ccm_rows(data, Eh, 1, 1, 0, True, r0 + p, r0 + p + 1) for p in pick])
        assert_rho_close(q[pick], ref)
    print(f"c3 u16 vs fp32 lookup, 768 rows x {N} targets: max |drho| = {worst:.3g}")
    assert worst <= RHO_TOL
