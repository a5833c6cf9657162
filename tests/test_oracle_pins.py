"""Pins of the fp64 CPU oracle against things other than itself (task rule 3):
SPEC.md worked examples (tests/golden/spec_examples.json), closed forms
(tests/golden/ccm_worked_example.json), library routines (numpy lexsort / corrcoef),
brute force on tiny inputs, and invariants. PAPER.md prints no numeric worked example.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2011_11082_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- SPEC examples
def test_pearson_spec_examples():
    for ex in _gold("spec_examples.json")["pearson"]:
        r = O.pearson(ex["a"], ex["b"])
        if ex["rho"] == "nan":
            assert math.isnan(r), ex["cite"]
        else:
            assert r == pytest.approx(ex["rho"], abs=1e-15), ex["cite"]


def test_embedding_coordinates_via_distance():
    # d2 against an all-zero partner series is sum_m x[t - m tau]^2: isolate one coordinate by
    # differencing E and E-1 (pins the backward-lag direction and tau).
    for ex in _gold("spec_examples.json")["embed_coordinate"]:
        x = np.array(ex["series"], float)
        z = np.zeros_like(x)
        t, k, tau = ex["t"], ex["k"], ex["tau"]
        hi = O.dist2(x, t, z, t, k + 1, tau)
        lo = O.dist2(x, t, z, t, k, tau) if k > 0 else 0.0
        assert math.sqrt(hi - lo) == pytest.approx(ex["value"]), ex["cite"]


def test_distance_examples():
    g = _gold("spec_examples.json")
    x = np.array(g["distances_E1"]["series"], float)
    d = [[O.dist2(x, t, x, s, 1, 1) for s in range(3)] for t in range(3)]
    assert d == g["distances_E1"]["d2"]
    e = g["distance_E2"]
    x = np.array(e["series"], float)
    assert O.dist2(x, e["t"], x, e["s"], 2, 1) == e["d2"]
    assert O.dist2(x, e["s"], x, e["t"], 2, 1) == e["d2"]  # symmetry


def test_partial_select_examples():
    # realise the raw distance rows of S:140-141 as 1-D kNN rows: query value 0 against
    # candidates +-sqrt(d2) (exact for perfect squares)
    for ex in _gold("spec_examples.json")["partial_select"]:
        d2 = np.array(ex["d2"], float)
        cand = np.sqrt(d2) * np.where(np.arange(len(d2)) % 2 == 0, 1, -1)
        b = cand
        a = np.array([0.0])
        idx, sel = O.knn(a, 0, 0, b, 0, len(b) - 1, 1, 1, False) if ex["k"] == 2 else (None, None)
        assert idx[0].tolist() == ex["idx"], ex["cite"]
        if "sel_d2" in ex:
            assert sel[0].tolist() == ex["sel_d2"]


def test_knn_exclusion_example():
    ex = _gold("spec_examples.json")["knn_exclusion"]
    idx, d2, w = O.ccm_table(np.array(ex["series"], float), ex["E"], ex["tau"], ex["Tp"], True)
    assert idx[ex["query_t"]].tolist() == ex["idx"], ex["cite"]
    # exclusion off: the query's own point is its nearest neighbour at distance 0
    idx0, d20, w0 = O.ccm_table(np.array(ex["series"], float), ex["E"], ex["tau"], ex["Tp"], False)
    assert idx0[ex["query_t"], 0] == ex["query_t"] and d20[ex["query_t"], 0] == 0.0
    assert w0[ex["query_t"], 0] == w0[ex["query_t"]].max()


def test_weights_examples():
    for ex in _gold("spec_examples.json")["weights"]:
        d2 = np.array(ex["d"], float) ** 2
        w = O.weights(d2)
        np.testing.assert_allclose(w, ex["w"], atol=ex["tol"], rtol=0, err_msg=ex["cite"])
        assert abs(w.sum() - 1.0) < 1e-15


def test_weights_closed_form_and_floor():
    # u_k = exp(-d_k/d_1): ratios of consecutive weights are exp(-(d_{k+1}-d_k)/d_1)
    d = np.array([0.5, 0.75, 1.5, 4.0])
    w = O.weights(d ** 2)
    for j in range(3):
        assert w[j + 1] / w[j] == pytest.approx(math.exp(-(d[j + 1] - d[j]) / d[0]), rel=1e-14)
    # the 1e-6 floor: a very far neighbour keeps weight 1e-6 / sum
    d = np.array([1.0, 100.0])
    w = O.weights(d ** 2)
    u = np.array([math.exp(-1.0), 1e-6])
    np.testing.assert_allclose(w, u / u.sum(), rtol=1e-15)


# ---------------------------------------------------------------- closed-form CCM example
def test_ccm_worked_example():
    g = _gold("ccm_worked_example.json")
    x = np.array(g["library"], float)
    y = np.array(g["target"], float)
    a = math.exp(-1.0)
    closed = {
        1: np.array([30 / (1 + a) + 40 * a / (1 + a), 30, 30 / (1 + a) + 20 * a / (1 + a)]),
        0: np.array([20 / (1 + a) + 30 * a / (1 + a), 20, 30, 30 / (1 + a) + 20 * a / (1 + a)]),
    }
    for case in g["cases"]:
        Tp = case["Tp"]
        idx, d2, w = O.ccm_table(x, g["E"], g["tau"], Tp, g["exclude_self"])
        assert idx.tolist() == case["idx"]
        rho, p, o = O.xmap(idx, w, 0, y, Tp)
        np.testing.assert_allclose(p, closed[Tp], rtol=1e-14)
        assert o.tolist() == case["o"]
        assert rho == pytest.approx(case["rho"], abs=case.get("tol", 1e-14))
        assert rho == pytest.approx(np.corrcoef(closed[Tp], case["o"])[0, 1], abs=1e-12)
        # and through the dataset-level phase-2 entry point (library row 0, target column 1)
        data = np.stack([x, y], axis=1).astype(np.float32)
        R = O.ccm_rows(data, np.array([1, 1]), 1, Tp, O.MODE_TARGET, True)
        assert R[0, 1] == pytest.approx(case["rho"], abs=1e-12)


# ---------------------------------------------------------------- library routines / brute force
def brute_knn(a, qlo, qhi, b, clo, chi, E, tau, excl):
    """Full distance matrix + full stable sort (np.lexsort by (d2, s)): the definition."""
    rows_i, rows_d = [], []
    for t in range(qlo, qhi + 1):
        s = np.arange(clo, chi + 1)
        if excl:
            s = s[s != t]
        acc = np.zeros(len(s))
        for m in range(E):
            diff = a[t - m * tau] - b[s - m * tau]
            acc = acc + diff * diff
        order = np.lexsort((s, acc))[: E + 1]
        rows_i.append(s[order])
        rows_d.append(acc[order])
    return np.array(rows_i), np.array(rows_d)


@pytest.mark.parametrize("seed", range(12))
def test_knn_matches_bruteforce(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(30, 200))
    E = int(rng.integers(1, 6))
    tau = int(rng.integers(1, 3))
    Tp = int(rng.integers(0, 2))
    if seed % 3 == 0:
        x = np.floor(rng.uniform(0, 6, L))  # heavy exact ties
    else:
        x = rng.standard_normal(L)
    for excl in (True, False):
        idx, d2, _ = O.ccm_table(x, E, tau, Tp, excl)
        lo, hi = (E - 1) * tau, L - 1 - Tp
        bi, bd = brute_knn(x, lo, hi, x, lo, hi, E, tau, excl)
        assert np.array_equal(idx, bi)
        assert np.array_equal(d2, bd)  # same op order -> bit-identical
    # disjoint library/target (phase-1 form)
    y = rng.standard_normal(L)
    lo = (E - 1) * tau
    idx, d2 = O.knn(x, lo, L - 2, y, lo, L - 2, E, tau, False)
    bi, bd = brute_knn(x, lo, L - 2, y, lo, L - 2, E, tau, False)
    assert np.array_equal(idx, bi) and np.array_equal(d2, bd)


def test_knn_E1_is_sorted_value_order():
    # at E=1 the neighbours of t are the points closest in value: argsort(|x - x[t]|, stable)
    rng = np.random.default_rng(7)
    x = rng.standard_normal(120)
    idx, _, _ = O.ccm_table(x, 1, 1, 0, True)
    for t in range(len(x)):
        s = np.array([u for u in range(len(x)) if u != t])
        order = s[np.argsort(np.abs(x[s] - x[t]), kind="stable")][:2]
        assert idx[t].tolist() == order.tolist()


def test_pearson_matches_numpy_and_invariants():
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(2, 500))
        a, b = rng.standard_normal(n), rng.standard_normal(n)
        r = O.pearson(a, b)
        assert r == pytest.approx(np.corrcoef(a, b)[0, 1], abs=1e-12)
        assert O.pearson(b, a) == pytest.approx(r, abs=1e-12)
        assert O.pearson(3.5 * a + 2.0, b) == pytest.approx(r, abs=1e-9)
    assert math.isnan(O.pearson([0.1] * 1449, list(range(1449))))  # constant -> NaN even when the mean rounds


def test_table_shapes_and_weight_rows():
    x = synth.coupled_network(3, 150, 5)[:, 0].astype(float)
    for E in (1, 3, 7):
        for Tp in (0, 1):
            idx, d2, w = O.ccm_table(x, E, 2, Tp, True)
            assert idx.shape == (150 - (E - 1) * 2 - Tp, E + 1)  # n_E rows
            np.testing.assert_allclose(w.sum(axis=1), 1.0, atol=1e-12)
            assert (w > 0).all() and (w <= 1).all()
            assert (np.diff(d2, axis=1) >= 0).all()  # ascending (P:449 garble, reading c.10)
            for r in range(len(idx)):
                assert len(set(idx[r])) == E + 1


# ---------------------------------------------------------------- simplex semantics
def test_simplex_sine_is_predictable():
    x = synth.sine(200)[:, 0].astype(float)
    assert O.simplex_rho_E(x, 2, 1) >= 0.99


def test_simplex_noise_is_not():
    vals = [O.simplex_rho_E(synth.noise(1, 500, s)[:, 0].astype(float), 3, 1) for s in range(20)]
    assert max(abs(v) for v in vals) < 0.2


def test_simplex_exact_repeat():
    # library half is an exact copy of the target half -> each query's nearest library
    # point is its twin at d=0 and the forecast equals the true next value
    rng = np.random.default_rng(1)
    half = rng.standard_normal(40)
    x = np.concatenate([half, half])
    for E in (1, 2, 3):
        assert O.simplex_rho_E(x, E, 1) == pytest.approx(1.0, abs=1e-5)


def test_simplex_split_at_ceil():
    # L odd: library = first ceil(L/2) samples. Build x so that the target half
    # under the ceil split is an exact copy of lib[0:Ltgt]: then rho = 1 (up to the 1e-6 floor).
    rng = np.random.default_rng(2)
    a = rng.standard_normal(30)
    x = np.concatenate([a, [5.0], a])  # L = 61, ceil split -> lib = a + [5], tgt = a
    assert O.simplex_rho_E(x, 1, 1) == pytest.approx(1.0, abs=1e-5)
    x_floor = np.concatenate([a, [5.0], a])[1:]  # shifting by one breaks the twin alignment
    assert O.simplex_rho_E(x_floor, 1, 1) < 0.999


def test_simplex_optE_rules():
    x = synth.sine(200)[:, 0].astype(float)
    e, rho, flag = O.simplex(x, 1)
    assert e == 1 and not flag  # E_max = 1 -> 1
    e, rho, flag = O.simplex(np.full(100, 0.3), 5)
    assert e == 1 and flag and np.isnan(rho).all()  # constant -> flagged, E=1
    x = synth.coupled_network(4, 400, 11)[:, 1].astype(float)
    e, rho, flag = O.simplex(x, 10)
    assert e == int(np.nanargmax(rho)) + 1  # argmax, first (smallest) E on ties


def test_simplex_too_short_is_nan():
    x = np.random.default_rng(0).standard_normal(20)
    # Llib = 10 -> candidates (E-1)..8: E=5 has 5 candidates < k=6 -> NaN
    assert math.isnan(O.simplex_rho_E(x, 5, 1))
    assert not math.isnan(O.simplex_rho_E(x, 4, 1))


# ---------------------------------------------------------------- CCM semantics
def test_alg1_equals_alg2_both_modes():
    # Alg. 2 is a pure reuse optimisation of Alg. 1: identical elementwise
    for seed in range(4):
        data = synth.random_dataset(12, 90, 100 + seed)
        E, _ = O.simplex_all(data, 5)
        for mode in (O.MODE_TARGET, O.MODE_LIBRARY):
            for Tp in (0, 1):
                a = O.ccm_rows(data, E, 1, Tp, mode, True, naive=False)
                b = O.ccm_rows(data, E, 1, Tp, mode, True, naive=True)
                assert np.array_equal(a, b, equal_nan=True)


def test_duplicated_series_rows_and_columns():
    data = synth.random_dataset(8, 120, 9)
    data[:, 5] = data[:, 2]
    E, _ = O.simplex_all(data, 6)
    assert E[5] == E[2]
    R = O.ccm_rows(data, E, 1, 1, O.MODE_TARGET, True)
    assert np.array_equal(R[5], R[2], equal_nan=True)
    assert np.array_equal(R[:, 5], R[:, 2], equal_nan=True)


def test_exclusion_off_is_trivial():
    # without self-exclusion each point's nearest neighbour is itself (d=0) and every
    # cross map is ~perfect: the reason exclusion is on by default
    data = synth.coupled_network(5, 100, 4, n_const=0, noise_frac=0.0)  # continuous: no duplicate points
    E = np.full(5, 2, np.int32)
    R = O.ccm_rows(data, E, 1, 1, O.MODE_TARGET, False)
    assert np.nanmin(R) > 0.9999


def test_sugihara_asymmetry_and_convergence():
    # x drives y (beta_yx = 0.1, beta_xy = 0): y's manifold encodes x, so the cross map from
    # library y to target x (rho[y, x]) is high and the reverse is low;
    # skill grows with library length (convergence). Uniform E = 2.
    out = {}
    for L in (200, 1000):
        data = synth.sugihara_pair(L)
        R = O.ccm_rows(data, np.array([2, 2]), 1, 1, O.MODE_TARGET, True)
        out[L] = R
        assert R[1, 0] > 0.6 and abs(R[0, 1]) < 0.2
        assert R[1, 0] - R[0, 1] > 0.5
    assert out[1000][1, 0] > out[200][1, 0] + 0.1
    # library mode with optimal E also detects the direction
    data = synth.sugihara_pair(400)
    E, _ = O.simplex_all(data, 10)
    R = O.ccm_rows(data, E, 1, 1, O.MODE_LIBRARY, True)
    assert R[1, 0] > R[0, 1] + 0.3


def test_zero_coupling_is_small():
    data = synth.sugihara_pair(500, beta_yx=0.0)
    R = O.ccm_rows(data, np.array([2, 2]), 1, 1, O.MODE_TARGET, True)
    assert abs(R[1, 0]) < 0.2 and abs(R[0, 1]) < 0.2


def test_constant_series_gives_nan_not_error():
    data = synth.random_dataset(6, 80, 3)
    data[:, 4] = 0.7
    E, _ = O.simplex_all(data, 4)
    assert E[4] == 1
    R = O.ccm_rows(data, E, 1, 1, O.MODE_TARGET, True)
    assert np.isnan(R[:, 4]).all()
    assert not np.isnan(np.delete(R, 4, axis=1)).any()
