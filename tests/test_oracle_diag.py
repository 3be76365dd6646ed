"""Pins of the oracle's selection diagnostics (App. A skewness, App. D ideal
lookup) against closed forms, brute force and invariants
(S:358-366)."""
import itertools

import numpy as np

import oracle


def _softmax(z):
    e = np.exp(z - z.max())
    return e / e.sum()


def test_uniform_logits_give_top_fraction():
    # uniform logits, top_frac = 0.01, L = 1000 -> 0.01 (q = 0 makes every z_j = 0)
    L, d = 1000, 16
    K = np.random.default_rng(0).standard_normal((1, L, d))
    Q = np.zeros((1, 1, d))
    out = oracle.diagnostics(Q, K, np.zeros((1, 1, L), bool), 1.0, 0.01)
    assert abs(out["skew"][0, 0] - 0.01) < 1e-12
    # the ideal k-set at k = 0 is empty: recall 1 by convention, no mass
    assert out["k"][0, 0] == 0 and out["recall"][0, 0] == 1.0 and out["mass_ideal"][0, 0] == 0.0


def test_dominant_key_concentrates_mass():
    # S:430 / S:363: one key with a logit margin >= 20 -> top-1% sum ~ 1 (1e-4) and the
    # ideal lookup at T = 0.5 returns exactly that key
    L, d = 500, 8
    rng = np.random.default_rng(1)
    K = 0.01 * rng.standard_normal((1, L, d))
    K[0, 123] = 0.0
    K[0, 123, 0] = 30.0
    Q = np.zeros((1, 1, d))
    Q[0, 0, 0] = 1.0
    sel = np.zeros((1, 1, L), bool)
    sel[0, 0, 123] = True
    out = oracle.diagnostics(Q, K, sel, 1.0, 0.01, T=0.5)
    assert out["skew"][0, 0] >= 1 - L * np.exp(-20) and abs(out["skew"][0, 0] - 1) < 1e-4
    assert out["n_T"][0, 0] == 1 and abs(out["mass_T"][0, 0] - out["mass_sel"][0, 0]) < 1e-15
    assert out["recall"][0, 0] == 1.0 and out["k"][0, 0] == 1


def test_full_fraction_and_monotone():
    # S:431 top_frac = 1 -> exactly 1; S:455 monotone non-decreasing in top_frac
    rng = np.random.default_rng(2)
    L, d = 300, 32
    K = rng.standard_normal((2, L, d))
    Q = 2.0 * rng.standard_normal((1, 2, d))
    prev = np.zeros((1, 2))
    for f in (0.001, 0.01, 0.05, 0.3, 0.9, 1.0):
        s = oracle.diagnostics(Q, K, np.zeros((1, 2, L), bool), 0.25, f)["skew"]
        assert (s >= prev - 1e-15).all()
        prev = s
    assert np.abs(prev - 1.0).max() < 1e-12


def test_threshold_zero_and_full_selection():
    # T = 0 selects every key (R6); a full selection retrieves all mass with recall 1
    rng = np.random.default_rng(3)
    L, d = 257, 16
    K = rng.standard_normal((1, L, d))
    Q = rng.standard_normal((2, 1, d))
    out = oracle.diagnostics(Q, K, np.ones((2, 1, L), bool), 0.5, 0.01, T=0.0)
    assert (out["n_T"] == L).all()
    assert np.abs(out["mass_T"] - 1).max() < 1e-12
    assert (out["recall"] == 1.0).all() and (out["k"] == L).all()
    assert np.abs(out["mass_sel"] - 1).max() < 1e-12 and np.abs(out["mass_ideal"] - 1).max() < 1e-12


def test_brute_force_matched_budget():
    # App. D: the ideal k-set is the best k-subset ("upper bound"): its mass equals the
    # maximum over ALL k-subsets (exhaustive on L = 10), recall = |sel n top_k| / k
    rng = np.random.default_rng(4)
    L, d = 10, 6
    K = rng.standard_normal((1, L, d))
    for trial in range(30):
        Q = rng.standard_normal((1, 1, d)) * 2
        k = int(rng.integers(1, L))
        sel = np.zeros((1, 1, L), bool)
        sel[0, 0, rng.choice(L, k, replace=False)] = True
        out = oracle.diagnostics(Q, K, sel, 1.0, 0.3, T=0.1)
        z = (K[0] @ Q[0, 0]) * 1.0
        a = _softmax(z)
        best = max(a[list(c)].sum() for c in itertools.combinations(range(L), k))
        assert abs(out["mass_ideal"][0, 0] - best) < 1e-12
        assert abs(out["mass_sel"][0, 0] - a[sel[0, 0]].sum()) < 1e-12
        assert out["mass_ideal"][0, 0] >= out["mass_sel"][0, 0] - 1e-15
        top = set(np.argsort(-a, kind="stable")[:k])
        assert abs(out["recall"][0, 0] - len(top & set(np.flatnonzero(sel[0, 0]))) / k) < 1e-15
        # skew over the top ceil(0.3 L) = 3 scores; ideal-at-threshold = {a_j > 0.1}
        assert abs(out["skew"][0, 0] - np.sort(a)[::-1][:3].sum()) < 1e-12
        assert out["n_T"][0, 0] == (a > 0.1).sum()
        assert abs(out["mass_T"][0, 0] - a[a > 0.1].sum()) < 1e-12
        # a selection that IS the top-k set has recall 1 and captures the ideal mass
        sel2 = np.zeros_like(sel)
        sel2[0, 0, list(top)] = True
        o2 = oracle.diagnostics(Q, K, sel2, 1.0, 0.3)
        assert o2["recall"][0, 0] == 1.0 and abs(o2["mass_sel"][0, 0] - best) < 1e-12


def test_top_count():
    assert oracle.top_count(0.01, 1000) == 10
    assert oracle.top_count(0.01, 32768) == 328
    assert oracle.top_count(1e-9, 50) == 1
    assert oracle.top_count(1.0, 77) == 77
