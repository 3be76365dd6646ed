"""Pins for the oracle's centroid scoring and thresholding (Eq. 1-3, section 4.1).

Each check is fixed by the paper / SPEC worked values, a closed form, or an
invariant of the definition -- never by re-typing the oracle's formula."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


@pytest.mark.parametrize("ex", GOLD["eq1_examples"], ids=lambda e: e["cite"][:12])
def test_eq1_worked_examples(ref, ex):
    _, S, _ = ref.scores(np.array(ex["q"]), np.array(ex["C"]), np.array(ex["N"]), ex["scale"])
    np.testing.assert_allclose(S, ex["S"], rtol=1e-13, atol=0)


@pytest.mark.parametrize("ex", GOLD["threshold_examples"], ids=lambda e: e["cite"][:12])
def test_threshold_worked_example(ref, ex):
    s, S, _ = ref.scores(np.array(ex["q"]), np.array(ex["C"]), np.array(ex["N"]), ex["scale"])
    assert list(S > ex["T"]) == ex["selected"]
    assert list(ref.select_singlepass(s, np.array(ex["N"]), ex["T"])) == ex["selected"]


def _rand_table(rng, c, d, nmax=50):
    C = rng.standard_normal((c, d))
    N = rng.integers(1, nmax, size=c)
    return C, N


@pytest.mark.parametrize("d", [8, 64, 128])
def test_normalisation_sum_N_S_is_one(ref, d):
    """S:219 / S:296: sum_i N_i S_i = 1 (Eq. 1 is a size-weighted softmax)."""
    rng = np.random.default_rng(d)
    for _ in range(200):
        c = int(rng.integers(1, 64))
        C, N = _rand_table(rng, c, d)
        q = rng.standard_normal(d) * rng.uniform(0.1, 5)
        _, S, _ = ref.scores(q, C, N, 1.0 / np.sqrt(d))
        assert abs(np.sum(N * S) - 1.0) < 1e-12
        assert np.all(S >= 0)


def test_closed_forms(ref):
    rng = np.random.default_rng(1)
    d = 16
    C = rng.standard_normal((1, d))
    for n in [1, 7, 1000]:
        _, S, lse = ref.scores(rng.standard_normal(d), C, np.array([n]), 0.3)
        assert S[0] == pytest.approx(1.0 / n, rel=1e-14)
    # equal logits -> S = 1 / sum N
    C = np.tile(rng.standard_normal(d), (5, 1))
    N = np.array([1, 2, 3, 4, 5])
    _, S, _ = ref.scores(rng.standard_normal(d), C, N, 1.0)
    np.testing.assert_allclose(S, 1.0 / 15, rtol=1e-13)


def test_lse_is_log_weighted_sum(ref):
    """lse = log sum_j N_j exp(s_j), checked against numpy's logaddexp.reduce."""
    rng = np.random.default_rng(2)
    C, N = _rand_table(rng, 40, 32)
    s, _, lse = ref.scores(rng.standard_normal(32) * 3, C, N, 0.5)
    assert lse == pytest.approx(np.logaddexp.reduce(s + np.log(N)), rel=1e-13)


@pytest.mark.parametrize("beta", [-500.0, -3.0, 7.5, 500.0])
def test_shift_invariance(ref, beta):
    """adding beta to every logit leaves every S_i (and the selection) unchanged.
    The shift is realised through an extra coordinate with q_extra = beta, C_extra = 1."""
    rng = np.random.default_rng(3)
    d, c = 24, 30
    C, N = _rand_table(rng, c, d)
    q = rng.standard_normal(d) * 2
    _, S0, _ = ref.scores(q, C, N, 1.0)
    q1 = np.concatenate([q, [beta]])
    C1 = np.concatenate([C, np.ones((c, 1))], axis=1)
    _, S1, _ = ref.scores(q1, C1, N, 1.0)
    np.testing.assert_allclose(S1, S0, rtol=1e-9)
    T = np.median(S0)
    assert np.array_equal(S0 > T, S1 > T)


def test_singlepass_equals_twopass(ref):
    """S:270-275 / S:481: single-pass e_i > D*T selects exactly S_i > T, logits up to 1e3."""
    rng = np.random.default_rng(4)
    mism = 0
    for trial in range(1000):
        c = int(rng.integers(1, 80))
        N = rng.integers(1, 40, size=c)
        s = rng.standard_normal(c) * rng.choice([1.0, 10.0, 100.0]) + rng.uniform(-1e3, 1e3)
        m = s.max()
        S = np.exp(s - m) / np.sum(N * np.exp(s - m))
        T = float(rng.choice(S)) * rng.uniform(0.5, 1.5) if trial % 10 else 0.0
        sp = ref.select_singlepass(s, N, T)
        # two-pass through the oracle's Eq. 1 path: logits via a 1-dim table
        _, S2, _ = ref.scores(np.array([1.0]), s.reshape(-1, 1), N, 1.0)
        tp = (S2 > T) if T > 0 else np.ones(c, bool)
        inband = np.abs(S2 - T) <= 1e-12 * max(T, 1e-300)
        mism += int(np.sum((sp != tp) & ~inband))
    assert mism == 0


def _single_level_index(ref, rng, H, c, d, levels=1):
    import oracle

    C2 = rng.standard_normal((H, c, d))
    N2 = rng.integers(1, 30, size=(H, c)).astype(np.int32)
    key_off = np.concatenate([np.zeros((H, 1), np.int32), np.cumsum(N2, axis=1, dtype=np.int32)],
                             axis=1)
    L = int(N2.sum(axis=1).max())
    return oracle.Index(levels=1, dtype=oracle.F32, H=H, L=L, d=d, c2=c, C2=C2, N2=N2,
                        key_off=key_off, perm=None)


def test_threshold_edges_and_monotonicity(ref):
    rng = np.random.default_rng(5)
    idx = _single_level_index(ref, rng, 2, 50, 16)
    Q = rng.standard_normal((3, 2, 1, 16)) * 2
    out0 = ref.lookup(Q, idx, 0.25, 0.0)
    assert out0["sel2"].all()  # T = 0 selects all (R6)
    Smax = np.nanmax(ref.lookup(Q, idx, 0.25, 1e-9)["Sbar2"])
    assert not ref.lookup(Q, idx, 0.25, Smax)["sel2"].any()  # T >= max S -> none
    prev = None
    for T in [1e-5, 1e-4, 1e-3, 5e-3, 2e-2]:
        sel = ref.lookup(Q, idx, 0.25, T)["sel2"]
        if prev is not None:
            assert not np.any(sel & ~prev)  # T' > T => sel(T') subset of sel(T)
        prev = sel


def test_prefill_averaging(ref):
    """one row = decode; duplicated rows = one row; 3-cluster direct evaluation."""
    rng = np.random.default_rng(6)
    idx = _single_level_index(ref, rng, 1, 3, 4)
    q = rng.standard_normal((1, 1, 1, 4))
    a = ref.lookup(q, idx, 1.0, 1e-3)
    b = ref.lookup(np.concatenate([q, q, q], axis=2), idx, 1.0, 1e-3)
    np.testing.assert_allclose(a["Sbar2"], b["Sbar2"], rtol=1e-14)
    # two rows concentrating on different clusters
    C = np.array([[10.0, 0, 0, 0], [0, 10.0, 0, 0], [0, 0, 0.0, 0]])
    idx.C2 = C[None]
    idx.N2 = np.array([[1, 1, 1]], np.int32)
    Q = np.array([[[[1.0, 0, 0, 0], [0, 1.0, 0, 0]]]])
    out = ref.lookup(Q, idx, 1.0, 0.3)
    e = np.exp(10.0)
    # S for row 1: (e, 1, 1)/(e+2); row 2: (1, e, 1)/(e+2); mean -> ((e+1)/2, (e+1)/2, 1)/(e+2)
    expect = np.array([(e + 1) / 2, (e + 1) / 2, 1.0]) / (e + 2)
    np.testing.assert_allclose(out["Sbar2"][0, 0], expect, rtol=1e-13)
    assert list(out["sel2"][0, 0]) == [True, True, False]
    # a threshold between the per-row max (~1) and the mean (~0.5) selects neither
    assert not ref.lookup(Q, idx, 1.0, 0.6)["sel2"].any()


def test_per_head_adaptivity(ref):
    """S:301 / P:229-233: one global T keeps more clusters of a flat head than of a skewed head."""
    import oracle

    d, c = 8, 16
    C = np.zeros((2, c, d))
    C[1, 0, 0] = 50.0  # head 1: one centroid aligned with q -> skewed
    N = np.ones((2, c), np.int32)
    idx = oracle.Index(levels=1, dtype=oracle.F32, H=2, L=c, d=d, c2=c, C2=C, N2=N,
                       key_off=None, perm=None)
    q = np.zeros((1, 2, 1, d))
    q[..., 0] = 1.0
    out = ref.lookup(q, idx, 1.0, 0.5 / c)
    assert out["sel2"][0, 0].sum() == c and out["sel2"][0, 1].sum() == 1
