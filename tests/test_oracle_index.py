"""Pins for the oracle's offline K-means and index build (section 3.1 P:165-178,
section 3.3), plus the KV-budget arithmetic (Table 2)."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2411_09688_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def test_c1_gives_global_raw_mean():
    """c = 1 -> one cluster, centroid = mean of all (raw) items, N = n."""
    rng = np.random.default_rng(30)
    X = rng.standard_normal((200, 12)) * 3 + 1
    a, _, _, _ = oracle.kmeans(X, 1, [17])
    C, N = oracle.cluster_means(X, a, 1)
    assert N[0] == 200
    np.testing.assert_allclose(C[0], X.mean(0), rtol=1e-13)


def test_distinct_points_are_their_own_clusters():
    """c distinct points, c clusters -> identity partition, centroids = points."""
    rng = np.random.default_rng(31)
    X = rng.standard_normal((9, 5))
    a, mu, it, _ = oracle.kmeans(X, 9, rng.permutation(9))
    assert sorted(a.tolist()) == list(range(9))
    C, N = oracle.cluster_means(X, a, 9)
    np.testing.assert_array_equal(N, 1)
    np.testing.assert_allclose(C[a], X, rtol=1e-15)


def _purity(assign, labels):
    tot = 0
    for c in np.unique(assign):
        tot += np.bincount(labels[assign == c]).max()
    return tot / len(assign)


def test_separated_mixture_recovered():
    """well-separated mixture (Delta/sigma >= 10), c = G -> >= 99% of items recovered.
    Uses the harness generator's SEP variant (DESIGN.md input recipe)."""
    fc = synth.fixed_context(H=1, L=2000, d=32, G=8, dtype=synth.F32, seed=7, sep=True)
    # init: one point of each component, so Lloyd starts in the right basin
    init = [int(np.nonzero(fc.labels[0] == g)[0][0]) for g in range(8)]
    a, _, _, _ = oracle.kmeans(oracle.to_f64(fc.K[0]), 8, init)
    assert _purity(a, fc.labels[0]) >= 0.99


def test_objective_monotone_and_deterministic():
    """S:183 objective non-increasing per iteration; S:180 same seed -> identical result."""
    fc = synth.fixed_context(H=1, L=1500, d=16, G=20, dtype=synth.F32, seed=8)
    init = synth.kmeans_init(1, 1500, 20, seed=9)[0]
    X = oracle.to_f64(fc.K[0])
    a1, mu1, it1, obj = oracle.kmeans(X, 20, init, max_iters=50, tol=0.0)
    assert np.all(np.diff(obj) <= 1e-9 * obj[0])
    a2, mu2, it2, _ = oracle.kmeans(X, 20, init, max_iters=50, tol=0.0)
    assert np.array_equal(a1, a2) and np.array_equal(mu1, mu2) and it1 == it2


def test_assignment_is_nearest_centroid_at_convergence():
    """Lloyd fixed point: with the returned normalised-space centroids every point's
    assigned centroid is the nearest one (distances via numpy, ties -> lowest id)."""
    fc = synth.fixed_context(H=1, L=800, d=16, G=12, dtype=synth.F32, seed=10)
    X = oracle.to_f64(fc.K[0])
    a, mu, it, _ = oracle.kmeans(X, 12, synth.kmeans_init(1, 800, 12, seed=11)[0], 200, 0.0)
    Xh = X / np.linalg.norm(X, axis=1, keepdims=True)
    D = ((Xh[:, None, :] - mu[None]) ** 2).sum(-1)
    assert np.array_equal(np.argmin(D, axis=1), a)


def test_empty_cluster_repair():
    """an initial centroid that attracts no point takes the farthest point."""
    X = np.array([[1.0, 0.0]] * 5 + [[0.0, 1.0]] * 5 + [[0.6, 0.8]])
    # init 0 and 1 are the same point -> cluster 1 ties to 0 (lowest id) and is empty
    a, _, _, _ = oracle.kmeans(X, 3, [0, 1, 5], max_iters=5)
    assert len(np.unique(a)) == 3


def test_empty_cluster_repair_exact_move():
    """S:191, the exact repair move after ONE Lloyd iteration.  Points 0-4 sit on
    centroid 0 (distance 0) and tie with the empty duplicate 1 (ties -> lowest id),
    points 5-9 sit on centroid 2; point 10 (0.6, 0.8) goes to centroid 2 at squared
    distance 0.4.  Cluster 1 is empty, so it takes the point FARTHEST from its own
    centroid among clusters with > 1 member: point 10.  A "nearest point" or
    "lowest index" repair would move point 0 instead."""
    X = np.array([[1.0, 0.0]] * 5 + [[0.0, 1.0]] * 5 + [[0.6, 0.8]])
    a, mu, it, _ = oracle.kmeans(X, 3, [0, 1, 5], max_iters=1)
    assert it == 1
    assert a.tolist() == [0] * 5 + [2] * 5 + [1]
    # the repaired cluster's normalised-space centroid is its single member
    np.testing.assert_allclose(mu[1], [0.6, 0.8], rtol=0, atol=1e-15)
    # two empty clusters are repaired in increasing id, each taking the farthest
    # remaining point (the second one: point 11 at squared distance 0.092 from (0, 1))
    X2 = np.concatenate([X, [[0.3, 0.95393920141694566]]])
    a2, _, _, _ = oracle.kmeans(X2, 4, [0, 1, 2, 5], max_iters=1)
    assert a2[10] == 1 and a2[11] == 2 and a2[:5].tolist() == [0] * 5


@pytest.mark.parametrize("levels", [1, 2])
def test_build_index_invariants(levels):
    H, L, d = 2, 600, 16
    c1, c2 = (6, 30) if levels == 2 else (0, 30)
    fc = synth.fixed_context(H=H, L=L, d=d, G=30, G1=6 if levels == 2 else 0,
                             dtype=synth.BF16, seed=12)
    init2 = synth.kmeans_init(H, L, c2, seed=13)
    init1 = synth.kmeans_init(H, c2, c1, seed=14) if levels == 2 else None
    idx = oracle.build_index(fc.K, c2, init2, c1, init1)
    K = oracle.to_f64(fc.K)
    for h in range(H):
        assert idx.N2[h].sum() == L                                    # sum N = L
        assert sorted(idx.perm[h].tolist()) == list(range(L))        # perm is a permutation
        assert np.array_equal(np.diff(idx.key_off[h]), idx.N2[h])
        for i in range(c2):
            members = idx.perm[h][idx.key_off[h, i]:idx.key_off[h, i + 1]]
            assert np.all(idx.assign2[h][members] == i)
            assert np.all(np.diff(members) > 0)                        # stable in original index
            mean = K[h][members].mean(0)                               # raw mean (R2), numpy
            bf = np.array([oracle.round_to(m, oracle.BF16) for m in [mean]])[0]
            np.testing.assert_array_equal(idx.C2[h, i], bf)
        if levels == 2:
            co = idx.child_off[h]
            assert co[0] == 0 and co[-1] == c2 and np.all(np.diff(co) >= 1)
            for p in range(c1):
                ch = np.arange(co[p], co[p + 1])
                assert idx.N1[h, p] == idx.N2[h][ch].sum()               # descendant keys (R4)
                np.testing.assert_array_equal(
                    idx.C1[h, p], oracle.round_to(idx.C2[h][ch].mean(0), oracle.BF16))
    # centroids are bf16-representable
    assert np.array_equal(oracle.to_f64(oracle.encode(idx.C2, oracle.BF16)), idx.C2)


def test_round_bf16_matches_torch():
    import torch

    rng = np.random.default_rng(15)
    x = rng.standard_normal(10000) * 10.0 ** rng.integers(-3, 4, size=10000)
    ours = oracle.round_to(x, oracle.BF16)
    # torch rounds fp32 -> bf16 RNE; feed values that are exact in fp32 to avoid double rounding
    xf = x.astype(np.float32).astype(np.float64)
    t = torch.tensor(xf, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(oracle.round_to(xf, oracle.BF16), t)
    assert np.all(np.abs(ours - x) <= np.abs(x) * 2.0 ** -8)


@pytest.mark.parametrize("ex", GOLD["budget"], ids=lambda e: e["cite"][:20])
def test_budget_table2(ex):
    """budget = (1 - sparsity) + centroid_frac / 2, exact."""
    L = 100000
    k = round((1 - ex["sparsity"]) * L)
    c = round(ex["centroid_frac"] * L)
    assert oracle.budget(k, L, [c]) == pytest.approx(ex["budget"], abs=1e-12)


def test_budget_dense_and_hierarchical():
    assert oracle.budget(1000, 1000) == 1.0
    # H-Squeeze-90: 1% Level 1 + half of the 5% Level 2 scanned + 10% keys = 0.1175,
    # within the profiled 0.112-0.122 of P:438/451/464 (consistency only).
    L = 100000
    b = oracle.budget(0.1 * L, L, [0.01 * L, 0.5 * 0.05 * L])
    vals = GOLD["hier_budget_profiled"]["values"]
    assert min(vals) - 0.01 <= b <= max(vals) + 0.01
    ex = GOLD["centroid_fractions"]["examples"][0]
    assert synth.centroid_counts(ex["L"]) == (ex["c1"], ex["c2"])
