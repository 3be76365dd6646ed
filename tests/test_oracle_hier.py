"""Pins for the oracle's hierarchical lookup (section 3.3, Eq. 2-3)."""
import numpy as np
import pytest

import oracle


def _hier_index(rng, H, c1, per, d, nmax=20):
    c2 = c1 * per
    C2 = rng.standard_normal((H, c2, d))
    N2 = rng.integers(1, nmax, size=(H, c2)).astype(np.int32)
    child_off = np.tile(np.arange(0, c2 + 1, per, dtype=np.int32), (H, 1))
    C1 = np.stack([C2[:, p * per:(p + 1) * per].mean(axis=1) for p in range(c1)], axis=1)
    N1 = N2.reshape(H, c1, per).sum(axis=2).astype(np.int32)
    key_off = np.concatenate([np.zeros((H, 1), np.int32), np.cumsum(N2, 1, dtype=np.int32)], 1)
    return oracle.Index(levels=2, dtype=oracle.F32, H=H, L=int(N2.sum(1).max()), d=d, c2=c2,
                        C2=C2, N2=N2, key_off=key_off, perm=None, c1=c1, C1=C1, N1=N1,
                        child_off=child_off)


def test_T1_zero_reduces_to_single_level(ref):
    """S:255 / S:300 / S:482: with T1 = 0 the candidate set is every Level-2 cluster and the
    restricted denominator equals the full one, so the selection equals single-level."""
    rng = np.random.default_rng(10)
    for trial in range(100):
        c1, per, d = int(rng.integers(1, 8)), int(rng.integers(1, 6)), int(rng.choice([4, 16, 64]))
        idx = _hier_index(rng, 2, c1, per, d)
        Q = rng.standard_normal((2, 2, int(rng.integers(1, 4)), d)) * 2
        T = float(rng.uniform(1e-4, 5e-2))
        h = ref.lookup(Q, idx, 1.0 / np.sqrt(d), T, T1=0.0)
        single = oracle.Index(levels=1, dtype=idx.dtype, H=idx.H, L=idx.L, d=d, c2=idx.c2,
                              C2=idx.C2, N2=idx.N2, key_off=idx.key_off, perm=None)
        s = ref.lookup(Q, single, 1.0 / np.sqrt(d), T)
        np.testing.assert_allclose(h["Sbar2"], s["Sbar2"], rtol=1e-12)
        assert np.array_equal(h["sel2"], s["sel2"])
        np.testing.assert_allclose(h["lse"], s["lse"], rtol=1e-13)


def test_selected_children_have_surviving_parents(ref):
    """North star: hierarchical masks are subsets of their Level-1 parents."""
    rng = np.random.default_rng(11)
    idx = _hier_index(rng, 4, 12, 5, 32)
    Q = rng.standard_normal((3, 4, 1, 32)) * 3
    out = ref.lookup(Q, idx, 1 / np.sqrt(32), 1e-3, T1=2e-3)
    parent = np.repeat(np.arange(12), 5)
    for b in range(3):
        for h in range(4):
            sel = np.nonzero(out["sel2"][b, h])[0]
            assert np.all(out["surv1"][b, h][parent[sel]])
            # unscanned children carry NaN scores
            assert np.all(np.isnan(out["Sbar2"][b, h][~out["surv1"][b, h][parent]]))


def test_restricted_denominator_sums_to_one_over_candidates(ref):
    """Eq. 3: sum over the surviving children of N_l S_l = 1."""
    rng = np.random.default_rng(12)
    idx = _hier_index(rng, 2, 10, 4, 16)
    Q = rng.standard_normal((2, 2, 1, 16)) * 2
    out = ref.lookup(Q, idx, 0.25, 1e-3, T1=5e-3)
    for b in range(2):
        for h in range(2):
            S = out["Sbar2"][b, h]
            m = ~np.isnan(S)
            if m.any():
                assert np.sum(idx.N2[h][m] * S[m]) == pytest.approx(1.0, rel=1e-12)


def test_all_level1_pruned_gives_empty(ref):
    """all coarse scores below T1 -> empty selection, no Level-2 row scanned."""
    rng = np.random.default_rng(13)
    idx = _hier_index(rng, 1, 6, 3, 8)
    Q = rng.standard_normal((1, 1, 1, 8))
    out = ref.lookup(Q, idx, 1.0, 1e-3, T1=1.0)  # S^(1) <= 1/N^(1) < 1
    assert not out["surv1"].any() and not out["sel2"].any()
    assert np.all(np.isnan(out["Sbar2"])) and np.all(np.isneginf(out["lse"]))


def test_forced_level1_set(ref):
    """Conditional parity: forcing the Level-1 survivors reproduces the natural run when the
    forced set equals the natural set, and restricts candidates otherwise."""
    rng = np.random.default_rng(14)
    idx = _hier_index(rng, 2, 8, 4, 16)
    Q = rng.standard_normal((1, 2, 1, 16)) * 2
    nat = ref.lookup(Q, idx, 0.25, 1e-3, T1=1e-2)
    forced = ref.lookup(Q, idx, 0.25, 1e-3, T1=1e-2, forced_l1=nat["surv1"])
    assert np.array_equal(nat["sel2"], forced["sel2"])
    f = np.zeros_like(nat["surv1"])
    f[..., 0] = True
    one = ref.lookup(Q, idx, 0.25, 0.0, T1=1e-2, forced_l1=f)
    assert np.array_equal(one["sel2"][0, 0], np.arange(idx.c2) < 4)


def test_brute_force_enumeration_16_keys(ref):
    """16 keys, 4 Level-2 / 2 Level-1 clusters.  Enumerate every T1 between distinct
    Level-1 scores: candidates are exactly the children of surviving parents, and a pruned
    parent removes only children with single-level S_i no larger than that parent's S^(1)
    times its descendant count (the parent score is the N-weighted mean of its children's
    exp(s) mass only when its centroid is the mean child -- here checked directly)."""
    d = 2
    C2 = np.array([[[3.0, 0.0], [2.5, 0.5], [-1.0, 0.0], [-1.5, -0.5]]])
    N2 = np.array([[4, 4, 4, 4]], np.int32)
    C1 = np.stack([C2[:, :2].mean(1), C2[:, 2:].mean(1)], axis=1)
    N1 = np.array([[8, 8]], np.int32)
    idx = oracle.Index(levels=2, dtype=oracle.F32, H=1, L=16, d=d, c2=4, C2=C2, N2=N2,
                       key_off=np.array([[0, 4, 8, 12, 16]], np.int32), perm=None, c1=2, C1=C1,
                       N1=N1, child_off=np.array([[0, 2, 4]], np.int32))
    q = np.array([[[[1.0, 0.0]]]])
    _, S1, _ = ref.scores(q[0, 0, 0], C1[0], N1[0], 1.0)
    assert S1[0] > S1[1]
    for T1, expect in [(0.0, [1, 1]), ((S1[0] + S1[1]) / 2, [1, 0]), (S1[0] * 1.01, [0, 0])]:
        out = ref.lookup(q, idx, 1.0, 0.0, T1=T1)
        assert list(out["surv1"][0, 0].astype(int)) == expect
        cand = np.repeat(np.array(expect, bool), 2)
        assert np.array_equal(out["sel2"][0, 0], cand)  # T = 0: every candidate selected


# ---- three levels ("extended to multiple levels"; NEXT-2) ----

def _three_level(rng, H, c0, per1, per2, d, nmax=20):
    idx = _hier_index(rng, H, c0 * per1, per2, d, nmax)
    c1 = idx.c1
    idx.levels = 3
    idx.c0 = c0
    idx.child_off0 = np.tile(np.arange(0, c1 + 1, per1, dtype=np.int32), (H, 1))
    idx.C0 = np.stack([idx.C1[:, g * per1:(g + 1) * per1].mean(axis=1) for g in range(c0)], axis=1)
    idx.N0 = idx.N1.reshape(H, c0, per1).sum(axis=2).astype(np.int32)
    return idx


def _two_level_of(idx):
    return oracle.Index(levels=2, dtype=idx.dtype, H=idx.H, L=idx.L, d=idx.d, c2=idx.c2,
                        C2=idx.C2, N2=idx.N2, key_off=idx.key_off, perm=None, c1=idx.c1,
                        C1=idx.C1, N1=idx.N1, child_off=idx.child_off)


def test_three_levels_T0_zero_reduces_to_two_levels(ref):
    """T0 = 0 keeps every Level-0 cluster, so the Level-1 candidates are all Level-1 rows
    and the restricted denominator is the full Eq. 2 one: the three-level lookup equals the
    (pinned) two-level lookup; T0 = T1 = 0 equals single level."""
    rng = np.random.default_rng(20)
    for trial in range(60):
        c0, per1, per2 = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 5))
        d = int(rng.choice([4, 16, 64]))
        idx = _three_level(rng, 2, c0, per1, per2, d)
        Q = rng.standard_normal((2, 2, int(rng.integers(1, 4)), d)) * 2
        T, T1 = float(rng.uniform(1e-4, 5e-2)), float(rng.uniform(0, 5e-2))
        three = ref.lookup(Q, idx, 1.0 / np.sqrt(d), T, T1=T1, T0=0.0)
        two = ref.lookup(Q, _two_level_of(idx), 1.0 / np.sqrt(d), T, T1=T1)
        assert np.array_equal(three["sel2"], two["sel2"])
        assert np.array_equal(three["surv1"], two["surv1"])
        np.testing.assert_allclose(three["Sbar1"], two["Sbar1"], rtol=1e-12)
        np.testing.assert_allclose(three["Sbar2"], two["Sbar2"], rtol=1e-12)
        np.testing.assert_allclose(three["lse"], two["lse"], rtol=1e-13)
        assert three["surv0"].all()
        single = oracle.Index(levels=1, dtype=idx.dtype, H=idx.H, L=idx.L, d=d, c2=idx.c2,
                              C2=idx.C2, N2=idx.N2, key_off=idx.key_off, perm=None)
        a = ref.lookup(Q, idx, 1.0 / np.sqrt(d), T, T1=0.0, T0=0.0)
        s = ref.lookup(Q, single, 1.0 / np.sqrt(d), T)
        assert np.array_equal(a["sel2"], s["sel2"])


def test_three_levels_ancestry_and_restricted_sums(ref):
    """Every selected Level-2 cluster has a surviving parent and grandparent; each level's
    restricted Eq. 3 scores satisfy sum N S = 1 over its candidates; unscanned rows are NaN."""
    rng = np.random.default_rng(21)
    idx = _three_level(rng, 3, 4, 3, 5, 32)
    Q = rng.standard_normal((2, 3, 1, 32)) * 3
    out = ref.lookup(Q, idx, 1 / np.sqrt(32), 1e-3, T1=3e-3, T0=2e-3)
    p2 = np.repeat(np.arange(idx.c1), 5)
    p1 = np.repeat(np.arange(idx.c0), 3)
    for b in range(2):
        for h in range(3):
            sel = np.nonzero(out["sel2"][b, h])[0]
            assert np.all(out["surv1"][b, h][p2[sel]]) and np.all(out["surv0"][b, h][p1[p2[sel]]])
            s1 = np.nonzero(out["surv1"][b, h])[0]
            assert np.all(out["surv0"][b, h][p1[s1]])
            for S, N in ((out["Sbar1"][b, h], idx.N1[h]), (out["Sbar2"][b, h], idx.N2[h])):
                m = ~np.isnan(S)
                if m.any():
                    assert np.sum(N[m] * S[m]) == pytest.approx(1.0, rel=1e-12)
            assert np.all(np.isnan(out["Sbar1"][b, h][~out["surv0"][b, h][p1]]))


def test_three_levels_all_pruned_and_forced(ref):
    """All Level-0 clusters pruned -> empty selection; forcing the natural survivor sets
    reproduces the natural run."""
    rng = np.random.default_rng(22)
    idx = _three_level(rng, 1, 3, 2, 3, 8)
    Q = rng.standard_normal((1, 1, 1, 8))
    out = ref.lookup(Q, idx, 1.0, 1e-3, T1=1e-3, T0=1.0)  # S^(0) <= 1/N^(0) < 1
    assert not out["surv0"].any() and not out["surv1"].any() and not out["sel2"].any()
    assert np.all(np.isneginf(out["lse"]))
    idx = _three_level(rng, 2, 4, 3, 3, 16)
    Q = rng.standard_normal((1, 2, 2, 16)) * 2
    nat = ref.lookup(Q, idx, 0.25, 1e-3, T1=5e-3, T0=1e-2)
    f = ref.lookup(Q, idx, 0.25, 1e-3, T1=5e-3, T0=1e-2, forced_l0=nat["surv0"], forced_l1=nat["surv1"])
    assert np.array_equal(nat["sel2"], f["sel2"])


def test_three_level_index_build_invariants():
    """build_index with c0 > 0: Level-1 ids grouped by their Level-0 parent, N0 = descendant
    keys, C0 = the (rounded) mean of its Level-1 rows, and the Level-2 / key order still
    grouped by parent; c0 = 1 puts every Level-1 cluster under one parent."""
    from paper_2411_09688_b200 import synth

    fc = synth.fixed_context(2, 3000, 32, 90, dtype=synth.F32, seed=23, G1=18)
    i2 = synth.kmeans_init(2, 3000, 90, seed=24)
    i1 = synth.kmeans_init(2, 90, 18, seed=25)
    for c0 in (1, 5):
        i0 = synth.kmeans_init(2, 18, c0, seed=26)
        idx = oracle.build_index(fc.K, 90, i2, 18, i1, c0=c0, init0=i0)
        assert idx.levels == 3
        for h in range(2):
            co0, co = idx.child_off0[h], idx.child_off[h]
            assert co0[0] == 0 and co0[-1] == 18 and np.all(np.diff(co0) >= 1)
            for g in range(c0):
                kids = np.arange(co0[g], co0[g + 1])
                assert idx.N0[h, g] == idx.N1[h, kids].sum()
                np.testing.assert_allclose(idx.C0[h, g], oracle.round_to(idx.C1[h, kids].mean(0), oracle.F32),
                                           rtol=1e-6, atol=1e-7)
            for p in range(18):
                assert idx.N1[h, p] == idx.N2[h, co[p]:co[p + 1]].sum()
            assert idx.N0[h].sum() == 3000 and np.array_equal(np.sort(idx.perm[h]), np.arange(3000))
        if c0 == 1:
            assert np.array_equal(idx.child_off0, np.tile([0, 18], (2, 1)))
