"""GPU offline clustering (sqz_cluster_keys) vs the oracle (section 3.1, 3.3).

K-means has many correct results, so general data is checked by invariants; on a
well-separated mixture started from the same seeded subset the partitions must be
identical (K-means pins)."""
import numpy as np
import pytest

import oracle
from paper_2411_09688_b200 import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _build(fc, c2, init2, c1=0, init1=None, iters=50):
    from paper_2411_09688_b200 import sqz

    K = sqz.to_device(fc.K)
    V = sqz.to_device(fc.V)
    i2 = torch.from_numpy(init2).cuda()
    i1 = None if init1 is None else torch.from_numpy(init1).cuda()
    idx, Kp, Vp, its = sqz.cluster_keys(K, V, c2, i2, c1, i1, max_iters=iters)
    torch.cuda.synchronize()
    sqz.index_validate(idx)
    return idx, Kp, Vp, its


def _np(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


@pytest.mark.parametrize("levels", [1, 2])
@pytest.mark.parametrize("dtype", [synth.BF16, synth.F32])
def test_separated_mixture_identical_to_oracle(levels, dtype):
    H, L, d, G = 2, 3000, 128, 16
    c1 = 4 if levels == 2 else 0
    fc = synth.fixed_context(H, L, d, G, dtype=dtype, seed=41, sep=True, G1=c1)
    # one initial point per generating component, same subset for GPU and oracle
    init2 = np.stack([[np.nonzero(fc.labels[h] == g)[0][0] for g in range(G)] for h in range(H)])
    init1 = np.stack([np.arange(c1) for _ in range(H)]) if c1 else None
    g, Kp, Vp, _ = _build(fc, G, init2.astype(np.int64), c1,
                          None if init1 is None else init1.astype(np.int64))
    r = oracle.build_index(fc.K, G, init2, c1, init1)
    assert np.array_equal(_np(g.N2), r.N2)
    assert np.array_equal(_np(g.key_off), r.key_off)
    assert np.array_equal(_np(g.perm), r.perm)
    assert np.array_equal(_np(g.C2), oracle.encode(r.C2, dtype))
    if levels == 2:
        assert np.array_equal(_np(g.child_off), r.child_off)
        assert np.array_equal(_np(g.N1), r.N1)
        assert np.array_equal(_np(g.C1), oracle.encode(r.C1, dtype))
    assert np.array_equal(_np(Kp), oracle.permute_kv(fc.K, r))
    assert np.array_equal(_np(Vp), oracle.permute_kv(fc.V, r))


@pytest.mark.parametrize("levels", [1, 2])
def test_generic_data_invariants_and_determinism(levels):
    H, L, d = 3, 5000, 128
    c2, c1 = 250, (50 if levels == 2 else 0)
    fc = synth.fixed_context(H, L, d, c2, dtype=synth.BF16, seed=42, G1=c1)
    init2 = synth.kmeans_init(H, L, c2, seed=43)
    init1 = synth.kmeans_init(H, c2, c1, seed=44) if c1 else None
    g, Kp, Vp, its = _build(fc, c2, init2, c1, init1, iters=20)
    g2, _, _, _ = _build(fc, c2, init2, c1, init1, iters=20)
    for f in ("C2", "N2", "key_off", "perm"):
        assert torch.equal(getattr(g, f), getattr(g2, f)), f  # bit-reproducible
    K = oracle.to_f64(fc.K)
    perm, ko, N2, C2 = _np(g.perm), _np(g.key_off), _np(g.N2), oracle.to_f64(_np(g.C2))
    for h in range(H):
        assert N2[h].min() >= 1 and N2[h].sum() == L
        for i in range(0, c2, 7):
            mem = perm[h, ko[h, i]:ko[h, i + 1]]
            assert np.all(np.diff(mem) > 0)
            mean = oracle.round_to(K[h][mem].mean(0), synth.BF16)
            # raw-mean centroid (R2), rounded once; allow 1 bf16 ulp for the tie cases
            assert np.all(np.abs(C2[h, i] - mean) <= np.abs(mean) * 2 ** -7 + 1e-30)
    assert np.array_equal(_np(Kp), np.stack([fc.K[h][perm[h]] for h in range(H)]))
    if levels == 2:
        co, N1 = _np(g.child_off), _np(g.N1)
        for h in range(H):
            for p in range(c1):
                assert N1[h, p] == N2[h, co[h, p]:co[h, p + 1]].sum()


def _repair_data(dtype, seed):
    """Keys with a forced empty cluster: 6 tight groups on orthogonal directions,
    init points 0 and 1 identical (so cluster 1 ties with cluster 0 everywhere and
    starts empty), plus two outliers at clearly different distances from their
    nearest centroid (squared distances ~0.5 and ~0.25 in the normalised space)."""
    rng = np.random.default_rng(seed)
    d, per = 64, 30
    X = []
    for g in range(6):
        e = np.zeros(d, np.float32)
        e[g] = 4.0
        X.append(e + 0.01 * rng.standard_normal((per, d)).astype(np.float32))
    X = np.concatenate(X)
    X[1] = X[0]
    o1 = np.zeros(d, np.float32)
    o1[0], o1[7] = 0.75, 0.66   # 1 - cos ~ 0.25 from group 0's direction -> dist^2 ~ 0.5
    o2 = np.zeros(d, np.float32)
    o2[3], o2[8] = 0.88, 0.47   # dist^2 ~ 0.24 from group 3
    X = np.concatenate([X, 4 * o1[None], 4 * o2[None]])
    stored = synth.to_storage(X, dtype)
    init = np.array([0, 1, per, 2 * per, 3 * per, 4 * per, 5 * per], np.int64)
    return stored, init


@pytest.mark.parametrize("dtype", [synth.F32, synth.BF16])
@pytest.mark.parametrize("iters", [1, 50])
def test_empty_cluster_repair_matches_oracle(dtype, iters):
    """S:191 on the GPU (k_repair): the empty cluster takes the farthest point,
    exactly as the oracle's repair does; after one Lloyd iteration the repaired
    cluster holds only that outlier, and the converged tables are identical."""
    stored, init = _repair_data(dtype, 7)
    L = stored.shape[0]
    K = np.stack([stored, stored[::-1].copy()])  # head 1: same points, reversed order
    inits = np.stack([init, L - 1 - init])
    V = synth.to_storage(np.random.default_rng(8).standard_normal(K.shape).astype(np.float32), dtype)
    from types import SimpleNamespace
    fc = SimpleNamespace(K=K, V=V)
    g, Kp, Vp, _ = _build(fc, 7, inits, iters=iters)
    r = oracle.build_index(K, 7, inits, max_iters=iters)
    assert np.array_equal(_np(g.N2), r.N2)
    assert np.array_equal(_np(g.key_off), r.key_off)
    assert np.array_equal(_np(g.perm), r.perm)
    assert np.array_equal(_np(g.C2), oracle.encode(r.C2, dtype))
    if iters == 1:
        # head 0: cluster 1 (the empty duplicate) took the farthest outlier, point L - 2
        assert r.N2[0, 1] == 1 and r.perm[0, r.key_off[0, 1]] == L - 2


def _assign_of(g, H, L):
    """Cluster id of every ORIGINAL key, from the cluster-major tables."""
    perm, ko = _np(g.perm), _np(g.key_off)
    a = np.zeros((H, L), np.int64)
    for h in range(H):
        a[h, perm[h]] = np.repeat(np.arange(ko.shape[1] - 1), np.diff(ko[h]))
    return a


def _build_mode(fc, c2, init2, iters, mode, c1=0, init1=None):
    from paper_2411_09688_b200 import sqz

    K, V = sqz.to_device(fc.K), sqz.to_device(fc.V)
    idx, Kp, Vp, its = sqz.cluster_keys(K, V, c2, torch.from_numpy(init2).cuda(), c1,
                                        None if init1 is None else torch.from_numpy(init1).cuda(),
                                        max_iters=iters, assign_mode=mode)
    torch.cuda.synchronize()
    sqz.index_validate(idx)
    return idx, Kp, Vp


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_tensor_core_assignment_separated_identical_to_oracle(levels):
    """NEXT-3: the tcgen05 split-bf16 assignment reproduces the oracle's partitions
    and tables bit for bit on the separated mixture (same shared init)."""
    from paper_2411_09688_b200 import sqz

    H, L, d, G = 2, 3000, 128, 16
    c1 = 4 if levels >= 2 else 0
    c0 = 2 if levels == 3 else 0
    fc = synth.fixed_context(H, L, d, G, dtype=synth.BF16, seed=41, sep=True, G1=c1)
    init2 = np.stack([[np.nonzero(fc.labels[h] == g)[0][0] for g in range(G)] for h in range(H)])
    init1 = np.stack([np.arange(c1) for _ in range(H)]).astype(np.int64) if c1 else None
    init0 = np.stack([np.arange(c0) for _ in range(H)]).astype(np.int64) if c0 else None
    K, V = sqz.to_device(fc.K), sqz.to_device(fc.V)
    g, Kp, Vp, _ = sqz.cluster_keys(K, V, G, torch.from_numpy(init2.astype(np.int64)).cuda(), c1,
                                    None if init1 is None else torch.from_numpy(init1).cuda(),
                                    max_iters=50, assign_mode=sqz.KMEANS_TENSOR, c0=c0,
                                    init0=None if init0 is None else torch.from_numpy(init0).cuda())
    torch.cuda.synchronize()
    sqz.index_validate(g)
    r = oracle.build_index(fc.K, G, init2, c1, init1, c0=c0, init0=init0)
    assert np.array_equal(_np(g.perm), r.perm) and np.array_equal(_np(g.key_off), r.key_off)
    assert np.array_equal(_np(g.C2), oracle.encode(r.C2, synth.BF16))
    if levels >= 2:
        assert np.array_equal(_np(g.child_off), r.child_off)
        assert np.array_equal(_np(g.C1), oracle.encode(r.C1, synth.BF16))
    if levels == 3:
        assert np.array_equal(_np(g.child_off0), r.child_off0)
        assert np.array_equal(_np(g.C0), oracle.encode(r.C0, synth.BF16))


@pytest.mark.parametrize("d", [64, 128])
def test_tensor_core_assignment_matches_exact_on_generic_data(d):
    """One Lloyd assignment from the same init, tensor-core vs exact fp32 path:
    every key gets a centroid whose fp64 distance is within 1e-5 (relative) of the
    minimum over all centroids, and at most a handful of near-tie keys differ."""
    from paper_2411_09688_b200 import sqz

    H, L, c2 = 2, 9000, 300
    fc = synth.fixed_context(H, L, d, c2, dtype=synth.BF16, seed=46)
    init2 = synth.kmeans_init(H, L, c2, seed=47)
    gt, _, _ = _build_mode(fc, c2, init2, 1, sqz.KMEANS_TENSOR)
    ge, _, _ = _build_mode(fc, c2, init2, 1, sqz.KMEANS_EXACT)
    at, ae = _assign_of(gt, H, L), _assign_of(ge, H, L)
    X = oracle.to_f64(fc.K)
    X = X / np.linalg.norm(X, axis=2, keepdims=True)
    diff = 0
    for h in range(H):
        mu = X[h][init2[h]]  # the first assignment is against the initial points
        D2 = ((X[h][:, None, :] - mu[None]) ** 2).sum(-1)
        dmin = D2.min(1)
        got = D2[np.arange(L), at[h]]
        assert np.all(got <= dmin * (1 + 1e-5) + 1e-6)
        diff += int((at[h] != ae[h]).sum())
    assert diff <= 0.001 * H * L, diff


def test_tensor_core_generic_invariants():
    """Full runs in tensor-core mode keep every index invariant and are bit-reproducible."""
    from paper_2411_09688_b200 import sqz

    H, L, d, c2, c1 = 2, 6000, 128, 240, 40
    fc = synth.fixed_context(H, L, d, c2, dtype=synth.BF16, seed=48, G1=c1)
    init2 = synth.kmeans_init(H, L, c2, seed=49)
    init1 = synth.kmeans_init(H, c2, c1, seed=50)
    g, Kp, _ = _build_mode(fc, c2, init2, 15, sqz.KMEANS_TENSOR, c1, init1)
    g2, _, _ = _build_mode(fc, c2, init2, 15, sqz.KMEANS_TENSOR, c1, init1)
    for f in ("C2", "N2", "key_off", "perm", "C1", "N1", "child_off"):
        assert torch.equal(getattr(g, f), getattr(g2, f)), f
    perm, N2 = _np(g.perm), _np(g.N2)
    for h in range(H):
        assert N2[h].min() >= 1 and N2[h].sum() == L
    assert np.array_equal(_np(Kp), np.stack([fc.K[h][perm[h]] for h in range(H)]))


@pytest.mark.parametrize("dtype", [synth.BF16, synth.F32])
def test_three_level_index_identical_to_oracle(dtype):
    """Three levels: on the separated mixture from the shared inits the GPU
    build equals the oracle's build_index bit for bit (Level-0 tables, the Level-1
    renumbering, and the Level-2 / key order that follows from it)."""
    from paper_2411_09688_b200 import sqz

    H, L, d, G, c1, c0 = 2, 4000, 128, 32, 8, 3
    fc = synth.fixed_context(H, L, d, G, dtype=dtype, seed=51, sep=True, G1=c1)
    init2 = np.stack([[np.nonzero(fc.labels[h] == g)[0][0] for g in range(G)] for h in range(H)])
    init1 = np.stack([np.arange(c1) for _ in range(H)]).astype(np.int64)
    init0 = np.stack([np.arange(c0) for _ in range(H)]).astype(np.int64)
    g, Kp, Vp, its = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), G,
                                      torch.from_numpy(init2.astype(np.int64)).cuda(), c1,
                                      torch.from_numpy(init1).cuda(), max_iters=50, c0=c0,
                                      init0=torch.from_numpy(init0).cuda())
    torch.cuda.synchronize()
    sqz.index_validate(g)
    r = oracle.build_index(fc.K, G, init2, c1, init1, c0=c0, init0=init0)
    for f in ("N2", "key_off", "perm", "N1", "child_off", "N0", "child_off0"):
        assert np.array_equal(_np(getattr(g, f)), getattr(r, f)), f
    for f in ("C2", "C1", "C0"):
        assert np.array_equal(_np(getattr(g, f)), oracle.encode(getattr(r, f), dtype)), f
    assert np.array_equal(_np(Kp), oracle.permute_kv(fc.K, r))
    assert np.array_equal(_np(Vp), oracle.permute_kv(fc.V, r))


@pytest.mark.parametrize("levels,dt", [(1, synth.F32), (2, synth.BF16), (3, synth.BF16)])
def test_index_save_load_round_trip(levels, dt, tmp_path):
    """sqz_index_save / sqz_index_load: load(save(x)) == x bit for bit, the
    loaded index validates, and a lookup on it selects exactly what the original's
    does (the offline index is the persisted artefact)."""
    from paper_2411_09688_b200 import sqz

    H, L, d, c2 = 2, 1200, 64, 48
    c1 = 12 if levels >= 2 else 0
    c0 = 4 if levels == 3 else 0
    fc = synth.fixed_context(H, L, d, c2, dtype=dt, seed=61)
    K, V = sqz.to_device(fc.K), sqz.to_device(fc.V)
    i2 = torch.from_numpy(synth.kmeans_init(H, L, c2, seed=62)).cuda()
    i1 = torch.from_numpy(synth.kmeans_init(H, c2, c1, seed=63)).cuda() if c1 else None
    i0 = torch.from_numpy(synth.kmeans_init(H, c1, c0, seed=64)).cuda() if c0 else None
    idx, Kp, Vp, _ = sqz.cluster_keys(K, V, c2, i2, c1, i1, max_iters=20, c0=c0, init0=i0)
    path = str(tmp_path / "ctx.sqzidx")
    sqz.save_index(idx, path)
    got = sqz.load_index(path)
    assert got.levels == idx.levels == levels
    for f in ("C2", "N2", "key_off", "perm", "C1", "N1", "child_off", "C0", "N0", "child_off0"):
        a, b = getattr(idx, f), getattr(got, f)
        assert (a is None) == (b is None), f
        if a is not None:
            assert torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                               b.view(torch.int16) if b.dtype == torch.bfloat16 else b), f
    Q = sqz.to_device(synth.decode_queries(fc.mix, 3, seed=65, dtype=dt))
    T1 = 1e-3 if levels >= 2 else 0.0
    s1 = sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), 2e-4, T1, T0=1e-3 if levels == 3 else 0.0)
    s2 = sqz.centroid_lookup(got, Q, 1 / np.sqrt(d), 2e-4, T1, T0=1e-3 if levels == 3 else 0.0)
    torch.cuda.synchronize()
    assert torch.equal(s1.n_clusters, s2.n_clusters) and torch.equal(s1.n_keys, s2.n_keys)
    nc = s1.n_clusters.cpu()
    for b in range(nc.shape[0]):
        for h in range(H):
            n = int(nc[b, h])
            assert torch.equal(s1.clusters[b, h, :n], s2.clusters[b, h, :n])
    # a dst of another geometry is refused
    other = sqz.Index.empty(H, d, L, c2 + 1, c1, sqz.sqz_dtype(K), "cuda", c0=c0)
    with pytest.raises(sqz.SqzError) as e:
        sqz._check(sqz.lib().sqz_index_load(path.encode(), sqz.ctypes.byref(other.struct()), sqz._stream()))
    assert e.value.code == sqz.SQZ_ERR_FORMAT
