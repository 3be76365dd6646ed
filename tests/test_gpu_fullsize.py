"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration, on
sampled outputs the oracle computes one by one.

cfg2 (32 heads x 32K keys, c = 1024, decode, n_u = 1024), cfg3 (the same context,
1024-row causal prefill + 1024 user keys) and cfg4 (128K keys, two-level c1 = 1311 /
c2 = 6554, B = 8 decode) are built, indexed and calibrated the way bench.py does it;
the oracle re-runs the lookup for two sampled heads (head 0 and the head with the
most selected keys) on the GPU-built tables and the attention on the GPU's
selected key set for those heads (64 sampled query rows, first and last
included, for the prefill).  Rules as in test_gpu_parity.py (band 1e-5, bf16 O
max-abs 2e-2 / rel-L2 5e-3, LSE 1e-3)."""
import numpy as np
import pytest

import oracle
from paper_2411_09688_b200 import calib, synth

from helpers import assert_selection_parity, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_09688_b200 import sqz

    sqz.device_check()


def _sqz():
    from paper_2411_09688_b200 import sqz

    return sqz


def _bits(t):  # bf16 tensor -> storage bits (uint16) on the host
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _oracle_index(g, heads):
    """oracle.Index of the sampled heads from the GPU-built tables."""
    hv = lambda t: t[heads].cpu().numpy()
    idx = oracle.Index(levels=g.levels, dtype=oracle.BF16, H=len(heads), L=g.L, d=g.d, c2=g.c2,
                       C2=oracle.to_f64(_bits(g.C2[heads])), N2=hv(g.N2), key_off=hv(g.key_off),
                       perm=hv(g.perm))
    if g.levels == 2:
        idx.c1 = g.c1
        idx.C1 = oracle.to_f64(_bits(g.C1[heads]))
        idx.N1 = hv(g.N1)
        idx.child_off = hv(g.child_off)
    return idx


def _gpu_sel_sets(sel, heads, c2):
    cl, n = sel.clusters.cpu().numpy(), sel.n_clusters.cpu().numpy()
    B = cl.shape[0]
    out = np.zeros((B, len(heads), c2), bool)
    for b in range(B):
        for j, h in enumerate(heads):
            out[b, j, cl[b, h, :n[b, h]]] = True
    return out


def _key_mask(sel, idx_sub, heads):
    ki, nk = sel.key_idx.cpu().numpy(), sel.n_keys.cpu().numpy()
    B = ki.shape[0]
    m = np.zeros((B, len(heads), idx_sub.L), bool)
    for b in range(B):
        for j, h in enumerate(heads):
            m[b, j, idx_sub.perm[j][ki[b, h, :nk[b, h]]]] = True
    return m


def _run(K, V, Q, Ku, Vu, c2, c1, init2, init1, prefill, retention, Qc, step=False):
    """GPU index + calibration + lookup + attention as bench.py runs them (step: one
    sqz_decode_step call, the path bench.py times for cfg2); returns the pieces the
    oracle needs."""
    sqz = _sqz()
    H, L, d = K.shape
    scale = 1.0 / np.sqrt(d)
    idx, Kp, Vp, _ = sqz.cluster_keys(K, V, c2, init2, c1, init1, max_iters=10)
    T1 = 0.0
    Bc = Qc.shape[0]
    if c1:
        s = sqz.centroid_lookup(idx, Qc, scale, 0.0, 0.0, debug=True)
        T1 = calib.distributed_threshold(s.dbg_S1, idx.N1[None], 0.5, float(Bc * idx.N1.sum()))
        s = sqz.centroid_lookup(idx, Qc, scale, 0.0, T1, debug=True)
        T = calib.distributed_threshold(s.dbg_S, idx.N2[None], retention, float(Bc * H * L))
    else:
        s = sqz.centroid_lookup(idx, Qc, scale, 0.0, T1, debug=True)
        T = calib.weighted_threshold(s.dbg_S.cpu().numpy(), idx.N2.cpu().numpy()[None], retention,
                                     total_weight=Bc * H * L)
    B, _, n_q, _ = Q.shape
    sel = sqz.Selection.empty(idx, B, n_q, True)
    if step:
        sel, O, LSE = sqz.decode_step(idx, Q, Kp, Vp, Ku, Vu, scale, T, T1, sel=sel)
    else:
        sqz.centroid_lookup(idx, Q, scale, T, T1, sel=sel)
        O, LSE = sqz.sparse_attention(Q, Kp, Vp, idx, sel, Ku, Vu, scale, causal=prefill)
    torch.cuda.synchronize()
    nk = sel.n_keys.cpu().numpy()
    heads = [0, int(np.argmax(nk.sum(0)))]
    if heads[1] == 0:
        heads[1] = H - 1
    return idx, sel, O, LSE, T, T1, scale, heads


def _check(idx, sel, O, LSE, T, T1, scale, heads, Q, K, V, Ku, Vu, prefill, rows=None):
    sub = _oracle_index(idx, heads)
    Q64 = oracle.to_f64(_bits(Q[:, heads]))
    forced = None
    if idx.levels == 2:
        g1 = sel.l1_surv[:, heads].cpu().numpy().astype(bool)
        ref1 = oracle.lookup(Q64, sub, scale, T, T1)
        assert_selection_parity(g1, ref1["surv1"], ref1["Sbar1"], T1, what="full-size level-1")
        forced = g1
    ref = oracle.lookup(Q64, sub, scale, T, T1, forced_l1=forced)
    g = _gpu_sel_sets(sel, heads, idx.c2)
    assert_selection_parity(g, ref["sel2"], ref["Sbar2"], T, what="full-size selection")
    mask = _key_mask(sel, sub, heads)
    qs = Q64 if rows is None else Q64[:, :, rows]
    Oref, Lref, rc = oracle.attention(qs, oracle.to_f64(_bits(K[heads])), oracle.to_f64(_bits(V[heads])),
                                      mask, oracle.to_f64(_bits(Ku[:, heads])),
                                      oracle.to_f64(_bits(Vu[:, heads])), prefill, scale,
                                      qpos=rows, n_q_total=Q.shape[2])
    assert rc == 0
    Og = O[:, heads].float().cpu().numpy()
    Lg = LSE[:, heads].cpu().numpy()
    if rows is not None:
        Og, Lg = Og[:, :, rows], Lg[:, :, rows]
    assert np.abs(Og - Oref).max() <= 2e-2
    assert rel_l2(Og, Oref) <= 5e-3
    assert np.abs(Lg - Lref).max() <= 1e-3


@pytest.fixture(scope="module")
def ctx32k():
    sqz = _sqz()
    H, L, d, c = 32, 32768, 128, 1024
    fc = synth.fixed_context(H, L, d, c, seed=1002)
    K, V = sqz.to_device(fc.K), sqz.to_device(fc.V)
    init2 = torch.from_numpy(synth.kmeans_init(H, L, c, seed=2002)).cuda()
    return fc, K, V, init2


def test_cfg2_decode_fullsize(ctx32k):
    sqz = _sqz()
    fc, K, V, init2 = ctx32k
    Qc = sqz.to_device(synth.decode_queries(fc.mix, 32, seed=3002))
    Q = sqz.to_device(synth.decode_queries(fc.mix, 1, seed=4002))
    Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, 1024, seed=5002))
    idx, sel, O, LSE, T, T1, scale, heads = _run(K, V, Q, Ku, Vu, 1024, 0, init2, None, False, 0.3, Qc)
    _check(idx, sel, O, LSE, T, T1, scale, heads, Q, K, V, Ku, Vu, False)


def test_cfg2_decode_step_fullsize(ctx32k):
    """cfg2 at full size through sqz_decode_step (user KV in chunks beside the lookup,
    rows merged behind the attention grid), on two sampled heads; run twice on the same
    workspace (self-cleaning counters)."""
    sqz = _sqz()
    fc, K, V, init2 = ctx32k
    Qc = sqz.to_device(synth.decode_queries(fc.mix, 32, seed=3002))
    Q = sqz.to_device(synth.decode_queries(fc.mix, 1, seed=4012))
    Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, 1024, seed=5012))
    for _ in range(2):
        idx, sel, O, LSE, T, T1, scale, heads = _run(K, V, Q, Ku, Vu, 1024, 0, init2, None, False, 0.3, Qc,
                                                     step=True)
        _check(idx, sel, O, LSE, T, T1, scale, heads, Q, K, V, Ku, Vu, False)


def test_cfg3_prefill_fullsize(ctx32k):
    sqz = _sqz()
    fc, K, V, init2 = ctx32k
    n_q = 1024
    Qc = sqz.to_device(synth.prefill_queries(fc.mix, 2, n_q, seed=3003))
    Q = sqz.to_device(synth.prefill_queries(fc.mix, 1, n_q, seed=4003))
    Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, n_q, seed=5003))
    idx, sel, O, LSE, T, T1, scale, heads = _run(K, V, Q, Ku, Vu, 1024, 0, init2, None, True, 0.3, Qc)
    rows = np.unique(np.concatenate([[0, n_q - 1], np.linspace(0, n_q - 1, 62).astype(np.int32)]))
    _check(idx, sel, O, LSE, T, T1, scale, heads, Q, K, V, Ku, Vu, True, rows=rows.astype(np.int32))


def test_cfg4_hier_decode_fullsize():
    sqz = _sqz()
    H, L, d, c2, c1, B = 32, 131072, 128, 6554, 1311, 8
    mix = synth.device_mixture(H, c2, d, G1=c1, seed=1004)
    K, V = synth.device_keys(mix, L, seed=1004)
    init2 = synth.device_kmeans_init(H, L, c2, 2004)
    init1 = synth.device_kmeans_init(H, c2, c1, 2104)
    Qc = synth.device_decode_queries(mix, 16, seed=3004)
    Q = synth.device_decode_queries(mix, B, seed=4004)
    Ku, Vu = synth.device_user_kv(mix, B, 1024, seed=5004)
    idx, sel, O, LSE, T, T1, scale, heads = _run(K, V, Q, Ku, Vu, c2, c1, init2, init1, False, 0.1, Qc)
    # Level-1 survivors of the GPU, for the conditional Level-2 comparison
    sel_dbg = sqz.Selection.empty(idx, B, 1, debug=True)
    sqz.centroid_lookup(idx, Q, scale, T, T1, sel=sel_dbg)
    torch.cuda.synchronize()
    assert torch.equal(sel_dbg.n_keys, sel.n_keys)
    _check(idx, sel_dbg, O, LSE, T, T1, scale, heads, Q, K, V, Ku, Vu, False)


def test_slim_layout_large_level2():
    """A Level-2 table large enough (47K rows) that the one-query decode lookup
    takes the 12-byte-per-row SLIM layout in 8-CTA clusters (cfg5's case), checked
    against the oracle on every head."""
    sqz = _sqz()
    H, L, d, c2, c1 = 2, 49152, 128, 47000, 9400
    fc = synth.fixed_context(H, L, d, c2, seed=1109, G1=c1)
    K, V = sqz.to_device(fc.K), sqz.to_device(fc.V)
    init2 = torch.from_numpy(synth.kmeans_init(H, L, c2, seed=2109)).cuda()
    init1 = torch.from_numpy(synth.kmeans_init(H, c2, c1, seed=2209)).cuda()
    Qc = sqz.to_device(synth.decode_queries(fc.mix, 16, seed=3109))
    Q = sqz.to_device(synth.decode_queries(fc.mix, 1, seed=4109))
    Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, 64, seed=5109))
    idx, Kp, Vp, _ = sqz.cluster_keys(K, V, c2, init2, c1, init1, max_iters=3)
    scale = 1.0 / np.sqrt(d)
    s = sqz.centroid_lookup(idx, Qc, scale, 0.0, 0.0, debug=True)
    T1 = calib.distributed_threshold(s.dbg_S1, idx.N1[None], 0.5, float(16 * idx.N1.sum()))
    s = sqz.centroid_lookup(idx, Qc, scale, 0.0, T1, debug=True)
    T = calib.distributed_threshold(s.dbg_S, idx.N2[None], 0.1, float(16 * H * L))
    sel = sqz.centroid_lookup(idx, Q, scale, T, T1, debug=True)
    O, LSE = sqz.sparse_attention(Q, Kp, Vp, idx, sel, Ku, Vu, scale)
    torch.cuda.synchronize()
    assert int(sel.n_keys.min()) > 0
    _check(idx, sel, O, LSE, T, T1, scale, [0, 1], Q, K, V, Ku, Vu, False)


def test_cfg5p_shape_hier_prefill():
    """The cfg5-prefill launch shape on a smaller context: hierarchical lookup with
    4096 query rows (32 query tiles of the tensor-core lookup, the Level-2 pass on
    the candidate-row list), 4096 causal user keys, c1 = 1% / c2 = 5% of L, 10%
    retention; two heads checked against the oracle (lookup on all 4096 rows, the
    attention on 64 sampled rows incl. the first and last)."""
    sqz = _sqz()
    H, L, d, n_q = 4, 32768, 128, 4096
    c1, c2 = synth.centroid_counts(L)
    fc = synth.fixed_context(H, L, d, c2, seed=1105, G1=c1)
    K, V = sqz.to_device(fc.K), sqz.to_device(fc.V)
    init2 = torch.from_numpy(synth.kmeans_init(H, L, c2, seed=2105)).cuda()
    init1 = torch.from_numpy(synth.kmeans_init(H, c2, c1, seed=2205)).cuda()
    Qc = sqz.to_device(synth.prefill_queries(fc.mix, 1, n_q, seed=3105))
    Q = sqz.to_device(synth.prefill_queries(fc.mix, 1, n_q, seed=4105))
    Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, n_q, seed=5105))
    idx, sel, O, LSE, T, T1, scale, heads = _run(K, V, Q, Ku, Vu, c2, c1, init2, init1, True, 0.1, Qc)
    sel_dbg = sqz.Selection.empty(idx, 1, n_q, debug=True)
    sqz.centroid_lookup(idx, Q, scale, T, T1, sel=sel_dbg)
    torch.cuda.synchronize()
    assert torch.equal(sel_dbg.n_keys, sel.n_keys)
    assert int(sel.n_keys.min()) > 0
    rows = np.unique(np.concatenate([[0, n_q - 1], np.linspace(0, n_q - 1, 62).astype(np.int32)]))
    _check(idx, sel_dbg, O, LSE, T, T1, scale, heads, Q, K, V, Ku, Vu, True, rows=rows.astype(np.int32))
