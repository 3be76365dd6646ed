"""GPU parity: libsqz (through the C ABI) vs the fp64 CPU oracle on the same seeded inputs.

Selection: identical finest-level cluster sets except clusters whose oracle score lies
within 1e-5 relative of the threshold; hierarchical Level 2 is compared conditioned on
the GPU's Level-1 survivors (parity rules).  Attention: evaluated by the
oracle on the GPU's selected key set ("given the same mask"); bf16 O max-abs <= 2e-2 and
rel-L2 <= 5e-3, fp32 O max-abs <= 1e-4, LSE within 1e-3 (north star)."""
import zlib

import numpy as np
import pytest

import oracle
from paper_2411_09688_b200 import calib, synth

from helpers import (assert_selection_parity, gpu_index, gpu_sets, key_mask_from_gpu,
                     oracle_problem, rel_l2)

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


def _calibrate(P, scale, retention, prefill=False, n_cal=24, ret1=0.5):
    """T (and T1) from oracle scores of separate calibration queries (R17)."""
    idx = P["idx"]
    mix = P["fc"].mix
    if prefill:
        Qc = synth.prefill_queries(mix, 4, 64, seed=777, dtype=P["dtype"])
    else:
        Qc = synth.decode_queries(mix, n_cal, seed=777, dtype=P["dtype"])
    Qc = oracle.to_f64(Qc)
    T1 = 0.0
    if idx.levels == 2:
        r = oracle.lookup(Qc, idx, scale, 0.0, 0.0)
        T1 = calib.weighted_threshold(r["Sbar1"], idx.N1[None], ret1)
    r = oracle.lookup(Qc, idx, scale, 0.0, T1)
    T = calib.weighted_threshold(r["Sbar2"], idx.N2[None], retention)
    return T, T1


def _check_lookup(P, sel, scale, T, T1, B, T0=0.0):
    idx = P["idx"]
    Q64 = oracle.to_f64(P["Q"])
    H = idx.H
    forced = forced0 = None
    if idx.levels == 3:  # Level 0, then Level 1 conditioned on the GPU's Level-0 set
        ref0 = oracle.lookup(Q64, idx, scale, T, T1, T0=T0)
        g0 = sel.l0_surv.cpu().numpy().astype(bool)
        assert_selection_parity(g0, ref0["surv0"], ref0["Sbar0"], T0, what="level-0")
        np.testing.assert_allclose(sel.dbg_S0.cpu().numpy(), ref0["Sbar0"], rtol=2e-5, atol=1e-12)
        forced0 = g0
    if idx.levels >= 2:
        ref1 = oracle.lookup(Q64, idx, scale, T, T1, T0=T0, forced_l0=forced0)
        g1 = sel.l1_surv.cpu().numpy().astype(bool)
        assert_selection_parity(g1, ref1["surv1"], ref1["Sbar1"], T1, what="level-1")
        np.testing.assert_allclose(sel.dbg_S1.cpu().numpy(), ref1["Sbar1"], rtol=2e-5, atol=1e-12)
        forced = g1
    ref = oracle.lookup(Q64, idx, scale, T, T1, forced_l1=forced, T0=T0, forced_l0=forced0)
    g = gpu_sets(sel, B, H, idx.c2)
    ndiff = assert_selection_parity(g, ref["sel2"], ref["Sbar2"], T)
    S_gpu = sel.dbg_S.cpu().numpy()
    assert np.array_equal(np.isnan(S_gpu), np.isnan(ref["Sbar2"]))
    m = ~np.isnan(ref["Sbar2"])
    np.testing.assert_allclose(S_gpu[m], ref["Sbar2"][m], rtol=2e-5, atol=1e-12)
    lse = sel.dbg_lse.cpu().numpy()
    fin = np.isfinite(ref["lse"])
    assert np.array_equal(np.isfinite(lse), fin)
    np.testing.assert_allclose(lse[fin], ref["lse"][fin], atol=1e-4, rtol=1e-5)
    # k = sum N over the selected clusters; key_idx is the concatenation of their ranges
    nk = sel.n_keys.cpu().numpy()
    ki = sel.key_idx.cpu().numpy()
    for b in range(B):
        for h in range(H):
            cl = np.nonzero(g[b, h])[0]
            assert nk[b, h] == idx.N2[h][cl].sum()
            exp = np.concatenate([np.arange(idx.key_off[h, i], idx.key_off[h, i + 1]) for i in cl]
                                 + [np.zeros(0, np.int64)])
            assert np.array_equal(ki[b, h, :nk[b, h]], exp)
    return ndiff


def _check_attention(P, sel, O, LSE, scale, causal, B, tol_abs, tol_rel):
    idx = P["idx"]
    mask = key_mask_from_gpu(sel, idx, B, idx.H)
    Ku = None if P["Ku"] is None else oracle.to_f64(P["Ku"])
    Vu = None if P["Vu"] is None else oracle.to_f64(P["Vu"])
    Oref, Lref, _ = oracle.attention(oracle.to_f64(P["Q"]), oracle.to_f64(P["fc"].K),
                                     oracle.to_f64(P["fc"].V), mask, Ku, Vu, causal, scale)
    Og = O.float().cpu().numpy().astype(np.float64)
    Lg = LSE.cpu().numpy().astype(np.float64)
    fin = np.isfinite(Lref)
    assert np.array_equal(np.isfinite(Lg), fin)
    assert np.abs(Og - Oref).max() <= tol_abs, np.abs(Og - Oref).max()
    if tol_rel is not None:
        assert rel_l2(Og, Oref) <= tol_rel, rel_l2(Og, Oref)
    np.testing.assert_allclose(Lg[fin], Lref[fin], atol=1e-3, rtol=0)


def _device(P):
    sqz = _sqz()
    t = {k: (None if P[k] is None else sqz.to_device(P[k])) for k in ("Q", "Ku", "Vu")}
    idx = P["idx"]
    t["Kp"] = sqz.to_device(oracle.permute_kv(P["fc"].K, idx))
    t["Vp"] = sqz.to_device(oracle.permute_kv(P["fc"].V, idx))
    t["idx"] = gpu_index(idx)
    return t


def _check_runs(t, sel, O, LSE, scale, T, T1, causal, partial):
    """The run-length selection (key_pref, no key_idx) gives the same selection and
    bit-identical attention: key_pref is the exclusive prefix of N over the
    selected clusters, and the attention kernels read the same positions."""
    sqz = _sqz()
    B, H = sel.n_keys.shape
    r = sqz.Selection.empty(t["idx"], B, t["Q"].shape[2], key_idx=False)
    sqz.centroid_lookup(t["idx"], t["Q"], scale, T, T1, sel=r)
    O2, L2 = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], r, t["Ku"], t["Vu"], scale,
                                  causal=causal, partial=partial)
    torch.cuda.synchronize()
    assert torch.equal(r.n_clusters, sel.n_clusters) and torch.equal(r.n_keys, sel.n_keys)
    N2 = t["idx"].N2.cpu().numpy()
    for b in range(B):
        for h in range(H):
            n = int(sel.n_clusters[b, h])
            cl = sel.clusters[b, h, :n].cpu().numpy()
            assert np.array_equal(r.clusters[b, h, :n].cpu().numpy(), cl)
            pref = np.concatenate([[0], np.cumsum(N2[h][cl])[:-1]]) if n else np.zeros(0)
            assert np.array_equal(r.key_pref[b, h, :n].cpu().numpy(), pref)
            assert np.array_equal(sel.key_pref[b, h, :n].cpu().numpy(), pref)
    assert torch.equal(O2, O) and torch.equal(L2, LSE), "run-length attention differs"


DECODE_CASES = [
    # id, H, L, d, c2, c1, dtype, B, n_u, retention
    ("cfg1_fp32", 1, 1024, 64, 32, 0, synth.F32, 1, 16, 0.3),
    ("bf16_d128", 4, 3000, 128, 97, 0, synth.BF16, 3, 37, 0.3),
    ("bf16_d64_B9", 2, 2500, 64, 61, 0, synth.BF16, 9, 5, 0.2),
    ("hier_bf16", 3, 4000, 128, 200, 40, synth.BF16, 2, 33, 0.1),
    ("hier_fp32_B8", 2, 3000, 64, 150, 30, synth.F32, 8, 0, 0.15),
    # B >= 4: Level 2 scans the whole table with per-query parent masks
    ("hier_bf16_B5", 3, 4000, 128, 200, 40, synth.BF16, 5, 20, 0.1),
    # many rows whose streams are shorter than the decode partition's per-segment
    # setup allowance (fewer CTAs than the grid, ranges mostly inside setup units)
    ("bf16_many_short_rows", 16, 640, 128, 40, 0, synth.BF16, 12, 3, 0.05),
    # no user keys and a very sparse selection: rows with no key at all
    ("bf16_d64_sparse_nu0", 8, 700, 64, 50, 0, synth.BF16, 16, 0, 0.03),
    # fp32 storage at d = 128 (k_lookup_decode<float,128>, k_attend<float,128>)
    ("fp32_d128", 3, 2000, 128, 64, 0, synth.F32, 2, 20, 0.3),
    ("hier_fp32_d128", 2, 3000, 128, 150, 30, synth.F32, 1, 16, 0.15),
]


@pytest.mark.parametrize("case", DECODE_CASES, ids=lambda c: c[0])
def test_decode_lookup_and_attention(case):
    sqz = _sqz()
    _, H, L, d, c2, c1, dt, B, n_u, ret = case
    P = oracle_problem(H, L, d, c2, c1, dt, seed=zlib.crc32(case[0].encode()) % 1000, B=B, n_u=n_u)
    scale = 1.0 / np.sqrt(d)
    T, T1 = _calibrate(P, scale, ret)
    t = _device(P)
    sel = sqz.centroid_lookup(t["idx"], t["Q"], scale, T, T1, debug=True)
    torch.cuda.synchronize()
    _check_lookup(P, sel, scale, T, T1, B)
    O, LSE = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, t["Ku"], t["Vu"], scale,
                                  partial=True)
    torch.cuda.synchronize()
    fp32 = dt == synth.F32
    _check_attention(P, sel, O, LSE, scale, False, B, 1e-4 if fp32 else 2e-2,
                     None if fp32 else 5e-3)
    _check_runs(t, sel, O, LSE, scale, T, T1, False, True)


SHARED_CASES = [
    # batch-shared decode (NEXT-1): B queries per head over one fixed context; the
    # union pass must give every query exactly its own selection's attention
    ("shared_B8", 4, 5000, 128, 120, 0, synth.BF16, 8, 64, 0.15),
    ("shared_B16_hier", 3, 6000, 128, 240, 40, synth.BF16, 16, 33, 0.1),
    ("shared_B2_nu0", 2, 3000, 128, 90, 0, synth.BF16, 2, 0, 0.3),
    ("shared_B5_dense", 2, 2100, 128, 50, 0, synth.BF16, 5, 17, 1.0),
]


@pytest.mark.parametrize("case", SHARED_CASES, ids=lambda c: c[0])
def test_decode_batch_shared(case):
    sqz = _sqz()
    name, H, L, d, c2, c1, dt, B, n_u, ret = case
    P = oracle_problem(H, L, d, c2, c1, dt, seed=zlib.crc32(name.encode()) % 1000, B=B, n_u=n_u)
    scale = 1.0 / np.sqrt(d)
    if ret >= 1.0:
        T, T1 = 0.0, 0.0
    else:
        T, T1 = _calibrate(P, scale, ret)
    t = _device(P)
    sel = sqz.centroid_lookup(t["idx"], t["Q"], scale, T, T1, debug=True)
    O, LSE = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, t["Ku"], t["Vu"], scale)
    Or, Lr = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, t["Ku"], t["Vu"], scale,
                                  per_row=True)
    torch.cuda.synchronize()
    _check_attention(P, sel, O, LSE, scale, False, B, 2e-2, 5e-3)
    # the two paths compute the same rows (different summation order only)
    assert (O.float() - Or.float()).abs().max().item() <= 2e-2
    assert (LSE - Lr).abs().max().item() <= 1e-3
    # repeated calls reuse the self-cleaning workspace
    O2, L2 = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, t["Ku"], t["Vu"], scale)
    torch.cuda.synchronize()
    assert torch.equal(O, O2) and torch.equal(LSE, L2)


# decode-step path (B = 1, single level, n_u > 0): a lean lookup grid, and the
# attention kernel attends the user KV in chunks before it waits for the lookup
STEP_CASES = [
    # id, H, L, d, c2, c1, dtype, B, n_u, retention
    ("step_bf16_d128_nu37", 4, 3000, 128, 97, 0, synth.BF16, 1, 37, 0.3),
    ("step_bf16_d64_nu9", 3, 2500, 64, 61, 0, synth.BF16, 1, 9, 0.2),
    ("step_fp32_d128", 3, 2000, 128, 64, 0, synth.F32, 1, 20, 0.3),
    ("step_fp32_d64_nu1", 2, 1500, 64, 40, 0, synth.F32, 1, 1, 0.3),
    # rows with no selected cluster (user keys only) and rows with nothing at all
    ("step_bf16_sparse_nu0", 8, 700, 64, 50, 0, synth.BF16, 1, 0, 0.03),
    ("step_bf16_sparse_nu5", 8, 700, 64, 50, 0, synth.BF16, 1, 5, 0.03),
    # many user chunks per row (a ragged last chunk)
    ("step_bf16_big_nu", 2, 2048, 128, 64, 0, synth.BF16, 1, 3000, 0.3),
    # many heads, cfg2-like clusters
    ("step_bf16_h32", 32, 4096, 128, 128, 0, synth.BF16, 1, 300, 0.3),
]


@pytest.mark.parametrize("case", DECODE_CASES + STEP_CASES, ids=lambda c: c[0])
def test_decode_step(case):
    """sqz_decode_step (one call: the user-chunk path for one single-level query
    row, else the two calls) against the oracle: the selection
    under the band rule, key_pref / key_idx consistent with it, and the attention
    on its key set."""
    sqz = _sqz()
    _, H, L, d, c2, c1, dt, B, n_u, ret = case
    P = oracle_problem(H, L, d, c2, c1, dt, seed=zlib.crc32(case[0].encode()) % 1000, B=B, n_u=n_u)
    scale = 1.0 / np.sqrt(d)
    T, T1 = _calibrate(P, scale, ret)
    t = _device(P)
    idx = P["idx"]
    for rep in range(2):  # the second call reuses the (self-cleaning) workspace
        sel = sqz.Selection.empty(t["idx"], B, 1)
        sel_l1 = sqz.Selection.empty(t["idx"], B, 1, debug=True) if idx.levels == 2 else None
        sel, O, LSE = sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], t["Ku"], t["Vu"], scale, T, T1,
                                      sel=sel, partial=True)
        torch.cuda.synchronize()
        Q64 = oracle.to_f64(P["Q"])
        forced = None
        if idx.levels == 2:  # Level-1 survivors of the GPU for the conditional comparison
            sqz.centroid_lookup(t["idx"], t["Q"], scale, T, T1, sel=sel_l1)
            torch.cuda.synchronize()
            forced = sel_l1.l1_surv.cpu().numpy().astype(bool)
        ref = oracle.lookup(Q64, idx, scale, T, T1, forced_l1=forced)
        g = gpu_sets(sel, B, H, idx.c2)
        assert_selection_parity(g, ref["sel2"], ref["Sbar2"], T)
        nk = sel.n_keys.cpu().numpy()
        ki = sel.key_idx.cpu().numpy()
        kp = sel.key_pref.cpu().numpy()
        for b in range(B):
            for h in range(H):
                cl = np.nonzero(g[b, h])[0]
                assert nk[b, h] == idx.N2[h][cl].sum()
                assert int(sel.n_clusters[b, h]) == len(cl)
                exp = np.concatenate([np.arange(idx.key_off[h, i], idx.key_off[h, i + 1]) for i in cl]
                                     + [np.zeros(0, np.int64)])
                assert np.array_equal(ki[b, h, :nk[b, h]], exp)
                pref = np.concatenate([[0], np.cumsum(idx.N2[h][cl])[:-1]]) if len(cl) else np.zeros(0)
                assert np.array_equal(kp[b, h, :len(cl)], pref)
        fp32 = dt == synth.F32
        _check_attention(P, sel, O, LSE, scale, False, B, 1e-4 if fp32 else 2e-2,
                         None if fp32 else 5e-3)


def test_decode_step_empty_rows_and_status():
    """A threshold no cluster passes: rows attend only their user keys; with no user
    keys either they are empty (identity partial, or SQZ_ERR_EMPTY when final)."""
    sqz = _sqz()
    P = oracle_problem(3, 900, 128, 30, 0, synth.BF16, seed=12, B=2, n_u=5)
    t = _device(P)
    scale = 1 / np.sqrt(128)
    sel, O, LSE = sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], t["Ku"], t["Vu"], scale, 1.0)
    torch.cuda.synchronize()
    assert int(sel.n_keys.sum()) == 0
    _check_attention(P, sel, O, LSE, scale, False, 2, 2e-2, 5e-3)
    sqz.attention_status()
    sel, O, LSE = sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], None, None, scale, 1.0, partial=True)
    torch.cuda.synchronize()
    assert torch.isneginf(LSE).all() and (O == 0).all()
    sqz.attention_status()
    sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], None, None, scale, 1.0, partial=False)
    with pytest.raises(sqz.SqzError) as e:
        sqz.attention_status()
    assert e.value.code == sqz.SQZ_ERR_EMPTY


def test_decode_step_user_chunks_empty_rows_and_status():
    """The user-chunk path (B = 1) with a threshold no cluster passes: rows attend
    only their user keys (the chunk partials alone); with no user keys they are
    empty (identity partial, or SQZ_ERR_EMPTY when final); the chunk counts
    self-clean across calls."""
    sqz = _sqz()
    P = oracle_problem(3, 900, 128, 30, 0, synth.BF16, seed=13, B=1, n_u=21)
    t = _device(P)
    scale = 1 / np.sqrt(128)
    for _ in range(2):
        sel, O, LSE = sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], t["Ku"], t["Vu"], scale, 1.0)
        torch.cuda.synchronize()
        assert int(sel.n_keys.sum()) == 0
        _check_attention(P, sel, O, LSE, scale, False, 1, 2e-2, 5e-3)
        sqz.attention_status()
    sel, O, LSE = sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], None, None, scale, 1.0, partial=True)
    torch.cuda.synchronize()
    assert torch.isneginf(LSE).all() and (O == 0).all()
    sqz.attention_status()
    sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], None, None, scale, 1.0, partial=False)
    with pytest.raises(sqz.SqzError) as e:
        sqz.attention_status()
    assert e.value.code == sqz.SQZ_ERR_EMPTY
    # and a normal step right after still selects and attends correctly
    T, _ = _calibrate(P, scale, 0.3)
    sel, O, LSE = sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], t["Ku"], t["Vu"], scale, T)
    torch.cuda.synchronize()
    assert int(sel.n_keys.sum()) > 0
    _check_attention(P, sel, O, LSE, scale, False, 1, 2e-2, 5e-3)


@pytest.mark.parametrize("shape", [(32, 4096, 128, 128, 300), (2, 1024, 64, 32, 16)],
                         ids=["h32_merge_kernel", "tiny_ticket_merge"])
def test_decode_step_repeat_bit_identical(shape):
    """The decode step is deterministic and its workspace self-cleaning: 12 calls on the
    same input, interleaved with debug calls (which run the two-call path on the same
    attention region), give bit-identical O, LSE and selections."""
    sqz = _sqz()
    H, L, d, c2, n_u = shape
    P = oracle_problem(H, L, d, c2, 0, synth.BF16, seed=77, B=1, n_u=n_u)
    scale = 1.0 / np.sqrt(d)
    T, _ = _calibrate(P, scale, 0.3)
    t = _device(P)
    ref = None
    for it in range(12):
        debug = it % 4 == 3
        sel = sqz.Selection.empty(t["idx"], 1, 1, debug=debug)
        sel, O, LSE = sqz.decode_step(t["idx"], t["Q"], t["Kp"], t["Vp"], t["Ku"], t["Vu"], scale, T, sel=sel)
        torch.cuda.synchronize()
        got = (O.clone(), LSE.clone(), sel.n_clusters.clone(), sel.n_keys.clone())
        if ref is None:
            ref = got
            _check_attention(P, sel, O, LSE, scale, False, 1, 2e-2, 5e-3)
            continue
        assert torch.equal(got[2], ref[2]) and torch.equal(got[3], ref[3])
        if debug:  # the two-call path: same rows, another summation order
            assert (got[0].float() - ref[0].float()).abs().max().item() <= 2e-2
            assert (got[1] - ref[1]).abs().max().item() <= 1e-3
        else:
            assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])


PREFILL_CASES = [
    # id, H, L, d, c2, c1, dtype, B, n_q, n_u, retention, causal
    ("bf16_single", 2, 2048, 128, 100, 0, synth.BF16, 1, 200, 200, 0.3, True),
    ("fp32_d64", 1, 1500, 64, 40, 0, synth.F32, 2, 70, 90, 0.3, True),
    ("hier_bf16", 2, 3000, 128, 150, 30, synth.BF16, 1, 130, 130, 0.15, True),
    # non-causal: every user key visible to every query row
    ("bf16_noncausal_B2", 2, 2048, 128, 100, 0, synth.BF16, 2, 300, 150, 0.3, False),
    ("fp32_d64_noncausal", 1, 1500, 64, 40, 0, synth.F32, 1, 50, 20, 0.3, False),
    # more 128-key tiles than SMs: segments cut across CTAs, multi-part merges,
    # several pieces per CTA, ragged last query pair
    ("bf16_multiseg", 4, 6000, 128, 150, 0, synth.BF16, 1, 600, 600, 0.4, True),
    # bf16 d = 64: k_prefill_lookup_tc<64, *> and the split-KV k_prefill_attend<64>
    ("bf16_d64", 2, 2048, 64, 100, 0, synth.BF16, 1, 200, 200, 0.3, True),
    ("bf16_d64_noncausal_B2", 2, 2048, 64, 100, 0, synth.BF16, 2, 300, 150, 0.3, False),
    ("hier_bf16_d64", 2, 3000, 64, 150, 30, synth.BF16, 1, 130, 130, 0.15, True),
    ("hier_bf16_d64_noncausal", 2, 3000, 64, 150, 30, synth.BF16, 1, 170, 60, 0.15, False),
    # 5 query tiles: the candidate rows are gathered once and TMA-loaded per tile
    ("hier_bf16_gathered", 2, 4000, 128, 200, 40, synth.BF16, 2, 600, 300, 0.15, True),
    ("hier_bf16_d64_gathered", 2, 3000, 64, 150, 30, synth.BF16, 1, 520, 100, 0.15, False),
    ("bf16_d64_multiseg", 4, 6000, 64, 150, 0, synth.BF16, 1, 600, 600, 0.4, True),
    # fp32 d = 128 prefill (k_prefill_rowlse / colsum<float,128>, exact FFMA attention)
    ("fp32_d128", 1, 1500, 128, 40, 0, synth.F32, 1, 70, 90, 0.3, True),
    ("hier_fp32_d128", 1, 2000, 128, 100, 20, synth.F32, 1, 65, 40, 0.2, True),
]


@pytest.mark.parametrize("case", PREFILL_CASES, ids=lambda c: c[0])
def test_prefill_lookup_and_attention(case):
    sqz = _sqz()
    _, H, L, d, c2, c1, dt, B, n_q, n_u, ret, causal = case
    P = oracle_problem(H, L, d, c2, c1, dt, seed=zlib.crc32(case[0].encode()) % 1000 + 7, B=B, n_u=n_u, n_q=n_q,
                       prefill=True)
    scale = 1.0 / np.sqrt(d)
    T, T1 = _calibrate(P, scale, ret, prefill=True)
    t = _device(P)
    sel = sqz.centroid_lookup(t["idx"], t["Q"], scale, T, T1, debug=True)
    torch.cuda.synchronize()
    _check_lookup(P, sel, scale, T, T1, B)
    O, LSE = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, t["Ku"], t["Vu"], scale,
                                  causal=causal)
    torch.cuda.synchronize()
    fp32 = dt == synth.F32
    _check_attention(P, sel, O, LSE, scale, causal, B, 1e-4 if fp32 else 2e-2,
                     None if fp32 else 5e-3)
    _check_runs(t, sel, O, LSE, scale, T, T1, causal, False)


def test_threshold_zero_is_dense_attention():
    """North star: T = 0 selects every key and reproduces dense attention."""
    sqz = _sqz()
    P = oracle_problem(2, 1800, 128, 60, 0, synth.BF16, seed=5, B=2, n_u=9)
    t = _device(P)
    scale = 1 / np.sqrt(128)
    sel = sqz.centroid_lookup(t["idx"], t["Q"], scale, 0.0, debug=True)
    O, LSE = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, t["Ku"], t["Vu"], scale)
    torch.cuda.synchronize()
    assert (sel.n_keys.cpu().numpy() == 1800).all()
    Oref, Lref, _ = oracle.attention(oracle.to_f64(P["Q"]), oracle.to_f64(P["fc"].K),
                                     oracle.to_f64(P["fc"].V), None, oracle.to_f64(P["Ku"]),
                                     oracle.to_f64(P["Vu"]), False, scale)
    assert np.abs(O.float().cpu().numpy() - Oref).max() <= 2e-2
    np.testing.assert_allclose(LSE.cpu().numpy(), Lref, atol=1e-3)


def test_empty_selection_edges():
    sqz = _sqz()
    P = oracle_problem(1, 512, 64, 16, 0, synth.F32, seed=6, B=1, n_u=0)
    t = _device(P)
    scale = 1 / 8.0
    sel = sqz.centroid_lookup(t["idx"], t["Q"], scale, 1.0, debug=True)  # S_i <= 1/N_i < 1
    assert int(sel.n_keys.sum()) == 0 and int(sel.n_clusters.sum()) == 0
    O, LSE = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, None, None, scale,
                                  partial=True)
    torch.cuda.synchronize()
    assert torch.isneginf(LSE).all() and (O == 0).all()
    sqz.attention_status()  # partial mode: not an error
    sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, None, None, scale, partial=False)
    with pytest.raises(sqz.SqzError) as e:
        sqz.attention_status()
    assert e.value.code == sqz.SQZ_ERR_EMPTY
    sqz.attention_status()  # flag cleared


def test_merge_partials_matches_oracle():
    sqz = _sqz()
    rng = np.random.default_rng(3)
    P, rows, d = 5, 77, 128
    Op = rng.standard_normal((P, rows, d)).astype(np.float32)
    Lp = (rng.standard_normal((P, rows)) * 4).astype(np.float32)
    Lp[1, :10] = -np.inf
    Lp[:, 20] = -np.inf
    O, L = sqz.merge_partials(torch.from_numpy(Op).cuda(), torch.from_numpy(Lp).cuda())
    Oref, Lref = oracle.merge(Op.astype(np.float64), Lp.astype(np.float64))
    np.testing.assert_allclose(O.cpu().numpy(), Oref, atol=1e-5)
    fin = np.isfinite(Lref)
    assert np.array_equal(np.isfinite(L.cpu().numpy()), fin)
    np.testing.assert_allclose(L.cpu().numpy()[fin], Lref[fin], atol=1e-5)


def test_invalid_arguments_rejected():
    sqz = _sqz()
    P = oracle_problem(1, 256, 64, 8, 0, synth.F32, seed=8)
    t = _device(P)
    with pytest.raises(sqz.SqzError) as e:
        sqz.centroid_lookup(t["idx"], t["Q"], 0.125, -1.0)
    assert e.value.code == sqz.SQZ_ERR_INVALID_ARG and "T" in str(e.value)
    with pytest.raises(sqz.SqzError):
        sqz.centroid_lookup(t["idx"], t["Q"], 0.125, float("nan"))


# ---- three levels (NEXT-2) ----
THREE_CASES = [
    # name, H, L, d, c2, c1, c0, dtype, B, n_q, n_u, prefill
    ("decode_bf16_B3", 3, 6000, 128, 240, 48, 8, synth.BF16, 3, 1, 33, False),
    ("decode_fp32_d64", 2, 5000, 64, 200, 40, 6, synth.F32, 2, 1, 16, False),
    ("prefill_bf16_causal", 2, 6000, 128, 240, 48, 8, synth.BF16, 1, 150, 150, True),
]


@pytest.mark.parametrize("case", THREE_CASES, ids=lambda c: c[0])
def test_three_level_lookup_and_attention(case):
    """Three-level index built on the GPU, then lookup + attention: every level's
    decision equals the oracle's (band rule) conditioned on the GPU's coarser sets,
    and attention over the selection equals the oracle's."""
    sqz = _sqz()
    name, H, L, d, c2, c1, c0, dt, B, n_q, n_u, prefill = case
    seed = zlib.crc32(name.encode()) % 1000
    fc = synth.fixed_context(H, L, d, c2, dtype=dt, seed=seed, G1=c1)
    i2 = synth.kmeans_init(H, L, c2, seed=seed + 1)
    i1 = synth.kmeans_init(H, c2, c1, seed=seed + 2)
    i0 = synth.kmeans_init(H, c1, c0, seed=seed + 5)
    gidx, Kp, Vp, its = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), c2,
                                         torch.from_numpy(i2).cuda(), c1, torch.from_numpy(i1).cuda(),
                                         max_iters=20, c0=c0, init0=torch.from_numpy(i0).cuda())
    torch.cuda.synchronize()
    sqz.index_validate(gidx)
    assert len(its) == 3
    # the oracle evaluates the GPU-built tables
    def f64(t):
        a = t.cpu()
        return oracle.to_f64(a.view(torch.int16).numpy().view(np.uint16) if a.dtype == torch.bfloat16
                             else a.numpy())
    idx = oracle.Index(levels=3, dtype=dt, H=H, L=L, d=d, c2=c2, C2=f64(gidx.C2),
                       N2=gidx.N2.cpu().numpy(), key_off=gidx.key_off.cpu().numpy(),
                       perm=gidx.perm.cpu().numpy(), c1=c1, C1=f64(gidx.C1), N1=gidx.N1.cpu().numpy(),
                       child_off=gidx.child_off.cpu().numpy(), c0=c0, C0=f64(gidx.C0),
                       N0=gidx.N0.cpu().numpy(), child_off0=gidx.child_off0.cpu().numpy())
    if prefill:
        Q = synth.prefill_queries(fc.mix, B, n_q, seed=seed + 3, dtype=dt)
        Qc = synth.prefill_queries(fc.mix, 2, 64, seed=777, dtype=dt)
    else:
        Q = synth.decode_queries(fc.mix, B, seed=seed + 3, dtype=dt)
        Qc = synth.decode_queries(fc.mix, 24, seed=777, dtype=dt)
    Ku, Vu = synth.user_kv(fc.mix, B, n_u, seed=seed + 4, dtype=dt)
    scale = 1.0 / np.sqrt(d)
    Qc64 = oracle.to_f64(Qc)
    r = oracle.lookup(Qc64, idx, scale, 0.0, 0.0, T0=0.0)
    T0 = calib.weighted_threshold(r["Sbar0"], idx.N0[None], 0.6)
    r = oracle.lookup(Qc64, idx, scale, 0.0, 0.0, T0=T0)
    T1 = calib.weighted_threshold(r["Sbar1"], idx.N1[None], 0.4,
                                  total_weight=Qc64.shape[0] * H * L)
    r = oracle.lookup(Qc64, idx, scale, 0.0, T1, T0=T0)
    T = calib.weighted_threshold(r["Sbar2"], idx.N2[None], 0.1, total_weight=Qc64.shape[0] * H * L)
    Qd = sqz.to_device(Q)
    sel = sqz.centroid_lookup(gidx, Qd, scale, T, T1, debug=True, T0=T0)
    torch.cuda.synchronize()
    P = dict(fc=fc, idx=idx, Q=Q, Ku=Ku, Vu=Vu, dtype=dt)
    assert sel.l0_surv.sum() < B * H * c0  # Level 0 prunes
    _check_lookup(P, sel, scale, T, T1, B, T0=T0)
    O, LSE = sqz.sparse_attention(Qd, Kp, Vp, gidx, sel, sqz.to_device(Ku), sqz.to_device(Vu), scale,
                                  causal=prefill, partial=True)
    torch.cuda.synchronize()
    fp32 = dt == synth.F32
    _check_attention(P, sel, O, LSE, scale, prefill, B, 1e-4 if fp32 else 2e-2, None if fp32 else 5e-3)


def test_batch_shared_empty_selections():
    """Batch-shared decode edges: thresholds that select no fixed key leave each query
    its own user keys only (exactly the oracle's user-only attention); with no user
    KV either, partial mode returns the identity (LSE = -inf, O = 0) for every row."""
    sqz = _sqz()
    P = oracle_problem(3, 2500, 128, 60, 0, synth.BF16, seed=611, B=4, n_u=9)
    scale = 1.0 / np.sqrt(128)
    t = _device(P)
    sel = sqz.centroid_lookup(t["idx"], t["Q"], scale, 0.9)  # S_i <= 1/N_i < 0.9: nothing selected
    torch.cuda.synchronize()
    assert int(sel.n_keys.sum()) == 0
    O, LSE = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, t["Ku"], t["Vu"], scale)
    torch.cuda.synchronize()
    Oref, Lref, _ = oracle.attention(oracle.to_f64(P["Q"]), oracle.to_f64(P["fc"].K),
                                     oracle.to_f64(P["fc"].V), np.zeros((4, 3, 2500), bool),
                                     oracle.to_f64(P["Ku"]), oracle.to_f64(P["Vu"]), False, scale)
    assert np.abs(O.float().cpu().numpy() - Oref).max() <= 2e-2
    assert np.abs(LSE.cpu().numpy() - Lref).max() <= 1e-3
    O2, L2 = sqz.sparse_attention(t["Q"], t["Kp"], t["Vp"], t["idx"], sel, None, None, scale, partial=True)
    torch.cuda.synchronize()
    assert torch.isneginf(L2).all() and (O2.float() == 0).all()


def test_three_level_with_T0_zero_equals_two_levels():
    """On the GPU: a three-level index with T0 = 0 keeps every Level-0 cluster, so its
    selection equals the two-level lookup on the same Level-1 / Level-2 tables."""
    sqz = _sqz()
    H, L, d, c2, c1, c0, B = 2, 5000, 128, 200, 40, 6, 3
    fc = synth.fixed_context(H, L, d, c2, dtype=synth.BF16, seed=612, G1=c1)
    g, Kp, Vp, _ = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), c2,
                                    torch.from_numpy(synth.kmeans_init(H, L, c2, seed=613)).cuda(), c1,
                                    torch.from_numpy(synth.kmeans_init(H, c2, c1, seed=614)).cuda(),
                                    max_iters=15, c0=c0,
                                    init0=torch.from_numpy(synth.kmeans_init(H, c1, c0, seed=615)).cuda())
    two = sqz.Index(H=H, d=d, L=L, c2=c2, dtype=g.dtype, C2=g.C2, N2=g.N2, key_off=g.key_off, perm=g.perm,
                    c1=c1, C1=g.C1, N1=g.N1, child_off=g.child_off)
    Q = sqz.to_device(synth.decode_queries(fc.mix, B, seed=616))
    scale = 1.0 / np.sqrt(d)
    for T, T1 in ((1e-4, 2e-4), (3e-5, 0.0)):
        a = sqz.centroid_lookup(g, Q, scale, T, T1, T0=0.0)
        b = sqz.centroid_lookup(two, Q, scale, T, T1)
        torch.cuda.synchronize()
        assert torch.equal(a.n_clusters, b.n_clusters) and torch.equal(a.n_keys, b.n_keys)
        for bb in range(B):
            for h in range(H):
                n = int(a.n_clusters[bb, h])
                assert torch.equal(a.clusters[bb, h, :n], b.clusters[bb, h, :n])
