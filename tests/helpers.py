"""Shared test helpers: build seeded problems, move oracle tables to the GPU, and
compare selections under the near-threshold band rule (parity)."""
import numpy as np

import oracle
from paper_2411_09688_b200 import synth


def oracle_problem(H, L, d, c2, c1=0, dtype=synth.BF16, seed=100, G=None, B=1, n_u=0, n_q=1,
                   prefill=False, sep=False, max_iters=50):
    G = G or c2
    fc = synth.fixed_context(H, L, d, G, dtype=dtype, seed=seed, sep=sep, G1=c1 if c1 else 0)
    init2 = synth.kmeans_init(H, L, c2, seed=seed + 1)
    init1 = synth.kmeans_init(H, c2, c1, seed=seed + 2) if c1 else None
    idx = oracle.build_index(fc.K, c2, init2, c1, init1, max_iters=max_iters)
    if prefill:
        Q = synth.prefill_queries(fc.mix, B, n_q, seed=seed + 3, dtype=dtype)
    else:
        Q = synth.decode_queries(fc.mix, B, seed=seed + 3, dtype=dtype, n=n_q)
    Ku = Vu = None
    if n_u:
        Ku, Vu = synth.user_kv(fc.mix, B, n_u, seed=seed + 4, dtype=dtype)
    return dict(fc=fc, idx=idx, Q=Q, Ku=Ku, Vu=Vu, init2=init2, init1=init1, dtype=dtype)


def gpu_index(idx: "oracle.Index", device="cuda"):
    import torch

    from paper_2411_09688_b200 import sqz

    def dev_i32(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)

    def dev_c(a):
        return sqz.to_device(oracle.encode(a, idx.dtype), device)

    g = sqz.Index(H=idx.H, d=idx.d, L=idx.L, c2=idx.c2, dtype=idx.dtype, C2=dev_c(idx.C2),
                  N2=dev_i32(idx.N2), key_off=dev_i32(idx.key_off), perm=dev_i32(idx.perm))
    if idx.levels == 2:
        g.c1 = idx.c1
        g.C1 = dev_c(idx.C1)
        g.N1 = dev_i32(idx.N1)
        g.child_off = dev_i32(idx.child_off)
    return g


def gpu_sets(sel, B, H, c):
    """GPU selection -> bool [B,H,c] of selected finest-level clusters, checking that the
    cluster lists are ascending."""
    cl = sel.clusters.cpu().numpy()
    n = sel.n_clusters.cpu().numpy()
    out = np.zeros((B, H, c), bool)
    for b in range(B):
        for h in range(H):
            lst = cl[b, h, :n[b, h]]
            assert np.all(np.diff(lst) > 0), "cluster list not ascending"
            out[b, h, lst] = True
    return out


def assert_selection_parity(gpu_sel, ref_sel, ref_S, T, rel=1e-5, what="selection"):
    """Selected cluster sets must be identical except clusters whose oracle score lies
    within rel*T of T (north star)."""
    diff = gpu_sel != ref_sel
    band = oracle.band(ref_S, T, rel)
    bad = diff & ~band
    assert not bad.any(), (f"{what}: {int(bad.sum())} clusters differ outside the band "
                           f"(first at {np.argwhere(bad)[:3].tolist()})")
    return int(diff.sum())


def key_mask_from_gpu(sel, idx: "oracle.Index", B, H):
    """GPU key_idx (cluster-major positions) -> bool [B,H,L] in ORIGINAL key order."""
    ki = sel.key_idx.cpu().numpy()
    nk = sel.n_keys.cpu().numpy()
    m = np.zeros((B, H, idx.L), bool)
    for b in range(B):
        for h in range(H):
            pos = ki[b, h, :nk[b, h]]
            assert np.all(np.diff(pos) > 0), "key_idx not ascending"
            m[b, h, idx.perm[h][pos]] = True
    return m


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
