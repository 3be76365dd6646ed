"""Pins for the oracle's masked attention and merge (section 4.2).

The independent library routine is torch fp64 softmax(QK^T*scale + mask) V and
torch.logsumexp; special cases come from SPEC."""
import numpy as np
import pytest
import torch

import oracle


def _torch_ref(Q, K, V, mask, Ku, Vu, causal, scale):
    B, H, nq, d = Q.shape
    out_O = np.zeros((B, H, nq, d))
    out_L = np.zeros((B, H, nq))
    n_u = 0 if Ku is None else Ku.shape[2]
    for b in range(B):
        for h in range(H):
            keys = [torch.tensor(K[h])]
            vals = [torch.tensor(V[h])]
            m = [torch.tensor(mask[b, h]) if mask is not None else torch.ones(K.shape[1], dtype=torch.bool)]
            m = m[0].unsqueeze(0).expand(nq, -1)
            if n_u:
                keys.append(torch.tensor(Ku[b, h]))
                vals.append(torch.tensor(Vu[b, h]))
                if causal:
                    t = torch.arange(nq).unsqueeze(1)
                    u = torch.arange(n_u).unsqueeze(0)
                    mu = u <= t + n_u - nq
                else:
                    mu = torch.ones(nq, n_u, dtype=torch.bool)
                m = torch.cat([m, mu], dim=1)
            Kc = torch.cat(keys)
            Vc = torch.cat(vals)
            z = (torch.tensor(Q[b, h]) @ Kc.T) * scale
            z = z.masked_fill(~m, float("-inf"))
            out_L[b, h] = torch.logsumexp(z, dim=1).numpy()
            out_O[b, h] = (torch.softmax(z, dim=1) @ Vc).numpy()
    return out_O, out_L


@pytest.mark.parametrize("causal", [False, True])
def test_matches_torch_fp64(causal):
    rng = np.random.default_rng(20)
    B, H, nq, d, L, nu = 2, 3, 5, 16, 37, 6
    Q = rng.standard_normal((B, H, nq, d))
    K = rng.standard_normal((H, L, d))
    V = rng.standard_normal((H, L, d))
    Ku = rng.standard_normal((B, H, nu, d))
    Vu = rng.standard_normal((B, H, nu, d))
    mask = rng.random((B, H, L)) < 0.4
    O, LSE, rc = oracle.attention(Q, K, V, mask, Ku, Vu, causal, 0.25)
    assert rc == 0
    Ot, Lt = _torch_ref(Q, K, V, mask, Ku, Vu, causal, 0.25)
    np.testing.assert_allclose(O, Ot, atol=1e-12)
    np.testing.assert_allclose(LSE, Lt, atol=1e-12)


def test_special_cases():
    rng = np.random.default_rng(21)
    d = 8
    q = rng.standard_normal((1, 1, 1, d))
    # L = 1 -> v
    K = rng.standard_normal((1, 1, d))
    V = rng.standard_normal((1, 1, d))
    O, LSE, _ = oracle.attention(q, K, V)
    np.testing.assert_allclose(O[0, 0, 0], V[0, 0], atol=1e-15)
    assert LSE[0, 0, 0] == pytest.approx(float(q[0, 0, 0] @ K[0, 0]) / np.sqrt(d), rel=1e-14)
    # identical keys -> mean of values
    K = np.tile(rng.standard_normal(d), (1, 9, 1))
    V = rng.standard_normal((1, 9, d))
    O, _, _ = oracle.attention(q, K, V)
    np.testing.assert_allclose(O[0, 0, 0], V[0].mean(0), atol=1e-14)
    # single selected key -> its value
    K = rng.standard_normal((1, 9, d))
    mask = np.zeros((1, 1, 9), bool)
    mask[0, 0, 4] = True
    O, _, _ = oracle.attention(q, K, V, mask)
    np.testing.assert_allclose(O[0, 0, 0], V[0, 4], atol=1e-15)
    # full selection == dense
    O1, L1, _ = oracle.attention(q, K, V, np.ones((1, 1, 9), bool))
    O2, L2, _ = oracle.attention(q, K, V, None)
    np.testing.assert_array_equal(O1, O2)
    # empty selection -> identity partial and error code 7
    O, LSE, rc = oracle.attention(q, K, V, np.zeros((1, 1, 9), bool))
    assert rc == 7 and np.isneginf(LSE).all() and not O.any()


def test_causal_edges():
    """R8: query t (of n_q) sees user keys u <= t + n_u - n_q; the first query of a prompt
    with n_u = n_q sees exactly one user key."""
    rng = np.random.default_rng(22)
    d, nq = 4, 3
    Q = rng.standard_normal((1, 1, nq, d))
    K = np.zeros((1, 0, d))
    V = np.zeros((1, 0, d))
    Ku = rng.standard_normal((1, 1, nq, d))
    Vu = rng.standard_normal((1, 1, nq, d))
    O, _, rc = oracle.attention(Q, K, V, None, Ku, Vu, causal=True)
    assert rc == 0
    np.testing.assert_allclose(O[0, 0, 0], Vu[0, 0, 0], atol=1e-15)
    # qpos / n_q_total select a row of a longer prompt
    Osub, _, _ = oracle.attention(Q[:, :, 2:], K, V, None, Ku, Vu, True, qpos=[2], n_q_total=nq)
    np.testing.assert_allclose(Osub[0, 0, 0], O[0, 0, 2], atol=1e-15)


@pytest.mark.parametrize("block", [1, 7, 128])
def test_block_partition_and_merge_invariance(block):
    """S:357 / S:378-380: partials over any block partition, merged in any order, equal the
    whole; merge(a, identity) = a."""
    rng = np.random.default_rng(23)
    d, L = 16, 300
    q = rng.standard_normal((1, 1, 1, d)) * 2
    K = rng.standard_normal((1, L, d))
    V = rng.standard_normal((1, L, d))
    Ow, Lw, _ = oracle.attention(q, K, V)
    Os, Ls = [], []
    for s in range(0, L, block):
        m = np.zeros((1, 1, L), bool)
        m[..., s:s + block] = True
        O, LSE, _ = oracle.attention(q, K, V, m)
        Os.append(O.reshape(1, d))
        Ls.append(LSE.reshape(1))
    order = rng.permutation(len(Os))
    Om, Lm = oracle.merge(np.stack(Os)[order], np.stack(Ls)[order])
    np.testing.assert_allclose(Om[0], Ow[0, 0, 0], atol=1e-12)
    assert Lm[0] == pytest.approx(Lw[0, 0, 0], abs=1e-12)
    Oi, Li = oracle.merge(np.stack([Os[0], np.zeros_like(Os[0])]),
                          np.stack([Ls[0], np.array([-np.inf])]))
    np.testing.assert_array_equal(Oi, Os[0])
    np.testing.assert_array_equal(Li, Ls[0])


def test_dropped_mass_error_bound():
    """||sparse - dense||_inf <= 2 * dropped_mass * max|v|."""
    rng = np.random.default_rng(24)
    d, L = 8, 64
    for trial in range(50):
        q = rng.standard_normal((1, 1, 1, d)) * 3
        K = rng.standard_normal((1, L, d))
        V = rng.standard_normal((1, L, d))
        mask = rng.random((1, 1, L)) < rng.uniform(0.1, 0.95)
        mask[0, 0, 0] = True
        Od, _, _ = oracle.attention(q, K, V)
        Os, _, _ = oracle.attention(q, K, V, mask)
        z = (K[0] @ q[0, 0, 0]) / np.sqrt(d)
        a = np.exp(z - z.max())
        a /= a.sum()
        dropped = a[~mask[0, 0]].sum()
        assert np.abs(Os - Od).max() <= 2 * dropped * np.abs(V).max() + 1e-12
