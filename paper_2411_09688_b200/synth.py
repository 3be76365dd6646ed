"""Seeded synthetic workload generator ``SYN-MIX v1`` ("Input recipe").

This module holds NO arithmetic of the method: it only draws random inputs
(fixed-context K/V as a clustered mixture, queries, user KV, the K-means
initial subset) and rounds them once to the storage dtype.  It is the one
module both the CUDA path's harness and the CPU oracle's tests consume.

Stand-in for the paper's PG-19-derived KV: keys are a mixture of
directions so that clustering is meaningful (north star), cluster sizes are
uneven (Dirichlet weights), and per-head query sharpness varies to imitate the
flat vs skewed heads of App. A.

Storage convention: bf16 as ``np.uint16`` bit patterns, fp32 as ``np.float32``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

F32, BF16 = 0, 1


def to_storage(x: np.ndarray, dtype: int) -> np.ndarray:
    """Round fp32 values once to the storage dtype (round-to-nearest-even)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == F32:
        return f
    bits = f.view(np.uint32).astype(np.uint64)
    rounded = (bits + 0x7FFF + ((bits >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def storage_to_f32(a: np.ndarray) -> np.ndarray:
    """Decode stored bits back to fp32 (bf16 is a prefix of fp32)."""
    a = np.asarray(a)
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32)
    return a.astype(np.float32)


def _unit(rng, shape):
    u = rng.standard_normal(shape, dtype=np.float32)
    return u / np.linalg.norm(u, axis=-1, keepdims=True)


@dataclass
class Mixture:
    """Per-head generating mixture: directions u[H,G,d], weights pi[H,G], sharpness beta[H]."""
    u: np.ndarray
    pi: np.ndarray
    beta: np.ndarray
    rho: float
    sigma: float


@dataclass
class FixedContext:
    K: np.ndarray        # [H,L,d] storage
    V: np.ndarray        # [H,L,d] storage
    labels: np.ndarray   # [H,L] generating component of each key
    mix: Mixture
    dtype: int


def fixed_context(H, L, d, G, dtype=BF16, seed=1000, rho=4.0, sigma=None, sep=False,
                  G1=0, beta_range=(0.5, 2.5)):
    """Fixed-context K/V drawn as a clustered mixture (SYN-MIX v1).

    Keys k = rho * u_g + sigma * eps with g ~ Categorical(pi), pi ~ Dirichlet(1),
    sigma = rho / (2 sqrt d) by default (clustered but overlapping); the parity
    variant ``sep`` uses rho / (10 sqrt d).  With ``G1 > 0`` the G directions are
    grouped under G1 super-directions: u_g = normalize(u_super(g % G1) + 0.5 u_rand),
    so a 2-level hierarchy exists in the data.  Values ~ N(0, 1)."""
    rng = np.random.default_rng(seed)
    if sigma is None:
        sigma = rho / ((10.0 if sep else 2.0) * np.sqrt(d))
    if G1 > 0:
        sup = _unit(rng, (H, G1, d))
        u = sup[:, np.arange(G) % G1, :] + 0.5 * _unit(rng, (H, G, d))
        u = (u / np.linalg.norm(u, axis=-1, keepdims=True)).astype(np.float32)
    else:
        u = _unit(rng, (H, G, d))
    pi = rng.dirichlet(np.ones(G), size=H).astype(np.float64)
    lo, hi = np.log(beta_range[0]), np.log(beta_range[1])
    beta = np.exp(rng.uniform(lo, hi, size=H)).astype(np.float32)
    labels = np.empty((H, L), np.int32)
    K = np.empty((H, L, d), np.float32)
    for h in range(H):
        labels[h] = rng.choice(G, size=L, p=pi[h])
        K[h] = rho * u[h][labels[h]] + sigma * rng.standard_normal((L, d), dtype=np.float32)
    V = rng.standard_normal((H, L, d), dtype=np.float32)
    mix = Mixture(u=u, pi=pi, beta=beta, rho=rho, sigma=float(sigma))
    return FixedContext(K=to_storage(K, dtype), V=to_storage(V, dtype), labels=labels, mix=mix,
                        dtype=dtype)


def decode_queries(mix: Mixture, B, seed=4000, dtype=BF16, n=1):
    """Decode queries Q[B,H,n,d]: q = beta_h sqrt(d) normalize(u_g1 + u_g2 + 0.3 xi)
    with two "topics" g1, g2 ~ pi (per head)."""
    rng = np.random.default_rng(seed)
    H, G, d = mix.u.shape
    Q = np.empty((B, H, n, d), np.float32)
    for b in range(B):
        for h in range(H):
            for t in range(n):
                g = rng.choice(G, size=2, p=mix.pi[h])
                v = mix.u[h, g[0]] + mix.u[h, g[1]] + 0.3 * _unit(rng, (d,))
                Q[b, h, t] = mix.beta[h] * np.sqrt(d) * v / np.linalg.norm(v)
    return to_storage(Q, dtype)


def prefill_queries(mix: Mixture, B, n_q, seed=4000, dtype=BF16):
    """Prefill queries Q[B,H,n_q,d]: the n_q tokens of one user input share 2-4
    topics (so the averaged selection stays sparse), each token
    q = beta_h sqrt(d) normalize(u_topic + 0.5 xi)."""
    rng = np.random.default_rng(seed)
    H, G, d = mix.u.shape
    Q = np.empty((B, H, n_q, d), np.float32)
    for b in range(B):
        for h in range(H):
            nt = int(rng.integers(2, 5))
            topics = rng.choice(G, size=nt, p=mix.pi[h])
            pick = topics[rng.integers(0, nt, size=n_q)]
            v = mix.u[h][pick] + 0.5 * _unit(rng, (n_q, d))
            v /= np.linalg.norm(v, axis=-1, keepdims=True)
            Q[b, h] = mix.beta[h] * np.sqrt(d) * v
    return to_storage(Q, dtype)


def user_kv(mix: Mixture, B, n_u, seed=5000, dtype=BF16):
    """User-input K/V [B,H,n_u,d]: keys from the same mixture, values N(0,1)."""
    rng = np.random.default_rng(seed)
    H, G, d = mix.u.shape
    Ku = np.empty((B, H, n_u, d), np.float32)
    for b in range(B):
        for h in range(H):
            g = rng.choice(G, size=n_u, p=mix.pi[h])
            Ku[b, h] = mix.rho * mix.u[h][g] + mix.sigma * rng.standard_normal((n_u, d),
                                                                               dtype=np.float32)
    Vu = rng.standard_normal((B, H, n_u, d), dtype=np.float32)
    return to_storage(Ku, dtype), to_storage(Vu, dtype)


def kmeans_init(H, n, c, seed=2000):
    """Seeded initial subset for K-means (R3): c distinct point indices per head."""
    rng = np.random.default_rng(seed)
    return np.stack([rng.choice(n, size=c, replace=False) for _ in range(H)]).astype(np.int64)


def centroid_counts(L, frac_fine=0.05, frac_coarse=0.01):
    """Centroid counts ceil(frac * L)."""
    return int(np.ceil(frac_coarse * L)), int(np.ceil(frac_fine * L))


# --------------------------------------------------------------------------
# Device-side SYN-MIX v1 (same recipe, torch Philox on the GPU) for the large
# configurations (128K-1M keys x 32 heads), where host generation would take
# minutes.  Not bit-identical to the numpy generator above (different RNG);
# the parity tests use the host generator, the benches at 128K+ this one.
# Every per-head draw uses its own generator seeded by (seed, head), so a rank
# holding a subset of the heads draws exactly the bits the full run draws for
# them: inputs do not change with the number of GPUs.
# --------------------------------------------------------------------------
def _head_gen(seed, h, device):
    import torch

    return torch.Generator(device=device).manual_seed(int(seed) * 1000003 + int(h))

@dataclass
class DeviceMixture:
    u: "torch.Tensor"      # [H,G,d] fp32 unit directions
    pi: "torch.Tensor"     # [H,G] fp32 weights
    beta: "torch.Tensor"   # [H] fp32 sharpness
    rho: float
    sigma: float


def _torch_storage(x, dtype):
    import torch

    return x.to(torch.bfloat16 if dtype == BF16 else torch.float32)


def device_mixture(H, G, d, G1=0, seed=1000, device="cuda", rho=4.0, beta_range=(0.5, 2.5)):
    """The generating mixture of fixed_context(), drawn on the device."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    unit = lambda *s: torch.nn.functional.normalize(torch.randn(*s, generator=g, device=device), dim=-1)
    if G1 > 0:
        sup = unit(H, G1, d)
        u = torch.nn.functional.normalize(sup[:, torch.arange(G, device=device) % G1] + 0.5 * unit(H, G, d),
                                          dim=-1)
    else:
        u = unit(H, G, d)
    e = -torch.log(torch.rand(H, G, generator=g, device=device).clamp_min(1e-30))  # Dirichlet(1)
    pi = e / e.sum(-1, keepdim=True)
    lo, hi = np.log(beta_range[0]), np.log(beta_range[1])
    beta = torch.exp(lo + (hi - lo) * torch.rand(H, generator=g, device=device))
    return DeviceMixture(u=u, pi=pi, beta=beta, rho=rho, sigma=rho / (2.0 * np.sqrt(d)))


def device_keys(mix: DeviceMixture, L, seed, dtype=BF16, heads=None):
    """K, V [len(heads), L, d] storage dtype on the mixture's device."""
    import torch

    dev = mix.u.device
    heads = range(mix.u.shape[0]) if heads is None else heads
    d = mix.u.shape[2]
    K = torch.empty(len(heads), L, d, dtype=torch.bfloat16 if dtype == BF16 else torch.float32, device=dev)
    V = torch.empty_like(K)
    for i, h in enumerate(heads):
        g = _head_gen(seed, h, dev)
        lab = torch.multinomial(mix.pi[h], L, replacement=True, generator=g)
        K[i] = _torch_storage(mix.rho * mix.u[h][lab] + mix.sigma * torch.randn(L, d, generator=g, device=dev),
                              dtype)
        V[i] = _torch_storage(torch.randn(L, d, generator=g, device=dev), dtype)
    return K, V


def device_decode_queries(mix: DeviceMixture, B, seed, dtype=BF16, heads=None):
    """decode_queries() on the device: Q [B, len(heads), 1, d]."""
    import torch

    dev = mix.u.device
    heads = range(mix.u.shape[0]) if heads is None else heads
    d = mix.u.shape[2]
    Q = torch.empty(B, len(heads), 1, d, device=dev)
    for i, h in enumerate(heads):
        g = _head_gen(seed, h, dev)
        tp = torch.multinomial(mix.pi[h], 2 * B, replacement=True, generator=g).view(B, 2)
        xi = torch.nn.functional.normalize(torch.randn(B, d, generator=g, device=dev), dim=-1)
        v = mix.u[h][tp[:, 0]] + mix.u[h][tp[:, 1]] + 0.3 * xi
        Q[:, i, 0] = mix.beta[h] * np.sqrt(d) * torch.nn.functional.normalize(v, dim=-1)
    return _torch_storage(Q, dtype)


def device_prefill_queries(mix: DeviceMixture, B, n_q, seed, dtype=BF16, heads=None):
    """prefill_queries() on the device: Q [B, len(heads), n_q, d]."""
    import torch

    dev = mix.u.device
    heads = range(mix.u.shape[0]) if heads is None else heads
    d = mix.u.shape[2]
    Q = torch.empty(B, len(heads), n_q, d, device=dev)
    for i, h in enumerate(heads):
        g = _head_gen(seed, h, dev)
        for b in range(B):
            nt = int(torch.randint(2, 5, (1,), generator=g, device=dev))
            topics = torch.multinomial(mix.pi[h], nt, replacement=True, generator=g)
            pick = topics[torch.randint(0, nt, (n_q,), generator=g, device=dev)]
            xi = torch.nn.functional.normalize(torch.randn(n_q, d, generator=g, device=dev), dim=-1)
            v = torch.nn.functional.normalize(mix.u[h][pick] + 0.5 * xi, dim=-1)
            Q[b, i] = mix.beta[h] * np.sqrt(d) * v
    return _torch_storage(Q, dtype)


def device_user_kv(mix: DeviceMixture, B, n_u, seed, dtype=BF16, heads=None):
    """user_kv() on the device: Ku, Vu [B, len(heads), n_u, d]."""
    import torch

    dev = mix.u.device
    heads = range(mix.u.shape[0]) if heads is None else heads
    d = mix.u.shape[2]
    Ku = torch.empty(B, len(heads), n_u, d, device=dev)
    Vu = torch.empty(B, len(heads), n_u, d, device=dev)
    for i, h in enumerate(heads):
        g = _head_gen(seed, h, dev)
        for b in range(B):
            lab = torch.multinomial(mix.pi[h], n_u, replacement=True, generator=g)
            Ku[b, i] = mix.rho * mix.u[h][lab] + mix.sigma * torch.randn(n_u, d, generator=g, device=dev)
            Vu[b, i] = torch.randn(n_u, d, generator=g, device=dev)
    return _torch_storage(Ku, dtype), _torch_storage(Vu, dtype)


def device_kmeans_init(H, n, c, seed, device="cuda", heads=None):
    """kmeans_init() on the device: [len(heads), c] int64 distinct indices per head."""
    import torch

    heads = range(H) if heads is None else heads
    return torch.stack([torch.randperm(n, generator=_head_gen(seed, h, device), device=device)[:c]
                        for h in heads])
