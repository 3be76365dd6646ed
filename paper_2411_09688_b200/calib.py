"""Global-threshold calibration (harness; App. C).

The paper picks ONE threshold T "to achieve the desired sparsity level" and keeps
it for prefill and generation; calibration uses 100 tokens at the end of
the fixed context, here 100 extra queries from the same generator (R17).
T is the N-weighted quantile of the calibration scores S_i (or S-bar_i): the
value at which the expected retained key fraction equals `retention`, placed at
the midpoint between the two adjacent distinct scores.  The Level-1
threshold T1 is the same quantile on S^(1) with N^(1) weights at retention 0.5
("50% of the keys would be ruled out").

Host-side logic over scores the CUDA lookup produced (sqz_selection.dbg_S).
"""
from __future__ import annotations

import numpy as np


def weighted_threshold(S, N, retention: float, total_weight: float = None) -> float:
    """S: [..., c] scores (NaN = not scanned, ignored), N: broadcastable [..., c]
    key counts.  Returns T with sum_{S > T} N / W ~= retention, where W is
    `total_weight` (default: the weight of the scanned rows; pass the number of
    keys x query-rows when Level-1 pruning left rows unscanned)."""
    S = np.asarray(S, dtype=np.float64)
    W = np.broadcast_to(np.asarray(N, dtype=np.float64), S.shape)
    m = ~np.isnan(S)
    s, w = S[m], W[m]
    if retention >= 1.0:
        return 0.0
    if retention <= 0.0:
        return float(s.max()) * 2.0
    order = np.argsort(-s, kind="stable")
    s, w = s[order], w[order]
    cum = np.cumsum(w) / (w.sum() if total_weight is None else float(total_weight))
    k = int(np.searchsorted(cum, retention))  # first index reaching the target
    k = min(k, len(s) - 1)
    hi = s[k]
    lower = s[k + 1:]
    lower = lower[lower < hi]
    lo = lower[0] if len(lower) else 0.0
    return float(0.5 * (hi + lo))


def distributed_threshold(S, N, retention: float, total_weight: float, allreduce=None,
                          iters: int = 80) -> float:
    """The same calibration when the scores are spread over ranks (head or
    cluster shards): bisection on log T of the global retained weight
    sum_{S > T} N (NaN = not scanned), each probe summed over the ranks by
    `allreduce` (float -> float; identity on one process), so every rank gets
    the identical T.  S, N: torch tensors (any device), N broadcastable to S."""
    import torch

    if retention >= 1.0:
        return 0.0
    S = S.double()
    W = torch.broadcast_to(N.double(), S.shape)
    ok = ~torch.isnan(S)
    S, W = S[ok], W[ok]
    red = allreduce or (lambda x: x)
    target = retention * float(total_weight)
    lo, hi = np.log(1e-30), np.log(2.0)  # retained(lo) >= target >= retained(hi)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        kept = red(float(W[S > np.exp(mid)].sum()))
        if kept > target:
            lo = mid
        else:
            hi = mid
    return float(np.exp(0.5 * (lo + hi)))
