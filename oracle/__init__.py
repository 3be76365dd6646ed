"""CPU oracle for Squeezed Attention (arXiv 2411.09688) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  It is a plain, slow,
fp64 implementation written from the paper (``sqzref.c`` holds the arithmetic;
this module only converts stored bits to fp64, calls it, and orchestrates the
index build in the order section 3.3 states).  It shares no code with
``paper_2411_09688_b200`` and never imports it.

Stored tensors use the project's storage convention: bf16 as ``np.uint16`` bit
patterns, fp32 as ``np.float32``.  Both are decoded to fp64 exactly.

Parity pins for every function live in ``tests/test_oracle_*.py``; the list of
readings (R1..R18) where the paper is silent is in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsqzref.so")
_lib = None

F32, BF16 = 0, 1


def build(force: bool = False) -> str:
    """Compile sqzref.c (plain gcc -O2, no fast-math) into libsqzref.so."""
    src = os.path.join(_HERE, "sqzref.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "sqzref.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-fopenmp", "-shared", src, "-o", _SO, "-lm"]
        )
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        dp, ip, i64p, u8p = (
            ctypes.POINTER(ctypes.c_double),
            ctypes.POINTER(ctypes.c_int32),
            ctypes.POINTER(ctypes.c_int64),
            ctypes.POINTER(ctypes.c_uint8),
        )
        c_int, c_i64, c_d = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.sqzref_round_bf16.restype = c_d
        L.sqzref_round_bf16.argtypes = [c_d]
        L.sqzref_round_array.argtypes = [dp, c_i64, c_int]
        L.sqzref_kmeans.restype = c_int
        L.sqzref_kmeans.argtypes = [dp, c_i64, c_int, c_int, i64p, c_int, c_d, ip, dp,
                                    ctypes.POINTER(c_int), dp]
        L.sqzref_cluster_means.argtypes = [dp, c_i64, c_int, c_int, ip, dp, ip]
        L.sqzref_build_order.restype = c_int
        L.sqzref_build_order.argtypes = [c_i64, c_int, ip, c_int, ip, ip, ip, ip, ip]
        L.sqzref_scores.argtypes = [dp, dp, ip, c_int, c_int, c_int, ip, c_d, dp, dp, dp]
        L.sqzref_select_singlepass.argtypes = [dp, ip, c_int, c_d, u8p]
        L.sqzref_lookup.restype = c_int
        L.sqzref_lookup.argtypes = [c_int, c_int, c_int, c_int, dp, c_int, c_int, dp, ip, ip,
                                    c_int, dp, ip, c_d, c_d, c_d, u8p, u8p, dp, u8p, dp, dp]
        L.sqzref_attention.restype = c_int
        L.sqzref_attention.argtypes = [c_int, c_int, c_int, c_int, c_i64, c_int, dp, dp, dp, u8p,
                                       dp, dp, c_int, c_int, ip, c_d, dp, dp]
        L.sqzref_merge.argtypes = [c_int, c_i64, c_int, dp, dp, dp, dp]
        vpp = ctypes.POINTER(ctypes.c_void_p)
        L.sqzref_lookup_ml.restype = c_int
        L.sqzref_lookup_ml.argtypes = [c_int, c_int, c_int, c_int, dp, c_int, ip, vpp, vpp, vpp, c_d,
                                       dp, vpp, vpp, vpp, dp]
        L.sqzref_diagnostics.restype = c_int
        L.sqzref_diagnostics.argtypes = [c_int, c_int, c_int, c_i64, dp, dp, u8p, c_d, c_i64, c_d,
                                         dp, dp, dp, dp, i64p, i64p, dp]
        _lib = L
    return _lib


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ct))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# --------------------------------------------------------------------------
# stored bits <-> fp64 (exact)
# --------------------------------------------------------------------------

def to_f64(stored: np.ndarray) -> np.ndarray:
    """Exact fp64 value of stored bf16 bits (uint16) or fp32 values."""
    a = np.asarray(stored)
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if a.dtype == np.float32:
        return a.astype(np.float64)
    if a.dtype == np.float64:
        return a.copy()
    raise TypeError(f"unsupported storage dtype {a.dtype}")


def round_to(x: np.ndarray, dtype: int) -> np.ndarray:
    """Round fp64 values once, to nearest-even, to bf16 or fp32 (R18)."""
    y = _f64(x).copy()
    lib().sqzref_round_array(_p(y, ctypes.c_double), y.size, dtype)
    return y


def encode(x_rounded: np.ndarray, dtype: int) -> np.ndarray:
    """Storage bits of already-rounded fp64 values (exact, no rounding)."""
    f = np.asarray(x_rounded, dtype=np.float64).astype(np.float32)
    if dtype == F32:
        return f
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def dtype_of(stored: np.ndarray) -> int:
    return BF16 if np.asarray(stored).dtype == np.uint16 else F32


# --------------------------------------------------------------------------
# offline index (section 3.1, section 3.3)
# --------------------------------------------------------------------------

def kmeans(X, c, init, max_iters=50, tol=1e-4):
    """Lloyd K-means on unit-normalised rows of X (R3).

    Returns (assign[n] int32, mu[c,d] normalised-space centroids, iters,
    objective[iters])."""
    X = _f64(X)
    n, d = X.shape
    init = np.ascontiguousarray(init, dtype=np.int64)
    assign = np.zeros(n, np.int32)
    mu = np.zeros((c, d), np.float64)
    obj = np.zeros(max(max_iters, 1), np.float64)
    iters = ctypes.c_int(0)
    rc = lib().sqzref_kmeans(_p(X, ctypes.c_double), n, d, c, _p(init, ctypes.c_int64), max_iters,
                             tol, _p(assign, ctypes.c_int32), _p(mu, ctypes.c_double),
                             ctypes.byref(iters), _p(obj, ctypes.c_double))
    if rc != 0:
        raise ValueError(f"sqzref_kmeans: error {rc}")
    return assign, mu, iters.value, obj[: iters.value]


def cluster_means(X, assign, c):
    """C_i = mean of raw member rows, N_i = member count (R2)."""
    X = _f64(X)
    n, d = X.shape
    a = _i32(assign)
    C = np.zeros((c, d), np.float64)
    N = np.zeros(c, np.int32)
    lib().sqzref_cluster_means(_p(X, ctypes.c_double), n, d, c, _p(a, ctypes.c_int32),
                               _p(C, ctypes.c_double), _p(N, ctypes.c_int32))
    return C, N


@dataclass
class Index:
    """Per-head index tables in the cluster-major layout (layout)."""
    levels: int
    dtype: int
    H: int
    L: int
    d: int
    c2: int
    C2: np.ndarray           # [H,c2,d] fp64, values exactly representable in `dtype`
    N2: np.ndarray           # [H,c2] int32
    key_off: np.ndarray      # [H,c2+1] int32
    perm: np.ndarray         # [H,L] int32: permuted position -> original key index
    c1: int = 0
    C1: np.ndarray = None    # [H,c1,d]
    N1: np.ndarray = None    # [H,c1] descendant keys (R4)
    child_off: np.ndarray = None  # [H,c1+1]
    assign2: np.ndarray = None    # [H,L] new level-2 id of every original key
    iters: list = field(default_factory=list)
    c0: int = 0                   # three levels: Level 0 above Level 1
    C0: np.ndarray = None         # [H,c0,d]
    N0: np.ndarray = None         # [H,c0] descendant keys (R4)
    child_off0: np.ndarray = None  # [H,c0+1] Level-1 children of each Level-0 cluster


def build_index(K_stored, c2, init2, c1=0, init1=None, max_iters=50, tol=1e-4, c0=0, init0=None):
    """Offline clustering of the fixed-context keys of every head.

    Level 2 = K-means(keys, c2); Level 1 = K-means(Level-2 centroids, c1)
    ("clustered into coarser-grained Level 1 centroids by repeating the same
    procedure").  C^(1) = unweighted mean of the child
    C^(2) rows (R5); N^(1) = descendant keys (R4).  Centroids are rounded once
    to the storage dtype (R18).  Keys are then ordered cluster-major (Level-2
    grouped by parent, keys by Level-2 cluster, both stable).
    c0 > 0: a third level ("extended to multiple levels"): Level 0 =
    K-means(Level-1 centroids, c0) by the same procedure, C^(0) = unweighted mean
    of the child C^(1) rows, N^(0) = descendant keys; Level-1 ids are then grouped
    by their Level-0 parent (stable in K-means id) before the Level-2 ids are
    grouped by their (renumbered) Level-1 parent."""
    dt = dtype_of(K_stored)
    K = to_f64(K_stored)
    H, L, d = K.shape
    levels = 3 if c0 > 0 else (2 if c1 > 0 else 1)
    if c0 > 0 and c1 <= 0:
        raise ValueError("three levels need c1 > 0")
    C0 = np.zeros((H, c0, d)) if levels == 3 else None
    N0 = np.zeros((H, c0), np.int32) if levels == 3 else None
    child_off0 = np.zeros((H, c0 + 1), np.int32) if levels == 3 else None
    C2o = np.zeros((H, c2, d))
    N2o = np.zeros((H, c2), np.int32)
    key_off = np.zeros((H, c2 + 1), np.int32)
    perm = np.zeros((H, L), np.int32)
    assign_new = np.zeros((H, L), np.int32)
    C1 = np.zeros((H, c1, d)) if levels >= 2 else None
    N1 = np.zeros((H, c1), np.int32) if levels >= 2 else None
    child_off = np.zeros((H, c1 + 1), np.int32) if levels >= 2 else None
    iters = []
    for h in range(H):
        a2, _, it2, _ = kmeans(K[h], c2, init2[h], max_iters, tol)
        C2, N2 = cluster_means(K[h], a2, c2)
        C2 = round_to(C2, dt)
        parent = None
        it1 = it0 = 0
        if levels >= 2:
            parent, _, it1, _ = kmeans(C2, c1, init1[h], max_iters, tol)
            C1h, _ = cluster_means(C2, parent, c1)
            C1h = round_to(C1h, dt)
            N1h = np.zeros(c1, np.int32)
            for o in range(c2):
                N1h[parent[o]] += N2[o]
            if levels == 3:
                # Level 0 on the stored Level-1 rows; Level-1 ids grouped by parent
                parent0, _, it0, _ = kmeans(C1h, c0, init0[h], max_iters, tol)
                C0h, _ = cluster_means(C1h, parent0, c0)
                C0[h] = round_to(C0h, dt)
                l1_order = [p for g in range(c0) for p in range(c1) if parent0[p] == g]
                new1 = np.empty(c1, np.int32)
                new1[l1_order] = np.arange(c1, dtype=np.int32)
                for g in range(c0):
                    child_off0[h, g + 1] = child_off0[h, g] + int((parent0 == g).sum())
                    N0[h, g] = int(N1h[parent0 == g].sum())
                C1h = C1h[l1_order]
                N1h = N1h[l1_order]
                parent = new1[parent]
            C1[h] = C1h
            N1[h] = N1h
        l2_order = np.zeros(c2, np.int32)
        coff = np.zeros(c1 + 1, np.int32)
        rc = lib().sqzref_build_order(
            L, c2, _p(_i32(a2), ctypes.c_int32), c1,
            _p(_i32(parent), ctypes.c_int32) if parent is not None else None,
            _p(l2_order, ctypes.c_int32), _p(perm[h], ctypes.c_int32),
            _p(key_off[h], ctypes.c_int32), _p(coff, ctypes.c_int32))
        if rc != 0:
            raise ValueError(f"sqzref_build_order: error {rc}")
        if levels >= 2:
            child_off[h] = coff
        C2o[h] = C2[l2_order]
        N2o[h] = N2[l2_order]
        new_of_old = np.empty(c2, np.int32)
        new_of_old[l2_order] = np.arange(c2, dtype=np.int32)
        assign_new[h] = new_of_old[a2]
        iters.append((it2, it1, it0) if levels == 3 else (it2, it1))
    return Index(levels=levels, dtype=dt, H=H, L=L, d=d, c2=c2, C2=C2o, N2=N2o, key_off=key_off,
                 perm=perm, c1=c1, C1=C1, N1=N1, child_off=child_off, assign2=assign_new,
                 iters=iters, c0=c0, C0=C0, N0=N0, child_off0=child_off0)


def permute_kv(X_stored, idx: Index):
    """Cluster-major copy: Xp[h, pos] = X[h, perm[h, pos]] (D1)."""
    X = np.asarray(X_stored)
    return np.stack([X[h][idx.perm[h]] for h in range(X.shape[0])])


# --------------------------------------------------------------------------
# online lookup (Eq. 1-3; prefill averaging P:330-335)
# --------------------------------------------------------------------------

def scores(q, C, N, scale, rows=None):
    """Eq. 1 (or Eq. 3 when `rows` restricts the denominator): returns (s, S, lse)."""
    q = _f64(q)
    C = _f64(C)
    N = _i32(N)
    c, d = C.shape
    s = np.full(c, np.nan)
    S = np.full(c, np.nan)
    lse = ctypes.c_double(0.0)
    r = None if rows is None else _i32(rows)
    lib().sqzref_scores(_p(q, ctypes.c_double), _p(C, ctypes.c_double), _p(N, ctypes.c_int32), d,
                        c, 0 if r is None else len(r), _p(r, ctypes.c_int32), scale,
                        _p(s, ctypes.c_double), _p(S, ctypes.c_double), ctypes.byref(lse))
    return s, S, lse.value


def select_singlepass(s, N, T):
    """Generation single-pass selection, e_i = exp(s_i - m) > D*T."""
    s = _f64(s)
    N = _i32(N)
    sel = np.zeros(len(s), np.uint8)
    lib().sqzref_select_singlepass(_p(s, ctypes.c_double), _p(N, ctypes.c_int32), len(s), T,
                                   _p(sel, ctypes.c_uint8))
    return sel.astype(bool)


def lookup_ml(Q, idx: Index, scale, T, T1=0.0, T0=0.0, forced_l1=None, forced_l0=None):
    """Multi-level lookup for a three-level index: Level 0 (all rows,
    Eq. 2) -> Level 1 over the survivors' children (Eq. 3) -> Level 2 likewise.
    Returns sel2/Sbar2, surv1/Sbar1, surv0/Sbar0, lse as lookup() does."""
    Q = _f64(Q)
    B, H, n_q, d = Q.shape
    Lv = idx.levels
    tabs = ([(idx.C0, idx.N0, idx.child_off0, idx.c0)] if Lv == 3 else []) + \
        ([(idx.C1, idx.N1, idx.child_off, idx.c1)] if Lv >= 2 else []) + [(idx.C2, idx.N2, None, idx.c2)]
    keep = []
    c = np.array([t[3] for t in tabs], np.int32)
    Cs = [_f64(t[0]) for t in tabs]
    Ns = [_i32(t[1]) for t in tabs]
    Os = [None if t[2] is None else _i32(t[2]) for t in tabs]
    Ts = np.array(([T0] if Lv == 3 else []) + ([T1] if Lv >= 2 else []) + [T], np.float64)
    forced = ([forced_l0] if Lv == 3 else []) + ([forced_l1] if Lv >= 2 else []) + [None]
    forced = [None if f is None else np.ascontiguousarray(f, dtype=np.uint8) for f in forced]
    surv = [np.zeros((B, H, ci), np.uint8) for ci in c]
    Sbar = [np.zeros((B, H, ci)) for ci in c]
    lse = np.zeros((B, H, n_q))
    keep += Cs + Ns + Os + forced + surv + Sbar

    def ptrs(arrs):
        a = (ctypes.c_void_p * len(arrs))(*[None if x is None else x.ctypes.data for x in arrs])
        keep.append(a)
        return ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))

    rc = lib().sqzref_lookup_ml(B, H, n_q, d, _p(Q, ctypes.c_double), Lv, _p(c, ctypes.c_int32),
                                ptrs(Cs), ptrs(Ns), ptrs(Os), scale, _p(Ts, ctypes.c_double),
                                ptrs(forced), ptrs(surv), ptrs(Sbar), _p(lse, ctypes.c_double))
    if rc != 0:
        raise ValueError(f"sqzref_lookup_ml: error {rc}")
    out = dict(sel2=surv[-1].astype(bool), Sbar2=Sbar[-1], lse=lse)
    if Lv >= 2:
        out["surv1"] = surv[-2].astype(bool)
        out["Sbar1"] = Sbar[-2]
    if Lv == 3:
        out["surv0"] = surv[0].astype(bool)
        out["Sbar0"] = Sbar[0]
    return out


def lookup(Q, idx: Index, scale, T, T1=0.0, forced_l1=None, T0=0.0, forced_l0=None):
    """Centroid lookup for Q[B,H,n_q,d] (decode: n_q = 1; prefill: averaged)."""
    if idx.levels == 3:
        return lookup_ml(Q, idx, scale, T, T1, T0, forced_l1, forced_l0)
    Q = _f64(Q)
    B, H, n_q, d = Q.shape
    c1, c2 = idx.c1, idx.c2
    sel2 = np.zeros((B, H, c2), np.uint8)
    Sbar2 = np.zeros((B, H, c2))
    surv1 = np.zeros((B, H, max(c1, 1)), np.uint8)
    Sbar1 = np.zeros((B, H, max(c1, 1)))
    lse = np.zeros((B, H, n_q))
    f = None if forced_l1 is None else np.ascontiguousarray(forced_l1, dtype=np.uint8)
    C1 = _f64(idx.C1) if idx.levels == 2 else None
    N1 = _i32(idx.N1) if idx.levels == 2 else None
    co = _i32(idx.child_off) if idx.levels == 2 else None
    C2 = _f64(idx.C2)
    N2 = _i32(idx.N2)
    rc = lib().sqzref_lookup(
        B, H, n_q, d, _p(Q, ctypes.c_double), idx.levels, c1, _p(C1, ctypes.c_double),
        _p(N1, ctypes.c_int32), _p(co, ctypes.c_int32), c2, _p(C2, ctypes.c_double),
        _p(N2, ctypes.c_int32), scale, T, T1, _p(f, ctypes.c_uint8), _p(sel2, ctypes.c_uint8),
        _p(Sbar2, ctypes.c_double), _p(surv1, ctypes.c_uint8), _p(Sbar1, ctypes.c_double),
        _p(lse, ctypes.c_double))
    if rc != 0:
        raise ValueError(f"sqzref_lookup: error {rc}")
    out = dict(sel2=sel2.astype(bool), Sbar2=Sbar2, lse=lse)
    if idx.levels == 2:
        out["surv1"] = surv1.astype(bool)
        out["Sbar1"] = Sbar1
    return out


def keymask(idx: Index, sel2):
    """Selected key set in ORIGINAL key indices: union of the members of the
    selected finest-level clusters.  Returns bool [B,H,L]."""
    sel2 = np.asarray(sel2, bool)
    B, H, _ = sel2.shape
    m = np.zeros((B, H, idx.L), bool)
    for b in range(B):
        for h in range(H):
            m[b, h] = sel2[b, h][idx.assign2[h]]
    return m


def band(Sbar, T, rel=1e-5):
    """Clusters inside the near-threshold band |S - T| <= rel*T (DESIGN.md parity rule)."""
    Sbar = np.asarray(Sbar)
    if T == 0:
        return np.zeros(Sbar.shape, bool)
    with np.errstate(invalid="ignore"):
        return np.abs(Sbar - T) <= rel * T


# --------------------------------------------------------------------------
# attention (section 4.2) and merge
# --------------------------------------------------------------------------

def attention(Q, K, V, mask=None, Ku=None, Vu=None, causal=False, scale=None, qpos=None,
              n_q_total=None):
    """Exact masked attention: Q[B,H,n_q,d], K/V[H,L,d] (original order),
    mask[B,H,L] bool or None, Ku/Vu[B,H,n_u,d].  Returns (O, LSE, rc)."""
    Q = _f64(Q)
    B, H, n_q, d = Q.shape
    K = _f64(K)
    V = _f64(V)
    L = K.shape[1]
    n_u = 0 if Ku is None else Ku.shape[2]
    Ku = None if Ku is None else _f64(Ku)
    Vu = None if Vu is None else _f64(Vu)
    mk = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    qp = None if qpos is None else _i32(qpos)
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    O = np.zeros((B, H, n_q, d))
    LSE = np.zeros((B, H, n_q))
    rc = lib().sqzref_attention(
        B, H, n_q, d, L, n_u, _p(Q, ctypes.c_double), _p(K, ctypes.c_double),
        _p(V, ctypes.c_double), _p(mk, ctypes.c_uint8), _p(Ku, ctypes.c_double),
        _p(Vu, ctypes.c_double), int(bool(causal)), n_q if n_q_total is None else n_q_total,
        _p(qp, ctypes.c_int32), scale, _p(O, ctypes.c_double), _p(LSE, ctypes.c_double))
    return O, LSE, rc


def merge(O_parts, LSE_parts):
    """Merge P partials O_parts[P,rows,d], LSE_parts[P,rows]."""
    O_parts = _f64(O_parts)
    LSE_parts = _f64(LSE_parts)
    P, rows, d = O_parts.shape
    O = np.zeros((rows, d))
    LSE = np.zeros(rows)
    lib().sqzref_merge(P, rows, d, _p(O_parts, ctypes.c_double), _p(LSE_parts, ctypes.c_double),
                       _p(O, ctypes.c_double), _p(LSE, ctypes.c_double))
    return O, LSE


def budget(k_selected, L, scanned_per_level=()):
    """KV budget (App. C, Table 2 caption P:414): fraction of KV
    loaded, counting centroid rows (key-only) at half weight:
    k/L + sum_l scanned_l / (2L)."""
    return k_selected / L + sum(scanned_per_level) / (2.0 * L)


# --------------------------------------------------------------------------
# selection diagnostics: App. A skewness, App. D ideal lookup (NEXT-4)
# --------------------------------------------------------------------------

def top_count(top_frac, L):
    """n_top = ceil(top_frac * L), at least 1 ("top 1%" of P:710)."""
    return max(1, int(np.ceil(float(top_frac) * L)))


def diagnostics(Q, K, sel, scale, top_frac=0.01, T=0.0):
    """Per (b,h) of one decode query row: App. A top-`top_frac` cumulative
    attention score, and the App. D ideal lookup (keys with a_j > T; and the
    k largest a_j at the centroid selection's budget k) vs the selection.
    Q[B,H,d] or [B,H,1,d]; K[H,L,d] original order; sel[B,H,L] bool (original
    order).  Returns a dict of [B,H] arrays (see sqzref_diagnostics)."""
    Q = _f64(Q)
    if Q.ndim == 4:
        Q = np.ascontiguousarray(Q[:, :, 0])
    B, H, d = Q.shape
    K = _f64(K)
    L = K.shape[1]
    sm = np.ascontiguousarray(sel, dtype=np.uint8)
    out = {k: np.zeros((B, H)) for k in ("skew", "mass_sel", "mass_ideal", "recall", "mass_T")}
    ks = np.zeros((B, H), np.int64)
    nT = np.zeros((B, H), np.int64)
    rc = lib().sqzref_diagnostics(
        B, H, d, L, _p(Q, ctypes.c_double), _p(K, ctypes.c_double), _p(sm, ctypes.c_uint8),
        float(scale), top_count(top_frac, L), float(T), _p(out["skew"], ctypes.c_double),
        _p(out["mass_sel"], ctypes.c_double), _p(out["mass_ideal"], ctypes.c_double),
        _p(out["recall"], ctypes.c_double), _p(ks, ctypes.c_int64), _p(nT, ctypes.c_int64),
        _p(out["mass_T"], ctypes.c_double))
    if rc:
        raise ValueError(f"sqzref_diagnostics rc={rc}")
    out["k"] = ks
    out["n_T"] = nT
    return out
