"""Thin ctypes binding of libsqz.so (include/sqz.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  PyTorch supplies device memory and the current stream.  There is
no CPU fallback -- if libsqz.so is missing or the device is not sm_100, calls
raise.

The raw entry points keep the C names (``sqz_centroid_lookup`` ...); the
snake-case helpers below (``cluster_keys``, ``centroid_lookup``,
``sparse_attention``, ``merge_partials``) allocate outputs / workspaces as
torch tensors and call them.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libsqz.so")

SQZ_F32, SQZ_BF16 = 0, 1
SQZ_OK, SQZ_ERR_INVALID_ARG, SQZ_ERR_FORMAT, SQZ_ERR_INVARIANT = 0, 2, 3, 4
SQZ_ERR_CUDA, SQZ_ERR_NCCL, SQZ_ERR_EMPTY, SQZ_ERR_UNSUPPORTED = 5, 6, 7, 8
ABI_VERSION = 6

EXPORTS = [
    "sqz_cluster_keys_workspace", "sqz_cluster_keys", "sqz_index_validate_workspace",
    "sqz_index_validate", "sqz_lookup_workspace", "sqz_centroid_lookup",
    "sqz_attention_workspace", "sqz_sparse_attention", "sqz_attention_status",
    "sqz_merge_partials", "sqz_workspace_init", "sqz_last_error", "sqz_abi_version",
    "sqz_device_check", "sqz_centroid_lookup_stage", "sqz_shard_plan_compute", "sqz_index_shard",
    "sqz_comm_unique_id", "sqz_comm_init", "sqz_comm_destroy", "sqz_lookup_workspace_comm",
    "sqz_comm_merge_workspace", "sqz_comm_allgather_merge", "sqz_decode_step_workspace",
    "sqz_decode_step", "sqz_selection_diagnostics_workspace", "sqz_selection_diagnostics",
    "sqz_comm_alltoall_merge_workspace", "sqz_comm_alltoall_merge",
    "sqz_index_save", "sqz_index_file_info", "sqz_index_load",
]


class sqz_index(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int32), ("d", ctypes.c_int32), ("L", ctypes.c_int64),
                ("levels", ctypes.c_int32), ("c1", ctypes.c_int32), ("c2", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("C1", ctypes.c_void_p), ("N1", ctypes.c_void_p),
                ("child_off", ctypes.c_void_p), ("C2", ctypes.c_void_p), ("N2", ctypes.c_void_p),
                ("key_off", ctypes.c_void_p), ("perm", ctypes.c_void_p),
                ("L_total", ctypes.c_int64), ("c0", ctypes.c_int32), ("C0", ctypes.c_void_p),
                ("N0", ctypes.c_void_p), ("child_off0", ctypes.c_void_p)]


class sqz_shard_plan(ctypes.Structure):
    _fields_ = [("c1", ctypes.c_int32), ("c2", ctypes.c_int32), ("L", ctypes.c_int64)] + [
        (n, ctypes.c_void_p) for n in ("c1_src", "c2_src", "key_src", "N1", "child_off", "N2",
                                       "key_off")]


class sqz_kmeans_params(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int32), ("tol", ctypes.c_float), ("assign_mode", ctypes.c_int32),
                ("init0", ctypes.c_void_p)]


KMEANS_AUTO, KMEANS_EXACT, KMEANS_TENSOR = 0, 1, 2


class sqz_lookup_params(ctypes.Structure):
    _fields_ = [("scale", ctypes.c_float), ("T", ctypes.c_float), ("T1", ctypes.c_float),
                ("comm", ctypes.c_void_p), ("T0", ctypes.c_float)]


class sqz_selection(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("clusters", "n_clusters", "n_keys", "key_idx", "l1_surv", "dbg_S", "dbg_S1",
                 "dbg_lse", "key_pref", "l0_surv", "dbg_S0")]


class sqz_attn_params(ctypes.Structure):
    _fields_ = [("scale", ctypes.c_float), ("causal", ctypes.c_int32), ("partial", ctypes.c_int32),
                ("out_dtype", ctypes.c_int32), ("per_row", ctypes.c_int32)]


class sqz_diagnostics(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("skew", "mass_sel", "mass_ideal", "recall", "n_T", "mass_T")]


class SqzError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libsqz error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libsqz.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise RuntimeError(f"{SO} is missing: build it with __graft_entry__.build(); "
                               "there is no CPU fallback")
        L = ctypes.CDLL(SO)
        vp, sz, szp = ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        ip = ctypes.POINTER(sqz_index)
        L.sqz_last_error.restype = ctypes.c_char_p
        L.sqz_cluster_keys_workspace.argtypes = [ip, szp]
        L.sqz_cluster_keys.argtypes = [vp, vp, vp, vp, ip, vp, vp,
                                       ctypes.POINTER(sqz_kmeans_params), vp, sz,
                                       ctypes.POINTER(ctypes.c_int32), vp]
        L.sqz_index_validate_workspace.argtypes = [ip, szp]
        L.sqz_index_validate.argtypes = [ip, vp, sz, vp]
        L.sqz_index_save.argtypes = [ip, ctypes.c_char_p, vp]
        L.sqz_index_file_info.argtypes = [ctypes.c_char_p, ip]
        L.sqz_index_load.argtypes = [ctypes.c_char_p, ip, vp]
        L.sqz_lookup_workspace.argtypes = [ip, i32, i32, szp]
        L.sqz_centroid_lookup.argtypes = [ip, vp, i32, i32, ctypes.POINTER(sqz_lookup_params),
                                          ctypes.POINTER(sqz_selection), vp, sz, vp]
        L.sqz_attention_workspace.argtypes = [ip, i32, i32, i32, szp]
        L.sqz_sparse_attention.argtypes = [vp, i32, i32, vp, vp, ip,
                                           ctypes.POINTER(sqz_selection), vp, vp, i32,
                                           ctypes.POINTER(sqz_attn_params), vp, vp, vp, sz, vp]
        L.sqz_attention_status.argtypes = [vp, sz, vp]
        L.sqz_merge_partials.argtypes = [i32, vp, vp, i64, i32, vp, vp, i32, vp]
        L.sqz_workspace_init.argtypes = [vp, sz, vp]
        L.sqz_centroid_lookup_stage.argtypes = [ip, vp, i32, i32, ctypes.POINTER(sqz_lookup_params),
                                                i32, i32, vp, vp, ctypes.POINTER(sqz_selection), vp,
                                                sz, vp]
        L.sqz_shard_plan_compute.argtypes = [i32, i32, i32, i32, i64, vp, vp, i32, i32,
                                             ctypes.POINTER(sqz_shard_plan)]
        L.sqz_index_shard.argtypes = [ip, vp, vp, vp, vp, vp, ip, vp, vp, vp]
        L.sqz_comm_unique_id.argtypes = [ctypes.c_char_p]
        L.sqz_comm_init.argtypes = [ctypes.c_char_p, i32, i32, ctypes.POINTER(ctypes.c_void_p)]
        L.sqz_comm_destroy.argtypes = [vp]
        L.sqz_lookup_workspace_comm.argtypes = [ip, i32, i32, i32, szp]
        L.sqz_comm_merge_workspace.argtypes = [i32, i64, i32, szp]
        L.sqz_comm_allgather_merge.argtypes = [vp, vp, vp, i64, i32, vp, vp, i32, vp, sz, vp]
        L.sqz_decode_step_workspace.argtypes = [ip, i32, i32, szp]
        L.sqz_decode_step.argtypes = [ip, vp, i32, vp, vp, vp, vp, i32,
                                      ctypes.POINTER(sqz_lookup_params),
                                      ctypes.POINTER(sqz_attn_params), ctypes.POINTER(sqz_selection),
                                      vp, vp, vp, sz, vp]
        L.sqz_comm_alltoall_merge_workspace.argtypes = [i32, i32, i32, i32, i32, szp]
        L.sqz_comm_alltoall_merge.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp, vp, i32, vp, sz, vp]
        L.sqz_selection_diagnostics_workspace.argtypes = [ip, i32, szp]
        L.sqz_selection_diagnostics.argtypes = [ip, vp, i32, vp, ctypes.POINTER(sqz_selection),
                                                ctypes.c_float, ctypes.c_double, ctypes.c_float,
                                                ctypes.POINTER(sqz_diagnostics), vp, sz, vp]
        if L.sqz_abi_version() != ABI_VERSION:
            raise RuntimeError(f"{SO} has ABI {L.sqz_abi_version()}, binding expects {ABI_VERSION}: "
                               "rebuild with __graft_entry__.build()")
        for n in EXPORTS:
            getattr(L, n).restype = ctypes.c_char_p if n == "sqz_last_error" else ctypes.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != SQZ_OK:
        raise SqzError(rc, lib().sqz_last_error().decode())


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def torch_dtype(dt):
    return torch.bfloat16 if dt == SQZ_BF16 else torch.float32


def sqz_dtype(t: torch.Tensor):
    if t.dtype == torch.bfloat16:
        return SQZ_BF16
    if t.dtype == torch.float32:
        return SQZ_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def to_device(stored: np.ndarray, device="cuda") -> torch.Tensor:
    """Storage-convention numpy array (bf16 bits as uint16, or fp32) -> device tensor."""
    a = np.ascontiguousarray(stored)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(a).to(device)


def workspace(nbytes: int, device="cuda") -> torch.Tensor:
    ws = torch.zeros(max(int(nbytes), 512), dtype=torch.uint8, device=device)
    return ws


# --------------------------------------------------------------------------
@dataclass
class Index:
    """Device-resident index tables (include/sqz.h, sqz_index)."""
    H: int
    d: int
    L: int
    c2: int
    dtype: int
    C2: torch.Tensor
    N2: torch.Tensor
    key_off: torch.Tensor
    perm: torch.Tensor
    c1: int = 0
    C1: torch.Tensor = None
    N1: torch.Tensor = None
    child_off: torch.Tensor = None
    L_total: int = 0          # > 0: a fixed-context shard (see shard_index)
    c2_src: torch.Tensor = None  # shard: global Level-2 id of each local row (-1 = padding)
    c1_src: torch.Tensor = None  # shard: global Level-1 id of each local row
    c0: int = 0                  # three levels: Level 0 above Level 1
    C0: torch.Tensor = None
    N0: torch.Tensor = None
    child_off0: torch.Tensor = None

    @property
    def levels(self):
        return 3 if self.c0 > 0 else (2 if self.c1 > 0 else 1)

    def struct(self) -> sqz_index:
        s = sqz_index()
        s.H, s.d, s.L, s.levels, s.c1, s.c2, s.dtype = (self.H, self.d, self.L, self.levels,
                                                        self.c1, self.c2, self.dtype)
        for f in ("C1", "N1", "child_off", "C2", "N2", "key_off", "perm", "C0", "N0", "child_off0"):
            t = getattr(self, f)
            setattr(s, f, None if t is None else t.data_ptr())
        s.L_total = self.L_total
        s.c0 = self.c0
        return s

    @staticmethod
    def empty(H, d, L, c2, c1=0, dtype=SQZ_BF16, device="cuda", c0=0):
        td = torch_dtype(dtype)
        i32 = dict(dtype=torch.int32, device=device)
        return Index(H=H, d=d, L=L, c2=c2, dtype=dtype,
                     C2=torch.empty(H, c2, d, dtype=td, device=device),
                     N2=torch.empty(H, c2, **i32), key_off=torch.empty(H, c2 + 1, **i32),
                     perm=torch.empty(H, L, **i32), c1=c1,
                     C1=torch.empty(H, c1, d, dtype=td, device=device) if c1 else None,
                     N1=torch.empty(H, c1, **i32) if c1 else None,
                     child_off=torch.empty(H, c1 + 1, **i32) if c1 else None, c0=c0,
                     C0=torch.empty(H, c0, d, dtype=td, device=device) if c0 else None,
                     N0=torch.empty(H, c0, **i32) if c0 else None,
                     child_off0=torch.empty(H, c0 + 1, **i32) if c0 else None)


def cluster_keys(K: torch.Tensor, V: torch.Tensor, c2: int, init2: torch.Tensor, c1: int = 0,
                 init1: torch.Tensor = None, max_iters: int = 50, tol: float = 1e-4,
                 assign_mode: int = KMEANS_AUTO, c0: int = 0, init0: torch.Tensor = None):
    """sqz_cluster_keys: returns (Index, Kp, Vp, (iters_level2, iters_level1)).
    assign_mode: KMEANS_EXACT (fp32 FFMA scores), KMEANS_TENSOR (split-bf16
    tcgen05 GEMM + exact re-rank of near ties) or KMEANS_AUTO."""
    H, L, d = K.shape
    idx = Index.empty(H, d, L, c2, c1, sqz_dtype(K), K.device, c0=c0)
    s = idx.struct()
    nb = ctypes.c_size_t(0)
    _check(lib().sqz_cluster_keys_workspace(ctypes.byref(s), ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=K.device)
    Kp = torch.empty_like(K)
    Vp = torch.empty_like(V)
    it = (ctypes.c_int32 * 3)()
    i2 = init2.to(device=K.device, dtype=torch.int64).contiguous()
    i1 = None if init1 is None else init1.to(device=K.device, dtype=torch.int64).contiguous()
    i0 = None if init0 is None else init0.to(device=K.device, dtype=torch.int64).contiguous()
    p = sqz_kmeans_params(max_iters, tol, assign_mode, None if i0 is None else i0.data_ptr())
    _check(lib().sqz_cluster_keys(_p(K), _p(V), _p(i2), _p(i1), ctypes.byref(s), _p(Kp), _p(Vp),
                                  ctypes.byref(p), _p(ws), nb.value, it, _stream()))
    return idx, Kp, Vp, ((it[0], it[1], it[2]) if c0 else (it[0], it[1]))


def index_validate(idx: Index):
    s = idx.struct()
    nb = ctypes.c_size_t(0)
    _check(lib().sqz_index_validate_workspace(ctypes.byref(s), ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=idx.C2.device)
    _check(lib().sqz_index_validate(ctypes.byref(s), _p(ws), nb.value, _stream()))


def save_index(idx: Index, path: str):
    """sqz_index_save: write the index tables to `path` (SQZIDX1 file)."""
    s = idx.struct()
    _check(lib().sqz_index_save(ctypes.byref(s), os.fsencode(path), _stream()))


def index_file_info(path: str) -> sqz_index:
    """sqz_index_file_info: the geometry recorded in a SQZIDX1 file (host only)."""
    g = sqz_index()
    _check(lib().sqz_index_file_info(os.fsencode(path), ctypes.byref(g)))
    return g


def load_index(path: str, device="cuda", validate: bool = True) -> Index:
    """sqz_index_load into freshly allocated device tables (then sqz_index_validate)."""
    g = index_file_info(path)
    idx = Index.empty(g.H, g.d, g.L, g.c2, g.c1 if g.levels >= 2 else 0, g.dtype, device,
                      c0=g.c0 if g.levels == 3 else 0)
    idx.L_total = g.L_total
    s = idx.struct()
    _check(lib().sqz_index_load(os.fsencode(path), ctypes.byref(s), _stream()))
    if validate:
        index_validate(idx)
    return idx


@dataclass
class Selection:
    clusters: torch.Tensor
    n_clusters: torch.Tensor
    n_keys: torch.Tensor
    key_idx: torch.Tensor          # optional expanded key positions (None: runs only)
    l1_surv: torch.Tensor = None
    dbg_S: torch.Tensor = None
    dbg_S1: torch.Tensor = None
    dbg_lse: torch.Tensor = None
    key_pref: torch.Tensor = None  # run-length key offsets of the selected clusters
    l0_surv: torch.Tensor = None   # three levels: Level-0 survivors (debug)
    dbg_S0: torch.Tensor = None

    @staticmethod
    def empty(idx: Index, B, n_q, debug=False, device="cuda", key_idx=True):
        """Output buffers of a lookup.  key_idx=False leaves the selection in its
        run-length form (clusters + key_pref), which sqz_sparse_attention reads
        directly; True also materialises the expanded key positions."""
        i32 = dict(dtype=torch.int32, device=device)
        f32 = dict(dtype=torch.float32, device=device)
        H = idx.H
        return Selection(
            clusters=torch.empty(B, H, idx.c2, **i32), n_clusters=torch.empty(B, H, **i32),
            n_keys=torch.empty(B, H, **i32),
            key_idx=torch.empty(B, H, idx.L, **i32) if key_idx else None,
            key_pref=torch.empty(B, H, idx.c2, **i32),
            l1_surv=torch.empty(B, H, idx.c1, dtype=torch.uint8, device=device)
            if (debug and idx.c1) else None,
            dbg_S=torch.empty(B, H, idx.c2, **f32) if debug else None,
            dbg_S1=torch.empty(B, H, idx.c1, **f32) if (debug and idx.c1) else None,
            dbg_lse=torch.empty(B, H, n_q, **f32) if debug else None,
            l0_surv=torch.empty(B, H, idx.c0, dtype=torch.uint8, device=device)
            if (debug and idx.c0) else None,
            dbg_S0=torch.empty(B, H, idx.c0, **f32) if (debug and idx.c0) else None)

    def struct(self) -> sqz_selection:
        s = sqz_selection()
        for f, _ in sqz_selection._fields_:
            t = getattr(self, f)
            setattr(s, f, None if t is None else t.data_ptr())
        return s


class Workspaces:
    """Cached zero-initialised workspaces, one per call geometry (the library
    leaves a workspace re-usable by later calls with the same geometry)."""

    def __init__(self):
        self._ws = {}
        self.last_attn = None

    def get(self, key, nbytes, device):
        t = self._ws.get(key)
        if t is None or t.numel() < nbytes:
            t = workspace(nbytes, device)
            self._ws[key] = t
        return t


_WS = Workspaces()


def lookup_workspace_bytes(idx: Index, B, n_q):
    s = idx.struct()
    nb = ctypes.c_size_t(0)
    _check(lib().sqz_lookup_workspace(ctypes.byref(s), B, n_q, ctypes.byref(nb)))
    return nb.value


def attention_workspace_bytes(idx: Index, B, n_q, n_u):
    s = idx.struct()
    nb = ctypes.c_size_t(0)
    _check(lib().sqz_attention_workspace(ctypes.byref(s), B, n_q, n_u, ctypes.byref(nb)))
    return nb.value


def centroid_lookup(idx: Index, Q: torch.Tensor, scale: float, T: float, T1: float = 0.0,
                    sel: Selection = None, ws: torch.Tensor = None, debug=False,
                    comm: "Comm" = None, T0: float = 0.0) -> Selection:
    """sqz_centroid_lookup on Q[B,H,n_q,d].  `comm`: idx is this rank's
    fixed-context shard; the lookup exchanges the per-level statistics."""
    B, H, n_q, d = Q.shape
    if sel is None:
        sel = Selection.empty(idx, B, n_q, debug, Q.device)
    s = idx.struct()
    if ws is None:
        if comm is None:
            nb = lookup_workspace_bytes(idx, B, n_q)
        else:
            nbc = ctypes.c_size_t(0)
            _check(lib().sqz_lookup_workspace_comm(ctypes.byref(s), B, n_q, comm.world,
                                                   ctypes.byref(nbc)))
            nb = nbc.value
        ws = _WS.get(("lookup", Q.device, idx.H, idx.L, idx.c0, idx.c1, idx.c2, B, n_q,
                      0 if comm is None else comm.world), nb, Q.device)
    p = sqz_lookup_params(scale, T, T1, None if comm is None else comm.handle, T0)
    ss = sel.struct()
    _check(lib().sqz_centroid_lookup(ctypes.byref(s), _p(Q), B, n_q, ctypes.byref(p),
                                     ctypes.byref(ss), _p(ws), ws.numel(), _stream()))
    return sel


def sparse_attention(Q, Kp, Vp, idx: Index, sel: Selection, Ku=None, Vu=None, scale=None,
                     causal=False, partial=False, out_dtype=None, O=None, LSE=None, ws=None,
                     per_row=False):
    """sqz_sparse_attention: returns (O[B,H,n_q,d], LSE[B,H,n_q]).  per_row=True
    disables the batch-shared decode pass (one key stream per (b,h))."""
    B, H, n_q, d = Q.shape
    n_u = 0 if Ku is None else Ku.shape[2]
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))
    if out_dtype is None:
        out_dtype = idx.dtype
    if O is None:
        O = torch.empty(B, H, n_q, d, dtype=torch_dtype(out_dtype), device=Q.device)
    if LSE is None:
        LSE = torch.empty(B, H, n_q, dtype=torch.float32, device=Q.device)
    s = idx.struct()
    if ws is None:
        ws = _WS.get(("attn", Q.device, idx.H, idx.L, B, n_q, n_u),
                     attention_workspace_bytes(idx, B, n_q, n_u), Q.device)
        _WS.last_attn = ws
    p = sqz_attn_params(scale, int(causal), int(partial), out_dtype, int(per_row))
    ss = sel.struct()
    _check(lib().sqz_sparse_attention(_p(Q), B, n_q, _p(Kp), _p(Vp), ctypes.byref(s),
                                      ctypes.byref(ss), _p(Ku), _p(Vu), n_u, ctypes.byref(p),
                                      _p(O), _p(LSE), _p(ws), ws.numel(), _stream()))
    return O, LSE


def decode_step(idx: Index, Q, Kp, Vp, Ku, Vu, scale, T, T1=0.0, sel: Selection = None,
                partial=False, out_dtype=None, O=None, LSE=None, ws=None, debug=False, T0=0.0):
    """sqz_decode_step: the centroid lookup and the sparse attention of one decode
    step (Q [B,H,1,d]) in one call.  Returns (Selection, O [B,H,1,d], LSE [B,H,1])."""
    B, H, n_q, d = Q.shape
    if n_q != 1:
        raise ValueError("decode_step takes one query row per (b, h)")
    n_u = 0 if Ku is None else Ku.shape[2]
    if sel is None:
        sel = Selection.empty(idx, B, 1, debug, Q.device)
    if out_dtype is None:
        out_dtype = idx.dtype
    if O is None:
        O = torch.empty(B, H, 1, d, dtype=torch_dtype(out_dtype), device=Q.device)
    if LSE is None:
        LSE = torch.empty(B, H, 1, dtype=torch.float32, device=Q.device)
    s = idx.struct()
    if ws is None:
        nb = ctypes.c_size_t(0)
        _check(lib().sqz_decode_step_workspace(ctypes.byref(s), B, n_u, ctypes.byref(nb)))
        ws = _WS.get(("step", Q.device, idx.H, idx.L, idx.c1, idx.c2, B, n_u), nb.value, Q.device)
        _WS.last_attn = ws
    lp = sqz_lookup_params(scale, T, T1, None, T0)
    ap = sqz_attn_params(scale, 0, int(partial), out_dtype)
    ss = sel.struct()
    _check(lib().sqz_decode_step(ctypes.byref(s), _p(Q), B, _p(Kp), _p(Vp), _p(Ku), _p(Vu), n_u,
                                 ctypes.byref(lp), ctypes.byref(ap), ctypes.byref(ss), _p(O), _p(LSE),
                                 _p(ws), ws.numel(), _stream()))
    return sel, O, LSE


def attention_status(ws: torch.Tensor = None):
    """sqz_attention_status on `ws` (default: the workspace of the last
    sparse_attention call made through this module)."""
    if ws is None:
        ws = _WS.last_attn
    _check(lib().sqz_attention_status(_p(ws), ws.numel(), _stream()))


def merge_partials(O_parts: torch.Tensor, LSE_parts: torch.Tensor, out_dtype=SQZ_F32):
    """sqz_merge_partials: O_parts[P,rows,d] fp32, LSE_parts[P,rows] fp32."""
    P, rows, d = O_parts.shape
    O = torch.empty(rows, d, dtype=torch_dtype(out_dtype), device=O_parts.device)
    LSE = torch.empty(rows, dtype=torch.float32, device=O_parts.device)
    _check(lib().sqz_merge_partials(P, _p(O_parts.contiguous()), _p(LSE_parts.contiguous()), rows,
                                    d, _p(O), _p(LSE), out_dtype, _stream()))
    return O, LSE


def device_check():
    _check(lib().sqz_device_check())


# --------------------------------------------------------------------------
# multi-GPU: fixed-context sharding by cluster
# --------------------------------------------------------------------------
def centroid_lookup_stage(idx: Index, Q, scale, T, T1, stage, stats_in, stats_out, sel: Selection,
                          ws: torch.Tensor):
    """sqz_centroid_lookup_stage: one stage of the sharded lookup (the caller
    exchanges the statistics between stages).  stats_in [P,B,H,n_q,2] fp32 or
    None (stage 0); stats_out [B,H,n_q,2] fp32 or None (last stage)."""
    B, H, n_q, d = Q.shape
    s = idx.struct()
    p = sqz_lookup_params(scale, T, T1, None)
    P = 0 if stats_in is None else stats_in.shape[0]
    ss = sel.struct()
    _check(lib().sqz_centroid_lookup_stage(ctypes.byref(s), _p(Q), B, n_q, ctypes.byref(p), stage,
                                           P, _p(stats_in), _p(stats_out), ctypes.byref(ss),
                                           _p(ws), ws.numel(), _stream()))


def shard_plan(H, levels, c1, c2, L, key_off: np.ndarray, child_off: np.ndarray, rank, world):
    """sqz_shard_plan_compute (host only): the rank's share of the clusters
    (Level-1 / single-level cluster p -> rank p mod world).  Returns a dict of
    numpy arrays: c1, c2, L and c1_src, c2_src, key_src, N1, child_off, N2,
    key_off of the shard."""
    ko = np.ascontiguousarray(key_off, dtype=np.int32)
    co = None if child_off is None else np.ascontiguousarray(child_off, dtype=np.int32)
    pl = sqz_shard_plan()
    cp = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)
    _check(lib().sqz_shard_plan_compute(H, levels, c1, c2, L, cp(ko), cp(co), rank, world,
                                        ctypes.byref(pl)))
    C1, C2, LL = pl.c1, pl.c2, pl.L
    out = dict(c1=C1, c2=C2, L=LL,
               c2_src=np.zeros((H, C2), np.int32), key_src=np.zeros((H, LL), np.int32),
               N2=np.zeros((H, C2), np.int32), key_off=np.zeros((H, C2 + 1), np.int32))
    if levels == 2:
        out.update(c1_src=np.zeros((H, C1), np.int32), N1=np.zeros((H, C1), np.int32),
                   child_off=np.zeros((H, C1 + 1), np.int32))
    for f in ("c1_src", "c2_src", "key_src", "N1", "child_off", "N2", "key_off"):
        setattr(pl, f, cp(out.get(f)))
    _check(lib().sqz_shard_plan_compute(H, levels, c1, c2, L, cp(ko), cp(co), rank, world,
                                        ctypes.byref(pl)))
    return out


def shard_index(idx: Index, Kp: torch.Tensor, Vp: torch.Tensor, rank: int, world: int):
    """This rank's fixed-context shard of a full index: (Index, Kp_local,
    Vp_local).  Offline step (copies the integer tables to the host once)."""
    dev = Kp.device
    plan = shard_plan(idx.H, idx.levels, idx.c1, idx.c2, idx.L, idx.key_off.cpu().numpy(),
                      None if idx.child_off is None else idx.child_off.cpu().numpy(), rank, world)
    td = torch_dtype(idx.dtype)
    up = lambda a: torch.from_numpy(a).to(dev)
    H, d = idx.H, idx.d
    loc = Index(H=H, d=d, L=plan["L"], c2=plan["c2"], dtype=idx.dtype,
                C2=torch.empty(H, plan["c2"], d, dtype=td, device=dev), N2=up(plan["N2"]),
                key_off=up(plan["key_off"]), perm=torch.empty(H, plan["L"], dtype=torch.int32,
                                                              device=dev),
                c1=plan["c1"], L_total=idx.L, c2_src=up(plan["c2_src"]),
                c1_src=up(plan["c1_src"]) if idx.levels == 2 else None)
    if idx.levels == 2:
        loc.C1 = torch.empty(H, plan["c1"], d, dtype=td, device=dev)
        loc.N1 = up(plan["N1"])
        loc.child_off = up(plan["child_off"])
    Kl = torch.empty(H, plan["L"], d, dtype=td, device=dev)
    Vl = torch.empty_like(Kl)
    c1s = loc.c1_src
    c2s, ks = loc.c2_src, up(plan["key_src"])
    sf, sl = idx.struct(), loc.struct()
    _check(lib().sqz_index_shard(ctypes.byref(sf), _p(Kp), _p(Vp), _p(c1s), _p(c2s), _p(ks),
                                 ctypes.byref(sl), _p(Kl), _p(Vl), _stream()))
    return loc, Kl, Vl


class Comm:
    """sqz_comm over the ranks of a torch.distributed process group (one
    process per GPU).  The NCCL unique id is created by rank 0 and broadcast
    through the process group (any backend)."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist

        self.rank, self.world = rank, world
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(lib().sqz_comm_unique_id(buf))
        t = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).clone()
        if world > 1:
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, 0, group=group)
        raw = bytes(t.cpu().numpy().tobytes())
        h = ctypes.c_void_p()
        _check(lib().sqz_comm_init(raw, rank, world, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            _check(lib().sqz_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def allgather_merge(comm: Comm, O_part: torch.Tensor, LSE_part: torch.Tensor, out_dtype=SQZ_BF16,
                    O=None, LSE=None, ws=None):
    """sqz_comm_allgather_merge: every rank's partial (O fp32 [..., d], LSE fp32
    [...]) -> the merged O (out_dtype) and LSE, identical on every rank."""
    d = O_part.shape[-1]
    rows = O_part.numel() // d
    if O is None:
        O = torch.empty(O_part.shape, dtype=torch_dtype(out_dtype), device=O_part.device)
    if LSE is None:
        LSE = torch.empty(LSE_part.shape, dtype=torch.float32, device=O_part.device)
    if ws is None:
        nb = ctypes.c_size_t(0)
        _check(lib().sqz_comm_merge_workspace(comm.world, rows, d, ctypes.byref(nb)))
        ws = _WS.get(("merge", O_part.device, comm.world, rows, d), nb.value, O_part.device)
    _check(lib().sqz_comm_allgather_merge(comm.handle, _p(O_part), _p(LSE_part), rows, d, _p(O),
                                          _p(LSE), out_dtype, _p(ws), ws.numel(), _stream()))
    return O, LSE


def selection_diagnostics(idx: Index, Q: torch.Tensor, Kp: torch.Tensor, sel: Selection, scale: float,
                          top_frac: float = 0.01, T: float = 0.0):
    """sqz_selection_diagnostics (App. A skewness, App. D ideal lookup) for one
    decode query per (b,h), Q [B,H,1,d].  Returns a dict of [B,H] tensors:
    skew, mass_sel, mass_ideal, recall, n_T, mass_T."""
    B = Q.shape[0]
    s = idx.struct()
    nb = ctypes.c_size_t(0)
    _check(lib().sqz_selection_diagnostics_workspace(ctypes.byref(s), B, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=Q.device)
    f32 = dict(dtype=torch.float32, device=Q.device)
    out = {k: torch.empty(B, idx.H, **f32) for k in ("skew", "mass_sel", "mass_ideal", "recall",
                                                     "mass_T")}
    out["n_T"] = torch.empty(B, idx.H, dtype=torch.int32, device=Q.device)
    d = sqz_diagnostics(*[out[k].data_ptr() for k, _ in sqz_diagnostics._fields_])
    ss = sel.struct()
    _check(lib().sqz_selection_diagnostics(ctypes.byref(s), _p(Q), B, _p(Kp), ctypes.byref(ss),
                                           float(scale), float(top_frac), float(T), ctypes.byref(d),
                                           _p(ws), nb.value, _stream()))
    return out


def alltoall_merge(comm: "Comm", O_part: torch.Tensor, LSE_part: torch.Tensor, out_dtype=SQZ_BF16,
                   O=None, LSE=None):
    """sqz_comm_alltoall_merge: partials O_part [B,H,n_q,d] fp32 / LSE_part [B,H,n_q]
    of this rank -> the merged output of this rank's head slice [B,H/world,n_q,d]."""
    B, H, n_q, d = O_part.shape
    Hs = H // comm.world
    if O is None:
        O = torch.empty(B, Hs, n_q, d, dtype=torch_dtype(out_dtype), device=O_part.device)
    if LSE is None:
        LSE = torch.empty(B, Hs, n_q, dtype=torch.float32, device=O_part.device)
    nb = ctypes.c_size_t(0)
    _check(lib().sqz_comm_alltoall_merge_workspace(comm.world, B, H, n_q, d, ctypes.byref(nb)))
    ws = _WS.get(("a2a", O_part.device, comm.world, B, H, n_q, d), nb.value, O_part.device)
    _check(lib().sqz_comm_alltoall_merge(comm.handle, _p(O_part), _p(LSE_part), B, H, n_q, d, _p(O),
                                         _p(LSE), out_dtype, _p(ws), ws.numel(), _stream()))
    return O, LSE
