"""The C-ABI library loads and exports every symbol include/sqz.h declares; the ctypes
struct layouts match the C header; host-side argument checks work without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sqz.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sqz_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2411_09688_b200 import build, sqz

    build.build()
    return sqz.lib()


def test_exports_every_declared_symbol(lib):
    from paper_2411_09688_b200 import sqz

    decl = _declared()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(sqz.EXPORTS) == decl
    assert lib.sqz_abi_version() == sqz.ABI_VERSION == 6


def test_struct_layout_matches_header(tmp_path):
    from paper_2411_09688_b200 import sqz

    prog = tmp_path / "lay.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "sqz.h"\n'
                    "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(sqz_index),"
                    " offsetof(sqz_index, C1), offsetof(sqz_index, perm), sizeof(sqz_selection),"
                    " sizeof(sqz_lookup_params), sizeof(sqz_attn_params), sizeof(sqz_kmeans_params),"
                    " offsetof(sqz_index, L_total), sizeof(sqz_shard_plan), offsetof(sqz_shard_plan, key_off));"
                    "printf(\"%zu %zu\\n\", sizeof(sqz_diagnostics), offsetof(sqz_diagnostics, n_T));"
                    "return 0;}\n")
    exe = tmp_path / "lay"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(sqz.sqz_index), sqz.sqz_index.C1.offset, sqz.sqz_index.perm.offset,
            ctypes.sizeof(sqz.sqz_selection), ctypes.sizeof(sqz.sqz_lookup_params),
            ctypes.sizeof(sqz.sqz_attn_params), ctypes.sizeof(sqz.sqz_kmeans_params),
            sqz.sqz_index.L_total.offset, ctypes.sizeof(sqz.sqz_shard_plan),
            sqz.sqz_shard_plan.key_off.offset, ctypes.sizeof(sqz.sqz_diagnostics),
            sqz.sqz_diagnostics.n_T.offset]
    assert got == want


def test_host_side_validation_without_gpu(lib):
    from paper_2411_09688_b200 import sqz

    s = sqz.sqz_index()
    s.H, s.d, s.L, s.levels, s.c2, s.dtype = 2, 128, 1000, 1, 50, sqz.SQZ_BF16
    n = ctypes.c_size_t(0)
    assert lib.sqz_lookup_workspace(ctypes.byref(s), 1, 1, ctypes.byref(n)) == 0 and n.value > 0
    assert lib.sqz_attention_workspace(ctypes.byref(s), 1, 1, 16, ctypes.byref(n)) == 0
    assert lib.sqz_cluster_keys_workspace(ctypes.byref(s), ctypes.byref(n)) == 0
    s.d = 96
    assert lib.sqz_lookup_workspace(ctypes.byref(s), 1, 1, ctypes.byref(n)) == sqz.SQZ_ERR_UNSUPPORTED
    assert b"head dimension" in lib.sqz_last_error()
    s.d, s.c2 = 128, 2000
    assert lib.sqz_lookup_workspace(ctypes.byref(s), 1, 1, ctypes.byref(n)) == sqz.SQZ_ERR_INVALID_ARG
    assert b"c2" in lib.sqz_last_error()
    s.c2, s.levels, s.c1 = 50, 2, 0
    assert lib.sqz_lookup_workspace(ctypes.byref(s), 1, 1, ctypes.byref(n)) == sqz.SQZ_ERR_INVALID_ARG
    s.levels = 1
    # missing tables are caught before anything is enqueued
    p = sqz.sqz_lookup_params(0.1, 0.01, 0.0)
    sel = sqz.sqz_selection()
    rc = lib.sqz_centroid_lookup(ctypes.byref(s), ctypes.c_void_p(16), 1, 1, ctypes.byref(p),
                                 ctypes.byref(sel), ctypes.c_void_p(16), 1 << 20, None)
    assert rc == sqz.SQZ_ERR_INVALID_ARG and b"C2" in lib.sqz_last_error()
    assert lib.sqz_merge_partials(0, None, None, 1, 1, None, None, 0, None) == sqz.SQZ_ERR_INVALID_ARG


def test_product_fails_loudly_without_library(monkeypatch):
    from paper_2411_09688_b200 import sqz

    monkeypatch.setattr(sqz, "_lib", None)
    monkeypatch.setattr(sqz, "SO", "/nonexistent/libsqz.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sqz.lib()


def test_calibration_quantile():
    import numpy as np

    from paper_2411_09688_b200 import calib

    S = np.array([[0.5, 0.1, 0.3, 0.05]])
    N = np.array([1, 1, 1, 1])
    assert calib.weighted_threshold(S, N, 0.25) == pytest.approx(0.4)   # keeps {0.5}
    assert calib.weighted_threshold(S, N, 0.5) == pytest.approx(0.2)    # keeps {0.5, 0.3}
    assert calib.weighted_threshold(S, N, 1.0) == 0.0
    N = np.array([2, 1, 1, 4])
    assert calib.weighted_threshold(S, N, 0.25) == pytest.approx(0.4)


def _index_file(path, geom, payload_bytes, magic=b"SQZIDX1\0", version=1):
    import struct
    with open(path, "wb") as f:
        f.write(magic)
        f.write(struct.pack("<I", version))
        f.write(struct.pack("<9q", *geom))
        f.write(b"\0" * payload_bytes)


def test_index_file_header_checks(lib, tmp_path):
    """sqz_index_file_info (host only): the geometry of a well-formed SQZIDX1 file; bad
    magic, bad version, invalid geometry and a payload of the wrong size are
    SQZ_ERR_FORMAT ('bad magic ... rejection')."""
    from paper_2411_09688_b200 import sqz

    H, d, L, c1, c2 = 2, 64, 100, 4, 10
    # two levels, bf16: C1, N1, child_off, C2, N2, key_off, perm
    need = H * c1 * d * 2 + H * c1 * 4 + H * (c1 + 1) * 4 + H * c2 * d * 2 + H * c2 * 4 + H * (c2 + 1) * 4 + H * L * 4
    geom = (H, d, L, 2, 0, c1, c2, sqz.SQZ_BF16, 0)
    ok = str(tmp_path / "ok.sqzidx")
    _index_file(ok, geom, need)
    g = sqz.index_file_info(ok)
    assert (g.H, g.d, g.L, g.levels, g.c1, g.c2, g.dtype, g.L_total) == (H, d, L, 2, c1, c2, sqz.SQZ_BF16, 0)
    bad = [("magic", dict(magic=b"XXXXXXX\0"), geom, need), ("version", dict(version=2), geom, need),
           ("short", {}, geom, need - 4), ("long", {}, geom, need + 4),
           ("geometry", {}, (H, 96, L, 2, 0, c1, c2, sqz.SQZ_BF16, 0), need)]
    for name, kw, gm, nb in bad:
        p = str(tmp_path / f"{name}.sqzidx")
        _index_file(p, gm, nb, **kw)
        with pytest.raises(sqz.SqzError) as e:
            sqz.index_file_info(p)
        assert e.value.code == sqz.SQZ_ERR_FORMAT, name
