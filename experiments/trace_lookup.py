"""Per-CTA timeline of the tensor-core prefill lookup (-DSQZ_TRACE build), cfg3 shape."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SQZ_NVCC_EXTRA"] = "-DSQZ_TRACE " + os.environ.get("TRACE_EXTRA", "")
from paper_2411_09688_b200 import build as bld  # noqa: E402
bld.build(force=True)
from paper_2411_09688_b200 import calib, sqz, synth  # noqa: E402

H, L, d, c, n_q = 32, 32768, 128, 1024, 1024
fc = synth.fixed_context(H, L, d, c, seed=1003)
idx, Kp, Vp, _ = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), c,
                                  torch.from_numpy(synth.kmeans_init(H, L, c, seed=2003)).cuda(),
                                  max_iters=10)
Q = sqz.to_device(synth.prefill_queries(fc.mix, 1, n_q, seed=4003))
s = sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), 0.0, debug=True)
T = calib.weighted_threshold(s.dbg_S.cpu().numpy(), idx.N2.cpu().numpy()[None], 0.3, total_weight=H * L)
sel = sqz.Selection.empty(idx, 1, n_q)
for _ in range(3):
    sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T, sel=sel)
torch.cuda.synchronize()
tr = np.zeros(2048 * 8, np.uint64)
sqz.lib().sqz_trace_pl(tr.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tr.nbytes))
tr = tr.reshape(2048, 8).astype(np.float64)
n = (n_q + 127) // 128 * H
tr = tr[:n]
base = tr[:, 0].min()
t = (tr - base) / 1e3
names = ["entry", "prologue", "pass2", "loopend", "final0", "final1"]
for i, nm in enumerate(names):
    col = t[:, i][tr[:, i] > 0]
    if len(col):
        print(f"{nm:9s} n={len(col):4d} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us")
fin = tr[:, 4] > 0
print("finalize durations (us):", np.round((tr[fin, 5] - tr[fin, 4]) / 1e3, 2)[:16])
print("loop durations min/med/max:", np.round(np.percentile((tr[:, 3] - tr[:, 1]) / 1e3, [0, 50, 100]), 2))
print("entry spread:", np.round(np.sort(t[:, 0])[::16], 2))
it = np.zeros(64 * 4, np.uint64)
sqz.lib().sqz_trace_pl_it(it.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(it.nbytes))
it = it.reshape(64, 4).astype(np.float64)
b0 = tr[0, 0]
print("CTA(0,0) per-iteration [top-sync, mbar done, epilogue done] us from entry:")
for k in range(16):
    print(k, np.round((it[k, :3] - b0) / 1e3, 2))
fn = np.zeros(64 * 8, np.uint64)
sqz.lib().sqz_trace_fin(fn.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(fn.nbytes))
fn = fn.reshape(64, 8).astype(np.float64)
print("finalize per bh [start, loads, tile0..3, end, t0-scan-done] us rel start:")
print("n_clusters", sel.n_clusters.cpu().numpy()[0, :8], "n_keys", sel.n_keys.cpu().numpy()[0, :8])
for bh in range(8):
    print(bh, np.round((fn[bh, [0, 1, 2, 3, 4, 5, 6, 7]] - fn[bh, 0]) / 1e3, 2))
