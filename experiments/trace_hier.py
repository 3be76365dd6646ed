"""Device timeline of the Level-2 decode lookup kernel (hierarchical, cfg4 shape or
cfg5 shape with argv[1] == 'cfg5'); builds libsqz with -DSQZ_TRACE."""
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

big = len(sys.argv) > 1 and sys.argv[1] == "cfg5"
H, d = 32, 128
L, c2, c1, B = (1048576, 52429, 10486, 1) if big else (131072, 6554, 1311, 8)
mix = synth.device_mixture(H, c2, d, G1=c1, seed=1004)
K, V = synth.device_keys(mix, L, seed=1004)
idx, Kp, Vp, _ = sqz.cluster_keys(K, V, c2, synth.device_kmeans_init(H, L, c2, 2004), c1,
                                  synth.device_kmeans_init(H, c2, c1, 2104), max_iters=2 if big else 10)
del K, V
Qc = synth.device_decode_queries(mix, 16, seed=3004)
s = sqz.centroid_lookup(idx, Qc, 1 / np.sqrt(d), 0.0, 0.0, debug=True)
T1 = calib.distributed_threshold(s.dbg_S1, idx.N1[None], 0.5, float(16 * idx.N1.sum()))
s = sqz.centroid_lookup(idx, Qc, 1 / np.sqrt(d), 0.0, T1, debug=True)
T = calib.distributed_threshold(s.dbg_S, idx.N2[None], 0.1, float(16 * H * L))
Q = synth.device_decode_queries(mix, B, seed=4004)
sel = sqz.Selection.empty(idx, B, 1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T, T1, sel=sel)
    e1.record()
    torch.cuda.synchronize()
tl = np.zeros(2048 * 8, np.uint64)
sqz.lib().sqz_trace_look(tl.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tl.nbytes))
tl = tl.reshape(2048, 8).astype(np.float64)
tl = tl[tl[:, 0] > 0]
tl = tl[tl[:, 0] > tl[:, 5].max() - 1e6]  # CTAs of the last launch (stale slots are older)
t0 = tl[:, 0].min()
print(f"lookup (both levels) {e0.elapsed_time(e1) * 1e3:.1f} us; L2 CTAs traced {len(tl)}; "
      f"candidates/bh {sel.n_clusters.float().mean().item():.0f} sel, keys {sel.n_keys.float().mean().item():.0f}")
for i, n in enumerate(["start", "scan done", "compaction done (pre-barrier)", "cluster.sync 2",
                       "writes done", "end"]):
    v = (tl[:, i] - t0) / 1e3
    print(f"  {n:28s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
if (tl[:, 7] > 0).any():
    v = (tl[:, 7] - t0) / 1e3
    print(f"  {'SLIM length pass done':28s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
if (tl[:, 6] > 0).any():
    v = (tl[:, 6] - t0) / 1e3
    print(f"  {'candidate slice ready':28s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
d_scan = (tl[:, 1] - tl[:, 0]) / 1e3
d_cmp = (tl[:, 3] - tl[:, 2]) / 1e3
d_wr = (tl[:, 4] - tl[:, 3]) / 1e3
print("per-CTA durations med/max: scan", np.round([np.median(d_scan), d_scan.max()], 2),
      "compaction", np.round([np.median(d_cmp), d_cmp.max()], 2), "writes", np.round([np.median(d_wr), d_wr.max()], 2))
