"""Timeline of the cfg3 prefill lookup (k_prefill_lookup_tc, -DSQZ_TRACE): per-CTA phase
statistics and CTA (0,0)'s per-iteration times."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SQZ_NVCC_EXTRA"] = "-DSQZ_TRACE"
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
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sel = sqz.Selection.empty(idx, 1, n_q)
for _ in range(4):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T, sel=sel)
    e1.record()
    torch.cuda.synchronize()
lib = sqz.lib()
tr = np.zeros(2048 * 8, np.uint64)
lib.sqz_trace_pl(tr.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tr.nbytes))
tr = tr.reshape(2048, 8).astype(np.float64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
print(f"event {e0.elapsed_time(e1) * 1e3:.1f} us; CTAs {len(tr)}")
for i, n in enumerate(["start", "prologue done", "pass 2 starts", "loop end", "finalize start", "end"]):
    v = tr[:, i]
    v = (v[v > 0] - t0) / 1e3
    if len(v):
        print(f"  {n:16s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us  (n={len(v)})")
it = np.zeros(64 * 4, np.uint64)
lib.sqz_trace_pl_it(it.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(it.nbytes))
it = it.reshape(64, 4).astype(np.float64)
it = it[it[:, 0] > 0]
print("CTA(0,0) iterations: [mma wait start, mma done, epilogue done] (us from t0)")
for k, r in enumerate(it[:20]):
    print(f"  {k:2d}: " + " ".join(f"{(x - t0) / 1e3:7.2f}" for x in r[:3]))
