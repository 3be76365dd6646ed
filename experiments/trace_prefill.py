"""Per-iteration timeline of CTA (0,0,0) of the prefill attention kernel (-DSQZ_TRACE)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_09688_b200 import calib, sqz, synth  # noqa: E402

H, L, d, c, n_q = 32, 32768, 128, 1024, 1024
fc = synth.fixed_context(H, L, d, c, seed=1003)
idx, Kp, Vp, _ = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), c,
                                  torch.from_numpy(synth.kmeans_init(H, L, c, seed=2003)).cuda(),
                                  max_iters=10)
Q = sqz.to_device(synth.prefill_queries(fc.mix, 1, n_q, seed=4003))
Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, n_q, seed=5003))
s = sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), 0.0, debug=True)
T = calib.weighted_threshold(s.dbg_S.cpu().numpy(), idx.N2.cpu().numpy()[None], 0.3,
                             total_weight=H * L)
sel = sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T)
for _ in range(3):
    O, LSE = sqz.sparse_attention(Q, Kp, Vp, idx, sel, Ku, Vu, causal=True)
torch.cuda.synchronize()
tr = np.zeros(64 * 8, np.uint64)
sqz.lib().sqz_trace_pf(tr.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tr.nbytes))
tr = tr.reshape(64, 8).astype(np.float64)
t0 = tr[0, 0]
names = ["start", "loads+sync", "S ready", "P written", "PV issued"]
for it in range(min(12, 64)):
    if tr[it, 0] == 0:
        break
    row = [(tr[it, k] - t0) / 1e3 for k in range(5)]
    print(f"it {it:2d}: " + "  ".join(f"{n}={v:7.2f}" for n, v in zip(names, row)))
