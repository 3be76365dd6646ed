"""Device timeline of one cfg2 fused decode step (sqz_decode_step), built with
-DSQZ_TRACE: per-phase globaltimer statistics (us from the first CTA start)."""
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

ret = float(sys.argv[1]) if len(sys.argv) > 1 else 0.3
H, L, d, c, n_u = 32, 32768, 128, 1024, 1024
fc = synth.fixed_context(H, L, d, c, seed=1002)
idx, Kp, Vp, _ = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), c,
                                  torch.from_numpy(synth.kmeans_init(H, L, c, seed=2002)).cuda(),
                                  max_iters=20)
Qc = sqz.to_device(synth.decode_queries(fc.mix, 64, seed=3002))
s = sqz.centroid_lookup(idx, Qc, 1 / np.sqrt(d), 0.0, debug=True)
T = calib.weighted_threshold(s.dbg_S.cpu().numpy(), idx.N2.cpu().numpy()[None], ret,
                             total_weight=64 * H * L)
Q = sqz.to_device(synth.decode_queries(fc.mix, 1, seed=4002))
Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, n_u, seed=5002))
sel = sqz.Selection.empty(idx, 1, 1)
O = torch.empty(1, H, 1, d, dtype=torch.bfloat16, device="cuda")
LSE = torch.empty(1, H, 1, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = sqz.lib()
for it in range(8):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sqz.decode_step(idx, Q, Kp, Vp, Ku, Vu, 1 / np.sqrt(d), T, sel=sel, O=O, LSE=LSE)
    e1.record()
    torch.cuda.synchronize()
tr = np.zeros(2048 * 8, np.uint64)
lib.sqz_trace_step(tr.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tr.nbytes))
tr = tr.reshape(2048, 8).astype(np.float64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
print(f"retention {ret}: event step time {e0.elapsed_time(e1) * 1e3:.1f} us; k = {int(sel.n_keys.sum())}; "
      f"CTAs {len(tr)}")
for i, n in enumerate(["start", "scan done", "barrier 1 passed", "B done", "barrier 2 passed",
                       "C done", "D (fixed streams) done"]):
    v = (tr[:, i] - t0) / 1e3
    print(f"  {n:28s} min {v.min():7.2f}  med {np.median(v):7.2f}  p90 {np.percentile(v, 90):7.2f}  max {v.max():7.2f} us")
nd = tr[:, 7]
print(f"  user chunks taken at barriers: total {int(nd.sum())}, per CTA max {int(nd.max())}")
