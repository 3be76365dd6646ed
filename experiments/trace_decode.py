"""Device timeline of one cfg2 decode step (build with SQZ_NVCC_EXTRA=-DSQZ_TRACE).
Prints per-phase globaltimer statistics (us, relative to the first lookup CTA start)."""
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
# SQZ_FLUSH=read: after the write flush, read a second 512 MB buffer (L2 left clean)
rflush = torch.ones(128 << 20, dtype=torch.float32, device="cuda") if os.environ.get("SQZ_FLUSH") == "read" else None
lib = sqz.lib()
for it in range(6):
    flush.zero_()  # no sync: the host runs ahead as in bench.py
    if rflush is not None:
        rflush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if os.environ.get("SQZ_STEP") == "1":  # the decode-step hand-off path
        sqz.decode_step(idx, Q, Kp, Vp, Ku, Vu, 1 / np.sqrt(d), T, sel=sel, O=O, LSE=LSE)
    else:
        sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T, sel=sel)
        sqz.sparse_attention(Q, Kp, Vp, idx, sel, Ku, Vu, O=O, LSE=LSE)
    e1.record()
    torch.cuda.synchronize()
tl = np.zeros(2048 * 8, np.uint64)
ta = np.zeros(2048 * 8, np.uint64)
lib.sqz_trace_look(tl.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tl.nbytes))
lib.sqz_trace_attn(ta.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(ta.nbytes))
tl = tl.reshape(2048, 8).astype(np.float64)
tl = tl[tl[:, 0] >= tl[:, 0].max() - 200e3]  # the last launch's CTAs only
ta = ta.reshape(2048, 8).astype(np.float64)
ta = ta[ta[:, 0] > 0]
t0 = tl[:, 0].min()
print(f"retention {ret}: event step time {e0.elapsed_time(e1) * 1e3:.1f} us; k = {int(sel.n_keys.sum())}")
def st(name, v):
    v = (v - t0) / 1e3
    print(f"  {name:38s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
for i, n in [(0, "lookup start"), (1, "lookup scan done"), (2, "lookup compaction done (pre-exchange)"),
             (3, "lookup count exchange done"), (6, "lookup prefix done"), (7, "lookup list/kpref stored"),
             (4, "lookup writes done"), (5, "lookup end")]:
    if (tl[:, i] > 0).all():
        st(n, tl[:, i])
for i, n in [(0, "attn entry"), (1, "attn after griddep wait"), (2, "attn prologue done"),
             (6, "attn merger's ticket taken"), (4, "attn streaming done (last seg)"), (5, "attn end")]:
    col = ta[:, i]
    if (col > 0).any():
        st(n, col[col > 0])
# per-CTA attribution of the tail: segments, merges, keys, SM
tm = np.zeros(2048 * 4, np.uint64)
lib.sqz_trace_mrg(tm.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tm.nbytes))
tm = tm.reshape(2048, 4)[:32].astype(np.float64)
for i, n in [(0, "merge start"), (1, "merge partials loaded"), (2, "merge end")]:
    st(n, tm[:, i])
info = ta[:, 3].astype(np.uint64)
nseg = (info & 0xff).astype(int)
nmer = ((info >> 8) & 0xff).astype(int)
keys = (info >> 16).astype(int)
smid = ta[:, 7].astype(int)
done = (ta[:, 4] - t0) / 1e3
end = (ta[:, 5] - t0) / 1e3
start = (ta[:, 2] - t0) / 1e3
print(f"  CTAs {len(ta)}; keys/CTA min {keys.min()} max {keys.max()}")
for k in sorted(set(nseg)):
    m = nseg == k
    print(f"  nseg={k}: {m.sum():4d} CTAs, done med {np.median(done[m]):.2f} max {done[m].max():.2f}; "
          f"end med {np.median(end[m]):.2f} max {end[m].max():.2f}")
for k in sorted(set(nmer)):
    m = nmer == k
    print(f"  merges={k}: {m.sum():4d} CTAs, end med {np.median(end[m]):.2f} max {end[m].max():.2f}")
rate = keys / np.maximum(done - start, 1e-3)  # keys per us
for lo, hi in [(0, 74), (74, 148)]:
    m = (smid >= lo) & (smid < hi)
    print(f"  SM {lo}-{hi - 1}: {m.sum()} CTAs, keys/us med {np.median(rate[m]):.1f}, done med {np.median(done[m]):.2f} max {done[m].max():.2f}")
per_sm = {}
for s_, d_ in zip(smid, done):
    per_sm.setdefault(s_, []).append(d_)
sm_max = np.array([max(v) for v in per_sm.values()])
sm_spread = np.array([max(v) - min(v) for v in per_sm.values()])
print(f"  per-SM last done: min {sm_max.min():.2f} med {np.median(sm_max):.2f} max {sm_max.max():.2f}; "
      f"within-SM spread med {np.median(sm_spread):.2f}")
order = np.argsort(-done)[:12]
print("  slowest CTAs (cta, sm, nseg, merges, keys, start, done, end):")
for i in order:
    print(f"    {i:4d} {smid[i]:4d} {nseg[i]} {nmer[i]} {keys[i]:5d} {start[i]:6.2f} {done[i]:6.2f} {end[i]:6.2f}")
np.savez(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "trace_decode_raw.npz"),
         tl=tl, ta=ta, t0=t0)
