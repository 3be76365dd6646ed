"""Per-iteration timeline of CTA (0,0,0) of the prefill attention kernel (-DSQZ_TRACE)."""
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
Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, n_q, seed=5003))
s = sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), 0.0, debug=True)
T = calib.weighted_threshold(s.dbg_S.cpu().numpy(), idx.N2.cpu().numpy()[None], 0.3,
                             total_weight=H * L)
sel = sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T)
for _ in range(3):
    O, LSE = sqz.sparse_attention(Q, Kp, Vp, idx, sel, Ku, Vu, causal=True)
torch.cuda.synchronize()
W = 24 if os.environ.get("SQZ_PF_LEGACY") is None else 8
NIT = 128 if os.environ.get("SQZ_PF_LEGACY") is None else 64
tr = np.zeros(NIT * W, np.uint64)
ws = os.environ.get("SQZ_PF_LEGACY") is None
(sqz.lib().sqz_trace_ws if ws else sqz.lib().sqz_trace_pf)(tr.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(tr.nbytes))
tr = tr.reshape(NIT, W).astype(np.float64)
names = (["S0rdy", "P0out", "S1rdy", "P1out", "mmaP0", "mmaV", "mmaK", "mmaP1", "Kiss", "Viss", "Kemp", "Vemp", "PV0iss", "S0iss", "sm0max", "mmaQ", "sm0ld", "sm0exp", "sm0st", "sm0epi", "-", "-", "-", "Qiss"] if ws else
         ["start", "loads+sync", "S ready", "P written", "PV issued"])
t0 = tr[0, 19] if ws else tr[0, 0]
if ws:
    ct = np.zeros(1024 * 4, np.uint64)
    sqz.lib().sqz_trace_ws_cta(ct.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(ct.nbytes))
    ct = ct.reshape(1024, 4).astype(np.float64)
    n = int((ct[:, 0] > 0).sum())
    base = ct[:n, 0].min()
    ent, lend, ex = (ct[:n, 0] - base) / 1e3, (ct[:n, 1] - base) / 1e3, (ct[:n, 2] - base) / 1e3
    print(f"CTAs {n}: entry max {ent.max():.1f}  loop-end min/med/max {lend.min():.1f}/{np.median(lend):.1f}/{lend.max():.1f}"
          f"  exit min/med/max {ex.min():.1f}/{np.median(ex):.1f}/{ex.max():.1f} us")
    order = np.argsort(-ex)
    # host replay of the piece walk (segment = (bh, pair of 128-row tiles))
    nk = sel.n_keys.cpu().numpy().reshape(-1)
    npairs = (n_q + 255) // 256
    seg_t = []
    for bh in range(len(nk)):
        for pr in range(npairs):
            last = min(pr * 256 + 256, n_q) - 1
            nuv = max(0, min(last + 1, n_q))  # causal, n_u == n_q
            nkf4 = (int(nk[bh]) + 3) // 4 * 4 if nuv else int(nk[bh])
            seg_t.append((nkf4 + nuv + 63) // 64)
    seg_t = np.array(seg_t)
    SEG_W = 6
    seg_c = np.where(np.array(seg_t) > 0, np.array(seg_t) + SEG_W, 0)
    st = np.concatenate([[0], np.cumsum(seg_c)])
    Ttot = int(st[-1])
    print(f"segments {len(seg_t)} tiles min/med/max {seg_t.min()}/{int(np.median(seg_t))}/{seg_t.max()} total {Ttot}")
    for cta in [int(i) for i in order[:6]] + [int(order[-1])]:
        lo_, hi_ = Ttot * cta // n, Ttot * (cta + 1) // n
        pcs = [(si, max(0, int(max(st[si], lo_) - st[si]) - SEG_W), max(0, int(min(st[si + 1], hi_) - st[si]) - SEG_W), int(seg_t[si]))
               for si in range(len(seg_t)) if st[si + 1] > lo_ and st[si] < hi_]
        print(f"CTA {cta} (loop end {lend[cta]:.1f}): units [{lo_},{hi_}) pieces (seg, from, to, seg_tiles): {pcs}")
    print("slowest CTAs:", [(int(i), round(ex[i], 1), round(lend[i], 1)) for i in order[:12]])
    f = 1.965e3
    print(f"entry 0  scan+setup {(tr[0,20]-t0)/f:.2f}  loop end {(tr[0,21]-t0)/f:.2f}  exit {(tr[0,22]-t0)/f:.2f} us")
    prev = None
    for it in range(NIT):
        if tr[it, 0] == 0:
            break
        v = [(tr[it, k] - t0) / f for k in (0, 1, 2, 3, 4, 8, 9)]
        per = "" if prev is None else f" dt={v[0]-prev:5.2f}"
        prev = v[0]
        print(f"t{it:3d} S0rdy={v[0]:7.2f} P0={v[1]:7.2f} S1rdy={v[2]:7.2f} P1={v[3]:7.2f} mmaP0={v[4]:7.2f} Kiss={v[5]:7.2f} Viss={v[6]:7.2f}{per}")
    full = os.environ.get("TRACE_FULL")
    if full:
        lo_, hi_ = (int(x) for x in full.split(":"))
        for it in range(lo_, hi_):
            print(f"t{it:3d} " + " ".join(f"{n}={(tr[it, k] - t0) / f:7.2f}" for k, n in enumerate(names) if n != "-"))
    sys.exit(0)
for it in range(min(20, 64)):
    if tr[it, 0] == 0:
        break
    row = [(tr[it, k] - t0) / (1.965e3 if ws else 1e3) for k in range(len(names))]
    print(f"it {it:2d}: " + "  ".join(f"{n}={v:6.2f}" for n, v in zip(names, row)))
