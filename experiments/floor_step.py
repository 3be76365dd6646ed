"""Where the cfg2 step's fixed time goes: CUDA-event time (graph replay, after the
bench's 512 MB write flush) of an empty kernel, the lookup alone, the attention
alone, and the two-call step; with and without the flush."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_09688_b200 import calib, sqz, synth  # noqa: E402

H, L, d, c, n_u = 32, 32768, 128, 1024, 1024
fc = synth.fixed_context(H, L, d, c, seed=1002)
idx, Kp, Vp, _ = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), c,
                                  torch.from_numpy(synth.kmeans_init(H, L, c, seed=2002)).cuda(),
                                  max_iters=20)
Qc = sqz.to_device(synth.decode_queries(fc.mix, 64, seed=3002))
s = sqz.centroid_lookup(idx, Qc, 1 / np.sqrt(d), 0.0, debug=True)
T = calib.weighted_threshold(s.dbg_S.cpu().numpy(), idx.N2.cpu().numpy()[None], 0.3,
                             total_weight=64 * H * L)
Q = sqz.to_device(synth.decode_queries(fc.mix, 1, seed=4002))
Ku, Vu = (sqz.to_device(a) for a in synth.user_kv(fc.mix, 1, n_u, seed=5002))
sel = sqz.Selection.empty(idx, 1, 1)
O = torch.empty(1, H, 1, d, dtype=torch.bfloat16, device="cuda")
LSE = torch.empty(1, H, 1, device="cuda")
x = torch.zeros(16, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def graph(fn):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="thread_local"):
        fn()
    return g


def t(g, fl=True, n=40):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        if fl:
            flush.zero_()
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)[3:-3]
    return sum(v) / len(v)


look = lambda: sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T, sel=sel)
attn = lambda: sqz.sparse_attention(Q, Kp, Vp, idx, sel, Ku, Vu, O=O, LSE=LSE)
look()
attn()
gs = {"empty kernel": graph(lambda: x.add_(1)),
      "lookup": graph(look),
      "attention": graph(attn),
      "lookup+attention": graph(lambda: (look(), attn())),
      "empty + lookup+attention": graph(lambda: (x.add_(1), look(), attn()))}
for fl in (True, False):
    print(f"flush={fl}: " + " | ".join(f"{k} {t(g, fl):.2f} us" for k, g in gs.items()))
