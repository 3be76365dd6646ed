"""How much of a batched decode step's selected fixed KV is shared between the batch's
queries (cfg4 shape: 128K, c1=1311 / c2=6554, B=8, 10%): sum over queries of the selected keys
vs the per-head union (the bytes a batch-shared attention pass would read)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_09688_b200 import calib, sqz, synth  # noqa: E402

H, d, L, c2, c1, B = 32, 128, 131072, 6554, 1311, 8
mix = synth.device_mixture(H, c2, d, G1=c1, seed=1004)
K, V = synth.device_keys(mix, L, seed=1004)
idx, Kp, Vp, _ = sqz.cluster_keys(K, V, c2, synth.device_kmeans_init(H, L, c2, 2004), c1,
                                  synth.device_kmeans_init(H, c2, c1, 2104), max_iters=10)
Qc = synth.device_decode_queries(mix, 16, seed=3004)
s = sqz.centroid_lookup(idx, Qc, 1 / np.sqrt(d), 0.0, 0.0, debug=True)
T1 = calib.distributed_threshold(s.dbg_S1, idx.N1[None], 0.5, float(16 * idx.N1.sum()))
s = sqz.centroid_lookup(idx, Qc, 1 / np.sqrt(d), 0.0, T1, debug=True)
T = calib.distributed_threshold(s.dbg_S, idx.N2[None], 0.1, float(16 * H * L))
for seed in (4004, 4104):
    Q = synth.device_decode_queries(mix, B, seed=seed)
    sel = sqz.centroid_lookup(idx, Q, 1 / np.sqrt(d), T, T1)
    torch.cuda.synchronize()
    cl, n = sel.clusters.cpu().numpy(), sel.n_clusters.cpu().numpy()
    N2 = idx.N2.cpu().numpy()
    tot = uni = 0
    per_head = []
    for h in range(H):
        m = np.zeros(c2, bool)
        t = 0
        for b in range(B):
            ids = cl[b, h, :n[b, h]]
            t += N2[h, ids].sum()
            m[ids] = True
        u = N2[h, m].sum()
        tot += t
        uni += u
        per_head.append(t / max(u, 1))
    print(f"queries seed {seed}: selected keys sum {tot}, per-head union {uni}, "
          f"sum/union {tot / uni:.2f} (per head min {min(per_head):.2f} max {max(per_head):.2f})")
