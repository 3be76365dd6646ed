"""Debug: sharded hierarchical prefill lookup vs oracle."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import oracle
from test_gpu_shard import _setup, _run_sharded
from paper_2411_09688_b200 import sqz
world = 3
P, idx, g, Kp, Vp, scale, T, T1 = _setup(2, True, B=1, n_q=200)
for rep in range(2):
    Q, shards, sels = _run_sharded(P, g, Kp, Vp, scale, T, T1, world)
    torch.cuda.synchronize()
    surv1 = np.zeros((1, idx.H, idx.c1), bool)
    for r, ((loc, _, _), s) in enumerate(zip(shards, sels)):
        surv1[:, :, np.arange(r, idx.c1, world)] |= s.l1_surv.cpu().numpy().astype(bool)
    Q64 = oracle.to_f64(P["Q"])
    ref = oracle.lookup(Q64, idx, scale, T, T1, forced_l1=surv1)
    ref1 = oracle.lookup(Q64, idx, scale, T, T1)
    print("T", T, "T1", T1)
    for r, ((loc, _, _), s) in enumerate(zip(shards, sels)):
        src = loc.c2_src.cpu().numpy()
        S = s.dbg_S.cpu().numpy(); S1 = s.dbg_S1.cpu().numpy()
        lse = s.dbg_lse.cpu().numpy()
        print(" shard", r, "lse err", np.nanmax(np.abs(lse - ref["lse"])), "S1 rel", np.nanmax(np.abs(S1[0] - ref1["Sbar1"][0][:, np.arange(r, idx.c1, world)]) / ref1["Sbar1"][0][:, np.arange(r, idx.c1, world)]))
        for h in range(idx.H):
            ok = (src[h] >= 0) & ~np.isnan(S[0, h])
            rr = S[0, h][ok] / ref["Sbar2"][0, h][src[h][ok]]
            bad = np.abs(rr - 1) > 1e-4
            if bad.any():
                print("   h", h, "rows", np.nonzero(ok)[0][bad].tolist(), "ratio", np.round(rr[bad], 4).tolist())
