"""Debug: sharded prefill lookup S-bar vs oracle (relative error per shard)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import oracle
from test_gpu_shard import _setup, _run_sharded
from paper_2411_09688_b200 import sqz
for world in (1, 2):
    P, idx, g, Kp, Vp, scale, T, T1 = _setup(1, True, B=1, n_q=200)
    Q, shards, sels = _run_sharded(P, g, Kp, Vp, scale, T, T1, world)
    torch.cuda.synchronize()
    ref = oracle.lookup(oracle.to_f64(P["Q"]), idx, scale, T, T1)
    full = sqz.centroid_lookup(g, Q, scale, T, T1, debug=True)
    Sf = full.dbg_S.cpu().numpy()
    print("world", world, "T", T, "unsharded max rel", np.nanmax(np.abs(Sf - ref["Sbar2"]) / ref["Sbar2"]))
    print("  lse unsharded max abs", np.abs(full.dbg_lse.cpu().numpy() - ref["lse"]).max())
    for r, ((loc, _, _), s) in enumerate(zip(shards, sels)):
        src = loc.c2_src.cpu().numpy()
        S = s.dbg_S.cpu().numpy()
        e = []
        for h in range(idx.H):
            ok = src[h] >= 0
            e.append(np.abs(S[0, h][ok] - ref["Sbar2"][0, h][src[h][ok]]) / ref["Sbar2"][0, h][src[h][ok]])
        e = np.concatenate(e)
        print("  shard", r, "max rel", e.max(), "lse max abs", np.abs(s.dbg_lse.cpu().numpy() - ref["lse"]).max())
# detail for world 2, head 0
P, idx, g, Kp, Vp, scale, T, T1 = _setup(1, True, B=1, n_q=200)
Q, shards, sels = _run_sharded(P, g, Kp, Vp, scale, T, T1, 2)
torch.cuda.synchronize()
ref = oracle.lookup(oracle.to_f64(P["Q"]), idx, scale, T, T1)
for r, ((loc, _, _), s) in enumerate(zip(shards, sels)):
    src = loc.c2_src.cpu().numpy()
    S = s.dbg_S.cpu().numpy()
    for h in range(idx.H):
        print(r, h, np.round(S[0, h] / ref["Sbar2"][0, h][src[h]], 4).tolist())
