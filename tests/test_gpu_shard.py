"""Fixed-context sharding by cluster on the GPU, through the C ABI.

One GPU emulates `world` ranks: every rank's shard index is built by
sqz_index_shard, the staged lookup (sqz_centroid_lookup_stage) runs on each
shard, and the statistics exchange between stages is a device concatenation in
rank order -- exactly the buffer the NCCL all-gather produces.  The union of
the shards' selections must equal the oracle's (band rule) and the unsharded
GPU lookup's; the shards' attention partials merged by sqz_merge_partials must
match the oracle on the union mask (north-star tolerances).  The NCCL path
itself (sqz_comm_*) is exercised with a world-1 communicator."""
import numpy as np
import pytest

import oracle
from paper_2411_09688_b200 import calib

from helpers import assert_selection_parity, gpu_index, gpu_sets, oracle_problem, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_09688_b200 import sqz

    sqz.device_check()


def _sqz():
    from paper_2411_09688_b200 import sqz

    return sqz


def _setup(levels, prefill, seed=71, H=4, L=4096, c2=64, dtype=1, B=2, n_q=1, n_u=24, d=128):
    sqz = _sqz()
    P = oracle_problem(H=H, L=L, d=d, c2=c2, c1=c2 // 8 if levels == 2 else 0, dtype=dtype,
                       seed=seed, B=B, n_q=n_q, prefill=prefill, n_u=n_u, max_iters=12)
    idx = P["idx"]
    scale = 1.0 / np.sqrt(d)
    Q64 = oracle.to_f64(P["Q"])
    T1 = 0.0
    r = oracle.lookup(Q64, idx, scale, 0.0, 0.0)
    if levels == 2:
        T1 = calib.weighted_threshold(r["Sbar1"], idx.N1[None], 0.5)
        r = oracle.lookup(Q64, idx, scale, 0.0, T1)
    T = calib.weighted_threshold(r["Sbar2"], idx.N2[None], 0.3)
    g = gpu_index(idx)
    Kp = sqz.to_device(oracle.permute_kv(P["fc"].K, idx))
    Vp = sqz.to_device(oracle.permute_kv(P["fc"].V, idx))
    return P, idx, g, Kp, Vp, scale, T, T1


def _run_sharded(P, g, Kp, Vp, scale, T, T1, world):
    sqz = _sqz()
    Q = sqz.to_device(P["Q"])
    B, H, n_q, d = Q.shape
    shards = [sqz.shard_index(g, Kp, Vp, r, world) for r in range(world)]
    for loc, _, _ in shards:
        sqz.index_validate(loc)
    sels = [sqz.Selection.empty(loc, B, n_q, debug=True) for loc, _, _ in shards]
    wss = [sqz.workspace(sqz.lookup_workspace_bytes(loc, B, n_q)) for loc, _, _ in shards]
    outs = [torch.empty(B, H, n_q, 2, device="cuda") for _ in range(world)]
    gathered = None
    for stage in range(g.levels + 1):
        for r, (loc, _, _) in enumerate(shards):
            sqz.centroid_lookup_stage(loc, Q, scale, T, T1, stage, gathered,
                                      outs[r] if stage < g.levels else None, sels[r], wss[r])
        gathered = torch.stack(outs).contiguous()  # the all-gather, in rank order
    return Q, shards, sels


@pytest.mark.parametrize("levels,prefill,world,B", [
    (1, False, 1, 2), (1, False, 2, 2), (1, False, 3, 2), (2, False, 2, 2), (2, False, 4, 2),
    (2, False, 3, 5), (1, True, 2, 1), (2, True, 3, 1)])
def test_sharded_lookup_and_merge_match_oracle(levels, prefill, world, B):
    sqz = _sqz()
    P, idx, g, Kp, Vp, scale, T, T1 = _setup(levels, prefill, B=B, n_q=200 if prefill else 1)
    Q, shards, sels = _run_sharded(P, g, Kp, Vp, scale, T, T1, world)
    B, H, n_q, d = Q.shape
    torch.cuda.synchronize()
    # union of the shards' selections, in global cluster ids
    sel_u = np.zeros((B, H, idx.c2), bool)
    surv1 = np.zeros((B, H, max(idx.c1, 1)), bool)
    for r, ((loc, _, _), s) in enumerate(zip(shards, sels)):
        src = loc.c2_src.cpu().numpy()
        cl, n = s.clusters.cpu().numpy(), s.n_clusters.cpu().numpy()
        for b in range(B):
            for h in range(H):
                ids = src[h][cl[b, h, :n[b, h]]]
                assert np.all(ids >= 0), "a padding row was selected"
                assert not sel_u[b, h, ids].any(), "cluster selected by two shards"
                sel_u[b, h, ids] = True
        if idx.levels == 2:
            c1s = np.arange(r, idx.c1, world)
            surv1[:, :, c1s] |= s.l1_surv.cpu().numpy().astype(bool)
    Q64 = oracle.to_f64(P["Q"])
    forced = surv1 if idx.levels == 2 else None
    if forced is not None:
        ref1 = oracle.lookup(Q64, idx, scale, T, T1)
        assert_selection_parity(surv1, ref1["surv1"], ref1["Sbar1"], T1, what="level-1")
    ref = oracle.lookup(Q64, idx, scale, T, T1, forced_l1=forced)
    assert_selection_parity(sel_u, ref["sel2"], ref["Sbar2"], T, what=f"sharded x{world}")
    # the unsharded GPU lookup on the same tables selects the same clusters up to the band
    full = sqz.centroid_lookup(g, Q, scale, T, T1, debug=True)
    assert_selection_parity(gpu_sets(full, B, H, idx.c2), sel_u, ref["Sbar2"], T,
                            what="sharded vs unsharded GPU")
    # attention: partial per shard (user KV on rank 0 only), merged
    Ku, Vu = sqz.to_device(P["Ku"]), sqz.to_device(P["Vu"])
    Op, Lp = [], []
    for r, ((loc, Kl, Vl), s) in enumerate(zip(shards, sels)):
        O, LSE = sqz.sparse_attention(Q, Kl, Vl, loc, s, Ku if r == 0 else None,
                                      Vu if r == 0 else None, scale, causal=prefill, partial=True,
                                      out_dtype=sqz.SQZ_F32)
        Op.append(O.reshape(-1, d))
        Lp.append(LSE.reshape(-1))
    Om, Lm = sqz.merge_partials(torch.stack(Op), torch.stack(Lp), out_dtype=sqz.SQZ_BF16)
    torch.cuda.synchronize()
    mask = oracle.keymask(idx, sel_u)
    O_ref, L_ref, rc = oracle.attention(Q64, oracle.to_f64(P["fc"].K), oracle.to_f64(P["fc"].V),
                                        mask, oracle.to_f64(P["Ku"]), oracle.to_f64(P["Vu"]),
                                        prefill, scale)
    assert rc == 0
    Og = Om.float().cpu().numpy().reshape(O_ref.shape)
    assert np.abs(Og - O_ref).max() <= 2e-2
    assert rel_l2(Og, O_ref) <= 5e-3
    assert np.abs(Lm.cpu().numpy().reshape(L_ref.shape) - L_ref).max() <= 1e-3


def test_comm_world1_matches_local_path():
    """NCCL communicator of one rank: the comm lookup (stats -> ncclAllGather ->
    fold -> select) equals the plain lookup, and allgather_merge equals the
    local merge."""
    sqz = _sqz()
    import torch.distributed as dist

    if not dist.is_initialized():
        import os
        import socket

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = sqz.Comm(0, 1)
    try:
        for levels in (1, 2):
            P, idx, g, Kp, Vp, scale, T, T1 = _setup(levels, False, seed=91)
            Q = sqz.to_device(P["Q"])
            a = sqz.centroid_lookup(g, Q, scale, T, T1, debug=True)
            b = sqz.centroid_lookup(g, Q, scale, T, T1, debug=True, comm=comm)
            torch.cuda.synchronize()
            for f in ("n_clusters", "n_keys"):
                assert torch.equal(getattr(a, f), getattr(b, f)), f
            B, H = Q.shape[:2]
            for bb in range(B):
                for h in range(H):
                    n = int(a.n_keys[bb, h])
                    assert torch.equal(a.key_idx[bb, h, :n], b.key_idx[bb, h, :n])
            O, LSE = sqz.sparse_attention(Q, Kp, Vp, g, a, sqz.to_device(P["Ku"]),
                                          sqz.to_device(P["Vu"]), scale, partial=True,
                                          out_dtype=sqz.SQZ_F32)
            Om, Lm = sqz.allgather_merge(comm, O, LSE, out_dtype=sqz.SQZ_F32)
            Oc, Lc = sqz.merge_partials(O.reshape(1, -1, idx.d), LSE.reshape(1, -1))
            torch.cuda.synchronize()
            assert torch.equal(Om.reshape(-1, idx.d), Oc) and torch.equal(Lm.reshape(-1), Lc)
            # the head-slice exchange of one rank is the merge of its own partial
            Oa, La = sqz.alltoall_merge(comm, O, LSE, out_dtype=sqz.SQZ_F32)
            torch.cuda.synchronize()
            assert Oa.shape == O.shape
            assert torch.equal(Oa.reshape(-1, idx.d), Oc) and torch.equal(La.reshape(-1), Lc)
    finally:
        comm.close()
