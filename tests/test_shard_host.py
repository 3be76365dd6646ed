"""Fixed-context sharding by cluster -- host side, no GPU.

* libsqz's host shard planner (sqz_shard_plan_compute, the product's partition
  logic; it needs no device) must partition every head's clusters and keys over
  the ranks, keep Level-1 subtrees intact and emit consistent local tables.
* The exchange protocol the GPU path implements -- per-level (m, D) statistics
  all-gathered and folded in rank order, local thresholds, (O, LSE) partials
  all-gathered and merged -- is run with world_size 2 over gloo, each rank
  computing its shard with the fp64 oracle, and must reproduce the unsharded
  oracle: the same selected clusters (band rule), the same attention output.
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2411_09688_b200 import calib, sqz

from helpers import oracle_problem

torch = pytest.importorskip("torch")


def _plan_all(idx, world):
    co = idx.child_off if idx.levels == 2 else None
    return [sqz.shard_plan(idx.H, idx.levels, idx.c1, idx.c2, idx.L, idx.key_off, co, r, world)
            for r in range(world)]


@pytest.mark.parametrize("levels,world", [(1, 1), (1, 2), (1, 3), (2, 2), (2, 4)])
def test_plan_partitions_clusters_and_keys(levels, world):
    P = oracle_problem(H=3, L=600, d=16, c2=24, c1=6 if levels == 2 else 0, seed=31, max_iters=8)
    idx = P["idx"]
    plans = _plan_all(idx, world)
    for h in range(idx.H):
        seen_c = np.concatenate([p["c2_src"][h][p["c2_src"][h] >= 0] for p in plans])
        assert np.array_equal(np.sort(seen_c), np.arange(idx.c2))
        seen_k = np.concatenate([p["key_src"][h][p["key_src"][h] >= 0] for p in plans])
        assert np.array_equal(np.sort(seen_k), np.arange(idx.L))
    for r, p in enumerate(plans):
        for h in range(idx.H):
            src = p["c2_src"][h]
            n = (src >= 0).sum()
            assert np.all(src[:n] >= 0) and np.all(src[n:] == -1), "padding only at the end"
            assert np.all(np.diff(src[:n]) > 0), "local ids keep the global order"
            # local N2 / key_off / key_src agree with the global tables
            np.testing.assert_array_equal(p["N2"][h][:n], idx.N2[h][src[:n]])
            assert np.all(p["N2"][h][n:] == 0)
            np.testing.assert_array_equal(np.diff(p["key_off"][h]), p["N2"][h])
            for i in range(n):
                g = src[i]
                a, b = p["key_off"][h][i], p["key_off"][h][i + 1]
                np.testing.assert_array_equal(p["key_src"][h][a:b],
                                              np.arange(idx.key_off[h][g], idx.key_off[h][g + 1]))
            if levels == 1:
                assert np.all(src[:n] % world == r)
            else:
                assert np.array_equal(p["c1_src"][h], np.arange(r, idx.c1, world))
                for j, g1 in enumerate(p["c1_src"][h]):
                    a, b = p["child_off"][h][j], p["child_off"][h][j + 1]
                    ga, gb = idx.child_off[h][g1], idx.child_off[h][g1 + 1]
                    np.testing.assert_array_equal(src[a:b], np.arange(ga, gb))
                    assert p["N1"][h][j] == idx.N1[h][g1]


def test_plan_rejects_bad_arguments():
    ko = np.array([[0, 2, 5]], np.int32)
    with pytest.raises(sqz.SqzError) as e:
        sqz.shard_plan(1, 1, 0, 2, 5, ko, None, 0, 3)  # 2 clusters < 3 ranks
    assert e.value.code == sqz.SQZ_ERR_INVALID_ARG
    with pytest.raises(sqz.SqzError):
        sqz.shard_plan(1, 1, 0, 2, 5, ko, None, 2, 2)  # rank out of range
    with pytest.raises(sqz.SqzError):
        sqz.shard_plan(1, 2, 1, 2, 5, ko, None, 0, 1)  # levels 2 without child_off


# ---------------------------------------------------------------------------
# world_size-2 exchange protocol over gloo
# ---------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fold(lse_parts):
    """Rank-order fold of per-shard log-denominators (the GPU folds (m, D) pairs;
    log-sum-exp is the same quantity)."""
    out = np.full(lse_parts.shape[1:], -np.inf)
    for p in lse_parts:
        out = np.logaddexp(out, p)
    return out


def _shard_lookup(dist, Q64, idx, plan, scale, T, T1):
    """Oracle arithmetic on this rank's shard + gloo all-gathers of the statistics."""
    B, H, n_q, d = Q64.shape
    world = dist.get_world_size()

    def gather(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return np.stack([o.numpy() for o in out])

    def level(C, N, rows_of, Tl):
        # rows_of[b][h] = local row ids scanned; returns (selected local rows, S-bar)
        s = {}
        lse = np.full((B, H, n_q), -np.inf)
        for b in range(B):
            for h in range(H):
                rows = rows_of[b][h]
                for t in range(n_q):
                    if len(rows):
                        sv, _, l = oracle.scores(Q64[b, h, t], C[h], N[h], scale, rows=rows)
                        s[b, h, t] = sv
                        lse[b, h, t] = l
        glse = _fold(gather(lse))
        sel, Sbar = {}, {}
        for b in range(B):
            for h in range(H):
                rows = np.asarray(rows_of[b][h], np.int64)
                acc = np.zeros(len(rows))
                for t in range(n_q):
                    if len(rows):
                        acc += np.exp(s[b, h, t][rows] - glse[b, h, t])
                Sb = acc / n_q
                Sbar[b, h] = (rows, Sb)
                sel[b, h] = rows[(Sb > Tl) | (Tl == 0)]
        return sel, Sbar

    def dense_C(Cg, src):
        return np.stack([np.where((src[h] >= 0)[:, None], Cg[h][np.maximum(src[h], 0)], 0.0)
                         for h in range(H)])

    C2 = dense_C(idx.C2, plan["c2_src"])
    surv1_global = None
    if idx.levels == 2:
        C1 = dense_C(idx.C1, plan["c1_src"])
        all1 = [[np.arange(plan["c1"]) for _ in range(H)] for _ in range(B)]
        sel1, _ = level(C1, plan["N1"], all1, T1)
        rows2 = [[np.concatenate([np.arange(plan["child_off"][h][p], plan["child_off"][h][p + 1])
                                  for p in sel1[b, h]] + [np.zeros(0, np.int64)]).astype(np.int64)
                  for h in range(H)] for b in range(B)]
        surv1 = np.zeros((B, H, idx.c1), bool)
        for b in range(B):
            for h in range(H):
                surv1[b, h, plan["c1_src"][h][sel1[b, h]]] = True
        surv1_global = gather(surv1).any(0)
    else:
        rows2 = [[np.arange(plan["c2"]) for _ in range(H)] for _ in range(B)]
        rows2 = [[r[plan["c2_src"][h][r] >= 0] for h, r in enumerate(rb)] for rb in rows2]
    sel2, Sb2 = level(C2, plan["N2"], rows2, T)
    sel_g = np.zeros((B, H, idx.c2), bool)
    S_g = np.full((B, H, idx.c2), np.nan)
    for b in range(B):
        for h in range(H):
            sel_g[b, h, plan["c2_src"][h][sel2[b, h]]] = True
            rows, Sb = Sb2[b, h]
            S_g[b, h, plan["c2_src"][h][rows]] = Sb
    return gather(sel_g).any(0), gather(S_g), surv1_global


def _worker(rank, world, port, case, errq):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        levels, prefill = case
        P = oracle_problem(H=2, L=480, d=16, c2=16, c1=4 if levels == 2 else 0, seed=57,
                           B=1 if prefill else 2, n_q=6 if prefill else 1, prefill=prefill,
                           n_u=5, max_iters=10)
        idx = P["idx"]
        scale = 1.0 / np.sqrt(idx.d)
        Q64 = oracle.to_f64(P["Q"])
        full = oracle.lookup(Q64, idx, scale, 0.0, 0.0)
        T1 = calib.weighted_threshold(full["Sbar1"], idx.N1[None], 0.5) if levels == 2 else 0.0
        full = oracle.lookup(Q64, idx, scale, 0.0, T1)
        T = calib.weighted_threshold(full["Sbar2"], idx.N2[None], 0.3)
        plan = sqz.shard_plan(idx.H, idx.levels, idx.c1, idx.c2, idx.L, idx.key_off,
                              idx.child_off if levels == 2 else None, rank, world)
        sel_u, S_parts, surv1 = _shard_lookup(dist, Q64, idx, plan, scale, T, T1)
        ref = oracle.lookup(Q64, idx, scale, T, T1, forced_l1=surv1)
        if surv1 is not None:
            ref1 = oracle.lookup(Q64, idx, scale, T, T1)
            bad1 = (surv1 != ref1["surv1"]) & ~oracle.band(ref1["Sbar1"], T1)
            assert not bad1.any(), "level-1 survivors differ outside the band"
        bad = (sel_u != ref["sel2"]) & ~oracle.band(ref["Sbar2"], T)
        assert not bad.any(), f"sharded selection differs outside the band: {np.argwhere(bad)[:3]}"
        # every cluster's S-bar comes from exactly its owner and equals the oracle's
        S_g = np.where(np.isnan(S_parts), 0.0, S_parts).sum(0)
        owned = ~np.isnan(S_parts).all(0)
        np.testing.assert_allclose(S_g[owned], ref["Sbar2"][owned], rtol=1e-9, atol=1e-15)
        # attention: each rank over its selected keys (user KV on rank 0), merged
        B, H = Q64.shape[:2]
        mask_full = oracle.keymask(idx, sel_u)
        mine = np.zeros((B, H, idx.L), bool)
        for h in range(H):
            ks = plan["key_src"][h]
            mine[:, h, idx.perm[h][ks[ks >= 0]]] = True
        mask = mask_full & mine
        K64, V64 = oracle.to_f64(P["fc"].K), oracle.to_f64(P["fc"].V)
        Ku = oracle.to_f64(P["Ku"]) if rank == 0 else None
        Vu = oracle.to_f64(P["Vu"]) if rank == 0 else None
        O_r, L_r, _ = oracle.attention(Q64, K64, V64, mask, Ku, Vu, prefill, scale)
        Ot = [torch.empty(O_r.shape, dtype=torch.float64) for _ in range(world)]
        Lt = [torch.empty(L_r.shape, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(Ot, torch.from_numpy(O_r))
        dist.all_gather(Lt, torch.from_numpy(L_r))
        d = idx.d
        O_m, L_m = oracle.merge(np.stack([o.numpy().reshape(-1, d) for o in Ot]),
                                np.stack([l.numpy().reshape(-1) for l in Lt]))
        O_ref, L_ref, rc = oracle.attention(Q64, K64, V64, mask_full, oracle.to_f64(P["Ku"]),
                                            oracle.to_f64(P["Vu"]), prefill, scale)
        assert rc == 0
        np.testing.assert_allclose(O_m, O_ref.reshape(-1, d), atol=1e-12)
        np.testing.assert_allclose(L_m, L_ref.reshape(-1), atol=1e-12)
        # head-slice exchange (the protocol of sqz_comm_alltoall_merge): rank r sends
        # its partial rows of heads [p Hs, (p+1) Hs) to rank p and merges, in rank
        # order, the rows of its own heads it receives from every rank
        Hs = H // world
        recv_O, recv_L, reqs = [None] * world, [None] * world, []
        for p in range(world):
            so = torch.from_numpy(np.ascontiguousarray(O_r[:, p * Hs:(p + 1) * Hs]))
            sl = torch.from_numpy(np.ascontiguousarray(L_r[:, p * Hs:(p + 1) * Hs]))
            if p == rank:
                recv_O[p], recv_L[p] = so, sl
                continue
            recv_O[p], recv_L[p] = torch.empty_like(so), torch.empty_like(sl)
            if rank < p:
                dist.send(so, p)
                dist.send(sl, p)
                dist.recv(recv_O[p], p)
                dist.recv(recv_L[p], p)
            else:
                dist.recv(recv_O[p], p)
                dist.recv(recv_L[p], p)
                dist.send(so, p)
                dist.send(sl, p)
        O_s, L_s = oracle.merge(np.stack([o.numpy().reshape(-1, d) for o in recv_O]),
                                np.stack([l.numpy().reshape(-1) for l in recv_L]))
        np.testing.assert_allclose(O_s, O_ref[:, rank * Hs:(rank + 1) * Hs].reshape(-1, d), atol=1e-12)
        np.testing.assert_allclose(L_s, L_ref[:, rank * Hs:(rank + 1) * Hs].reshape(-1), atol=1e-12)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        import traceback

        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


@pytest.mark.parametrize("case", [(1, False), (2, False), (1, True), (2, True)],
                         ids=["decode", "decode-hier", "prefill", "prefill-hier"])
def test_gloo_world2_exchange_reproduces_unsharded(case):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    msgs = []
    while not errq.empty():
        msgs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), "\n".join(msgs) or "worker failed"
