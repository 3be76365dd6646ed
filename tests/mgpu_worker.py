"""Worker of tests/test_gpu_multi.py (launched by torch.distributed.run, one
process per GPU, NCCL): the fixed context is sharded by cluster over the ranks
(interleaved, sqz_shard_plan_compute + sqz_index_shard), the lookup exchanges its
statistics with NCCL, each rank attends over its shard (the user KV on rank 0)
and the partials are merged -- all-gather for decode, the head-slice all-to-all
for prefill.  Every rank also runs the unsharded path on the full index and the
two must agree (selection up to the near-threshold band, outputs within the
bf16 tolerances)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_09688_b200 import calib, sqz, synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    dist.init_process_group("nccl", device_id=dev)
    H, L, d, c2, c1 = 4, 6000, 128, 200, 40
    fc = synth.fixed_context(H, L, d, c2, dtype=synth.BF16, seed=71, G1=c1)
    i2 = torch.from_numpy(synth.kmeans_init(H, L, c2, seed=72)).to(dev)
    i1 = torch.from_numpy(synth.kmeans_init(H, c2, c1, seed=73)).to(dev)
    idx, Kp, Vp, _ = sqz.cluster_keys(sqz.to_device(fc.K, dev), sqz.to_device(fc.V, dev), c2, i2, c1, i1,
                                      max_iters=20)
    scale = 1.0 / np.sqrt(d)
    loc, Kl, Vl = sqz.shard_index(idx, Kp, Vp, rank, world)
    comm = sqz.Comm(rank, world)
    bad = 0
    for prefill in (False, True):
        B, n_q, n_u = (1, 300, 300) if prefill else (3, 1, 40)
        Q = sqz.to_device(synth.prefill_queries(fc.mix, B, n_q, seed=74) if prefill else
                          synth.decode_queries(fc.mix, B, seed=74), dev)
        Ku, Vu = (sqz.to_device(a, dev) for a in synth.user_kv(fc.mix, B, n_u, seed=75))
        s = sqz.centroid_lookup(idx, Q, scale, 0.0, 0.0, debug=True)
        T1 = calib.weighted_threshold(s.dbg_S1.cpu().numpy(), idx.N1.cpu().numpy()[None], 0.5)
        s = sqz.centroid_lookup(idx, Q, scale, 0.0, T1, debug=True)
        T = calib.weighted_threshold(s.dbg_S.cpu().numpy(), idx.N2.cpu().numpy()[None], 0.2,
                                     total_weight=B * H * L)
        # unsharded reference on this GPU
        sf = sqz.centroid_lookup(idx, Q, scale, T, T1)
        O_ref, L_ref = sqz.sparse_attention(Q, Kp, Vp, idx, sf, Ku, Vu, scale, causal=prefill)
        # sharded path
        sl = sqz.centroid_lookup(loc, Q, scale, T, T1, comm=comm)
        Op, Lp = sqz.sparse_attention(Q, Kl, Vl, loc, sl, Ku if rank == 0 else None,
                                      Vu if rank == 0 else None, scale, causal=prefill, partial=True,
                                      out_dtype=sqz.SQZ_F32)
        k = sl.n_keys.to(torch.int64)
        dist.all_reduce(k)
        if not torch.equal(k, sf.n_keys.to(torch.int64)):
            print(f"rank {rank}: selected keys differ (prefill={prefill}): {k.tolist()} vs "
                  f"{sf.n_keys.tolist()}", flush=True)  # allowed only inside the band
        if prefill:
            O, LSE = sqz.alltoall_merge(comm, Op, Lp, out_dtype=sqz.SQZ_BF16)
            Hs = H // world
            O_ref, L_ref = O_ref[:, rank * Hs:(rank + 1) * Hs], L_ref[:, rank * Hs:(rank + 1) * Hs]
        else:
            O, LSE = sqz.allgather_merge(comm, Op, Lp, out_dtype=sqz.SQZ_BF16)
        torch.cuda.synchronize()
        err = (O.float() - O_ref.float()).abs().max().item()
        lerr = (LSE - L_ref).abs().max().item()
        print(f"rank {rank} prefill={prefill}: max|dO| {err:.3g} max|dLSE| {lerr:.3g}", flush=True)
        if not (err <= 2e-2 and lerr <= 1e-3):
            bad += 1
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
