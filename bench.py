#!/usr/bin/env python
"""Benchmark of the Squeezed Attention online hot path (lookup + sparse attention)
on B200 through libsqz's C ABI.

Default workload (BASELINE.json configs[1], the config the metric is quoted on):
LLaMA-2-7B-32K-shaped decode -- 32 heads x d128, 32K fixed context, 1024
centroids/head, single level, batch 1, 1K user KV, bf16, retention 30%
(3.1x KV-budget reduction).  One step = one decode token through one layer:
sqz_centroid_lookup + sqz_sparse_attention.  Metric: decode us/token/layer
(lower is better).  `--config cfg3` runs the 32K/1K-token prefill (tok/s per
layer), `cfg4` the 128K hierarchical decode at B=8, `cfg1` the tiny fp32 case.

Inputs: SYN-MIX v1 synthetic clustered keys; the index is built by
sqz_cluster_keys on the GPU; T is calibrated on 100 separate calibration queries
(App. C).  L2 is flushed (512 MB write) between timed steps; timing is CUDA
events on the launching stream, max over ranks.  The default run also measures
the cfg3 prefill (the other half of BASELINE's metric) and reports it as the
line's `prefill` object.  N > 1 (torchrun): cfg2/cfg3/cfg4 shard the heads over
the GPUs (no exchange on the hot path; strong scaling), cfg5 shards the fixed
context by cluster (statistics all-gather + (O, LSE) all-gather merge); every
input is a function of (seed, head) only, so the N-GPU run processes the inputs
of the 1-GPU run.

`--impl reference` times the CPU oracle (the paper-derived fp64 reference, the
only reference this build has) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(workload="cfg1: H=1 d64 L=1024 c=32 single-level decode B=1 n_u=16 fp32",
                 mode="decode", H=1, d=64, L=1024, c2=32, c1=0, B=1, n_q=1, n_u=16, dtype=0,
                 retention=0.3, cfgno=1),
    "cfg2": dict(workload="cfg2: LLaMA-2-7B-32K decode, H=32 d128, L=32768, c=1024 single-level, "
                          "B=1, n_u=1024, bf16, retention 30% (3.1x KV budget reduction)",
                 mode="decode", H=32, d=128, L=32768, c2=1024, c1=0, B=1, n_q=1, n_u=1024,
                 dtype=1, retention=0.3, cfgno=2, shard="heads"),
    "cfg3": dict(workload="cfg3: LongChat-7B-32K prefill, H=32 d128, L=32768, c=1024, n_q=n_u=1024 "
                          "causal, bf16, retention 30% (prefill-calibrated)",
                 mode="prefill", H=32, d=128, L=32768, c2=1024, c1=0, B=1, n_q=1024, n_u=1024,
                 dtype=1, retention=0.3, cfgno=3, shard="heads"),
    "cfg4": dict(workload="cfg4: 128K hierarchical decode, H=32 d128, L=131072, c1=1311, c2=6554, "
                          "L1 prunes 50%, retention 10%, B=8, n_u=1024, bf16; heads sharded over the GPUs",
                 mode="decode", H=32, d=128, L=131072, c2=6554, c1=1311, B=8, n_q=1, n_u=1024,
                 dtype=1, retention=0.1, cfgno=4, shard="heads", device_gen=True),
    "cfg5": dict(workload="cfg5: LWM-Text-Chat-1M decode, H=32 d128, L=1048576, c1=10486, c2=52429 "
                          "hierarchical, L1 prunes 50%, retention 10%, B=1, n_u=1024, bf16; fixed context "
                          "sharded by cluster over the GPUs (stats all-gather + (O, LSE) all-gather merge)",
                 mode="decode", H=32, d=128, L=1048576, c2=52429, c1=10486, B=1, n_q=1, n_u=1024,
                 dtype=1, retention=0.1, cfgno=5, shard="clusters", device_gen=True, kmeans_iters=10),
    "cfg5h3": dict(workload="cfg5 with THREE levels (P:269): LWM-Text-Chat-1M decode, H=32 d128, "
                            "L=1048576, c0=2097, c1=10486, c2=52429; Level 0 keeps 50% and Level 1 25% of "
                            "the keys, retention 10%, B=1, n_u=1024, bf16",
                   mode="decode", H=32, d=128, L=1048576, c2=52429, c1=10486, c0=2097, B=1, n_q=1,
                   n_u=1024, dtype=1, retention=0.1, cfgno=5, shard="heads", device_gen=True,
                   kmeans_iters=10),
    "cfg5p": dict(workload="cfg5 prefill: LWM-Text-Chat-1M, H=32 d128, L=1048576, c1=10486, c2=52429 "
                           "hierarchical, retention 10%, n_q=n_u=4096 causal, bf16; fixed context "
                           "sharded by cluster over the GPUs",
                  mode="prefill", H=32, d=128, L=1048576, c2=52429, c1=10486, B=1, n_q=4096, n_u=4096,
                  dtype=1, retention=0.1, cfgno=5, shard="clusters", device_gen=True, kmeans_iters=10),
}


def metric_of(cfg):
    if cfg["mode"] == "decode":
        return "decode_us_per_token_per_layer", "us/token/layer", False
    return "prefill_tokens_per_s_per_layer", "tok/s/layer", True


# --------------------------------------------------------------------------
# clocks sampler (NVML, during the timed region)
# --------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting"}

    def __init__(self, dev_index, period=0.002):
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)
# --------------------------------------------------------------------------
def cpu_oracle_run(cfg, steps=None, warmup=0, seconds=12.0, h_sample=4):
    """Time the fp64 oracle as it stands on a bounded sample: `h_sample` of the H
    heads at full L / c / n_u, index from the oracle's own K-means (10 Lloyd
    iterations, same seeded init as the GPU arm), T calibrated by the oracle on 16
    calibration queries.  A step = oracle lookup + oracle attention for one decode
    token (or one prefill block of 64 query rows) on the sample, scaled to the full
    head count.  Returns (value in the metric's unit, sample description, cores,
    per-step seconds)."""
    import oracle
    from paper_2411_09688_b200 import calib, synth

    hs = min(h_sample, cfg["H"])
    # contexts beyond 32K keys: a 32K-key sample with the same centroid fractions,
    # time scaled linearly in L (lookup rows and selected keys are both ~ L)
    Ls = min(cfg["L"], 32768)
    fL = cfg["L"] / Ls
    L_full = cfg["L"]
    c2s = int(np.ceil(cfg["c2"] / fL))
    c1s = int(np.ceil(cfg["c1"] / fL)) if cfg["c1"] else 0
    c0s = int(np.ceil(cfg.get("c0", 0) / fL)) if cfg.get("c0", 0) else 0
    cfg = dict(cfg, L=Ls, c2=c2s, c1=c1s, c0=c0s)
    fc = synth.fixed_context(hs, cfg["L"], cfg["d"], cfg["c2"], dtype=cfg["dtype"],
                             seed=1000 + cfg["cfgno"], G1=cfg["c1"])
    K, V = fc.K, fc.V
    init2 = synth.kmeans_init(hs, cfg["L"], cfg["c2"], seed=2000 + cfg["cfgno"])
    init1 = (synth.kmeans_init(hs, cfg["c2"], cfg["c1"], seed=2100 + cfg["cfgno"])
             if cfg["c1"] else None)
    init0 = (synth.kmeans_init(hs, cfg["c1"], cfg["c0"], seed=2200 + cfg["cfgno"])
             if cfg["c0"] else None)
    idx = oracle.build_index(K, cfg["c2"], init2, cfg["c1"], init1, max_iters=10, c0=cfg["c0"],
                             init0=init0)
    scale = 1.0 / np.sqrt(cfg["d"])
    mix = fc.mix
    if cfg["mode"] == "decode":
        Qc = synth.decode_queries(mix, 16, seed=3000 + cfg["cfgno"], dtype=cfg["dtype"])[:, :hs]
        Qt = synth.decode_queries(mix, 32, seed=4000 + cfg["cfgno"], dtype=cfg["dtype"])[:, :hs]
        Ku, Vu = synth.user_kv(mix, 1, cfg["n_u"], seed=5000 + cfg["cfgno"], dtype=cfg["dtype"])
    else:
        Qc = synth.prefill_queries(mix, 2, cfg["n_q"], seed=3000 + cfg["cfgno"],
                                   dtype=cfg["dtype"])[:, :hs]
        Qt = synth.prefill_queries(mix, 1, cfg["n_q"], seed=4000 + cfg["cfgno"],
                                   dtype=cfg["dtype"])[:, :hs]
        Ku, Vu = synth.user_kv(mix, 1, cfg["n_u"], seed=5000 + cfg["cfgno"], dtype=cfg["dtype"])
    Ku64, Vu64 = oracle.to_f64(Ku[:, :hs]), oracle.to_f64(Vu[:, :hs])
    K64, V64 = oracle.to_f64(K), oracle.to_f64(V)
    T1 = T0 = 0.0
    Qc64 = oracle.to_f64(Qc)
    tw = Qc64.shape[0] * hs * cfg["L"]
    if idx.levels == 3:
        r = oracle.lookup(Qc64, idx, scale, 0.0, 0.0)
        T0 = calib.weighted_threshold(r["Sbar0"], idx.N0[None], 0.5)
        r = oracle.lookup(Qc64, idx, scale, 0.0, 0.0, T0=T0)
        T1 = calib.weighted_threshold(r["Sbar1"], idx.N1[None], 0.25, total_weight=tw)
    elif idx.levels == 2:
        r = oracle.lookup(Qc64, idx, scale, 0.0, 0.0)
        T1 = calib.weighted_threshold(r["Sbar1"], idx.N1[None], 0.5)
    r = oracle.lookup(Qc64, idx, scale, 0.0, T1, T0=T0)
    T = calib.weighted_threshold(r["Sbar2"], idx.N2[None], cfg["retention"],
                                 total_weight=r["Sbar2"].shape[0] * hs * cfg["L"])
    Qt64 = oracle.to_f64(Qt)

    def step(i):
        if cfg["mode"] == "decode":
            q = Qt64[i % Qt64.shape[0]][None]
            out = oracle.lookup(q, idx, scale, T, T1, T0=T0)
            mask = oracle.keymask(idx, out["sel2"])
            oracle.attention(q, K64, V64, mask, Ku64, Vu64, False, scale)
        else:
            # prefill sample: the full lookup (needs all rows), attention on 64 rows
            out = oracle.lookup(Qt64, idx, scale, T, T1, T0=T0)
            mask = oracle.keymask(idx, out["sel2"])
            rows = np.linspace(0, cfg["n_q"] - 1, 64).astype(np.int32)
            oracle.attention(Qt64[:, :, rows], K64, V64, mask, Ku64, Vu64, True, scale, qpos=rows,
                             n_q_total=cfg["n_q"])

    for i in range(warmup):
        step(i)
    times = []
    t_start = time.perf_counter()
    i = 0
    while True:
        t0 = time.perf_counter()
        step(i)
        times.append(time.perf_counter() - t0)
        i += 1
        if steps is not None and i >= steps:
            break
        if steps is None and (time.perf_counter() - t_start > seconds or i >= 2000) and i >= 3:
            break
    per = float(np.mean(times)) * fL
    scale_h = cfg["H"] / hs
    if cfg["mode"] == "decode":
        value = per * scale_h * 1e6 / cfg["B"] if cfg["B"] == 1 else per * scale_h * 1e6
        sample = (f"{hs} of {cfg['H']} heads, L={cfg['L']} (x{fL:g} to L={L_full}), c={cfg['c2']}, "
                  f"c1={cfg['c1']}, n_u={cfg['n_u']}; "
                  f"oracle K-means index (10 Lloyd iters); {len(times)} decode tokens x 1 layer; "
                  f"time x{scale_h:g} to all heads")
    else:
        # lookup on all n_q rows + attention on 64 rows: scale the attention part
        value = cfg["n_q"] / (per * scale_h * (cfg["n_q"] / 64.0))
        sample = (f"{hs} of {cfg['H']} heads, L={cfg['L']} (x{fL:g} to L={L_full}); lookup over all "
                  f"{cfg['n_q']} rows + attention on 64 "
                  f"of {cfg['n_q']} rows; {len(times)} prefill blocks; scaled x{scale_h:g} heads and "
                  f"x{cfg['n_q'] / 64:g} rows (upper bound on oracle throughput)")
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return value, sample, cores, times


def oracle_parity(sqz, gidx, q, sel, O, LSE, T, T1, scale, K0, V0, Ku0, Vu0, loc, causal,
                  rows_sample=None, T0=0.0):
    """Rank 0, after the timed region (part of the oracle leg): the fp64 oracle
    re-runs the lookup of head 0 on the GPU-built global tables and the
    attention of that head on the selected keys, and compares them with the GPU
    output of the same input (band rule 1e-5, bf16 O max-abs 2e-2, LSE 1e-3;
    DESIGN.md parity rules).  `loc` = rank 0's index (a shard in cluster mode:
    only its clusters' selections are compared, the attention output is the
    merged one).  Returns a small dict for the bench line."""
    import torch

    import oracle

    def bits(t):
        return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16) \
            if t.dtype == torch.bfloat16 else t.contiguous().cpu().numpy()

    h = 0
    sub = oracle.Index(levels=gidx.levels, dtype=gidx.dtype, H=1, L=gidx.L, d=gidx.d, c2=gidx.c2,
                       C2=oracle.to_f64(bits(gidx.C2[h:h + 1])), N2=gidx.N2[h:h + 1].cpu().numpy(),
                       key_off=gidx.key_off[h:h + 1].cpu().numpy(),
                       perm=gidx.perm[h:h + 1].cpu().numpy())
    if gidx.levels >= 2:
        sub.c1 = gidx.c1
        sub.C1 = oracle.to_f64(bits(gidx.C1[h:h + 1]))
        sub.N1 = gidx.N1[h:h + 1].cpu().numpy()
        sub.child_off = gidx.child_off[h:h + 1].cpu().numpy()
    if gidx.levels == 3:
        sub.c0 = gidx.c0
        sub.C0 = oracle.to_f64(bits(gidx.C0[h:h + 1]))
        sub.N0 = gidx.N0[h:h + 1].cpu().numpy()
        sub.child_off0 = gidx.child_off0[h:h + 1].cpu().numpy()
    B, _, n_q, d = q.shape
    Q64 = oracle.to_f64(bits(q[:, h:h + 1]))
    out = {"head": h, "queries": int(B * n_q)}
    sharded = loc.L_total > 0
    forced = forced0 = None
    if gidx.levels == 3:
        ref0 = oracle.lookup(Q64, sub, scale, T, T1, T0=T0)
        g0 = sel.l0_surv[:, h:h + 1].cpu().numpy().astype(bool)
        out["level0_outside_band"] = int(((g0 != ref0["surv0"]) & ~oracle.band(ref0["Sbar0"], T0)).sum())
        forced0 = g0
    if gidx.levels >= 2:
        ref1 = oracle.lookup(Q64, sub, scale, T, T1, T0=T0, forced_l0=forced0)
        g1 = ref1["surv1"].copy()
        mine = np.arange(gidx.c1) if not sharded else loc.c1_src[h].cpu().numpy()
        gl = sel.l1_surv[:, h].cpu().numpy().astype(bool)[:, :len(mine)]
        g1[:, 0, mine] = gl
        flips = (g1 != ref1["surv1"])
        band1 = oracle.band(ref1["Sbar1"], T1)
        out["level1_outside_band"] = int((flips & ~band1).sum())
        forced = g1
    ref = oracle.lookup(Q64, sub, scale, T, T1, forced_l1=forced, T0=T0, forced_l0=forced0)
    cl, n = sel.clusters[:, h].cpu().numpy(), sel.n_clusters[:, h].cpu().numpy()
    src = None if not sharded else loc.c2_src[h].cpu().numpy()
    gsel = np.zeros_like(ref["sel2"])
    own = np.zeros(gidx.c2, bool)
    own[np.arange(gidx.c2) if src is None else src[src >= 0]] = True
    for b in range(B):
        ids = cl[b, :n[b]]
        gsel[b, 0, ids if src is None else src[ids]] = True
    band = oracle.band(ref["Sbar2"], T)
    diff = (gsel != ref["sel2"]) & own[None, None, :]
    out["selection_outside_band"] = int((diff & ~band).sum())
    out["selection_in_band_flips"] = int((diff & band).sum())
    out["clusters_compared"] = int(own.sum()) * B
    any_band = bool((band & ref["sel2"]).any() or (band & ~ref["sel2"]).any())
    if out["selection_outside_band"] == 0 and not (any_band and sharded):
        # mask = the GPU's selection (unsharded) or the oracle's (sharded, no band clusters)
        m = gsel if not sharded else ref["sel2"]
        mask = oracle.keymask(sub, m) if sub.assign2 is not None else None
        if mask is None:  # GPU-built tables: members from key_off / perm
            mask = np.zeros((B, 1, gidx.L), bool)
            for b in range(B):
                for i in np.nonzero(m[b, 0])[0]:
                    mask[b, 0, sub.perm[0][sub.key_off[0, i]:sub.key_off[0, i + 1]]] = True
        Ku64 = None if Ku0 is None else oracle.to_f64(bits(Ku0))[:, None]
        Vu64 = None if Vu0 is None else oracle.to_f64(bits(Vu0))[:, None]
        qs = Q64 if rows_sample is None else Q64[:, :, rows_sample]
        Oref, Lref, rc = oracle.attention(qs, oracle.to_f64(bits(K0))[None], oracle.to_f64(bits(V0))[None],
                                          mask, Ku64, Vu64, causal, scale, qpos=rows_sample,
                                          n_q_total=n_q)
        Og = O[:, h:h + 1].float().cpu().numpy()
        Lg = LSE[:, h:h + 1].cpu().numpy()
        if rows_sample is not None:
            Og, Lg = Og[:, :, rows_sample], Lg[:, :, rows_sample]
        out["attention_rows"] = int(Og.shape[0] * Og.shape[2])
        out["O_max_abs"] = float(np.abs(Og - Oref).max())
        out["O_rel_l2"] = float(np.linalg.norm(Og - Oref) / max(np.linalg.norm(Oref), 1e-30))
        out["LSE_max_abs"] = float(np.abs(Lg - Lref).max())
        tol_o = 2e-2 if gidx.dtype == 1 else 1e-4
        out["ok"] = bool(rc == 0 and out["O_max_abs"] <= tol_o and out["LSE_max_abs"] <= 1e-3
                         and out.get("level1_outside_band", 0) == 0)
    else:
        out["ok"] = out["selection_outside_band"] == 0 and out.get("level1_outside_band", 0) == 0
        out["attention"] = "skipped: near-threshold clusters on a sharded run"
    return out


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def selection_quality(sqz, idx, Qt, Kp, scale, T, T1, n_in, B, dev, T0=0.0):
    """sqz_selection_diagnostics over the first n_in test inputs: App. A's top-1%
    cumulative attention score per (b,h) and App. D's ideal lookup at
    the same T against the centroid selection at matched budget."""
    import torch

    sel = sqz.Selection.empty(idx, B, 1, False, dev, key_idx=False)
    acc = {k: [] for k in ("skew", "mass_sel", "mass_ideal", "recall", "n_T", "mass_T", "k")}
    for i in range(n_in):
        sqz.centroid_lookup(idx, Qt[i], scale, T, T1, sel=sel, T0=T0)
        out = sqz.selection_diagnostics(idx, Qt[i], Kp, sel, scale, 0.01, T)
        for k, v in out.items():
            acc[k].append(v.float().cpu().numpy().ravel())
        acc["k"].append(sel.n_keys.float().cpu().numpy().ravel())
    torch.cuda.synchronize()
    a = {k: np.concatenate(v) for k, v in acc.items()}
    L = idx.L
    sk = a["skew"]
    ret = a["k"] / L
    corr = float(np.corrcoef(sk, ret)[0, 1]) if sk.std() > 0 and ret.std() > 0 else None
    r4 = lambda x: round(float(x), 4)
    return {"rows": int(sk.size), "top_frac": 0.01,
            "skew_top1pct": {"min": r4(sk.min()), "median": r4(np.median(sk)), "max": r4(sk.max())},
            "corr_skew_vs_retention": None if corr is None else r4(corr),
            "mass_retrieved_mean": r4(a["mass_sel"].mean()),
            "mass_ideal_same_budget_mean": r4(a["mass_ideal"].mean()),
            "recall_vs_ideal_same_budget_mean": r4(a["recall"].mean()),
            "ideal_at_T_retention_mean": r4((a["n_T"] / L).mean()),
            "ideal_at_T_mass_mean": r4(a["mass_T"].mean()),
            "what": "sqz_selection_diagnostics (App. A skewness; App. D ideal lookup), fixed keys only"}


def capture_graph(fn):
    """Capture `fn` (a sequence of libsqz calls on the current stream) into a CUDA
    graph; one eager warm-up call first fills the library's host-side caches."""
    import torch

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="thread_local"):
        fn()
    return g


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def traffic_for(workload_key, kernel):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d.get(workload_key, {}).get(kernel)
    except Exception:
        return None


def run_gpu(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2411_09688_b200 import calib, sqz, synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    sqz.device_check()
    dt = cfg["dtype"]
    H, d, L, c2, c1, B, n_q, n_u = (cfg[k] for k in ("H", "d", "L", "c2", "c1", "B", "n_q", "n_u"))
    c0 = cfg.get("c0", 0)
    scale = 1.0 / float(np.sqrt(d))
    # ---- sharding of the work over the ranks ----
    shard = cfg.get("shard", "replicas") if world > 1 else "none"
    cno = cfg["cfgno"]
    if shard == "heads":  # H/g heads per GPU, no exchange on the hot path
        if H % world:
            raise SystemExit(f"{H} heads do not split over {world} GPUs")
        heads = list(range(rank * H // world, (rank + 1) * H // world))
    else:
        heads = list(range(H))
    Hl = len(heads)
    kiters = cfg.get("kmeans_iters", args.kmeans_iters) if args.kmeans_iters_set is None \
        else args.kmeans_iters_set
    # ---- offline: data + index (not timed) ----
    # Every input is a function of (config seed, head) only, so the N-GPU run
    # processes exactly the inputs of the 1-GPU run: head shards slice them,
    # cluster shards split ONE global index (sqz_shard_plan_compute +
    # sqz_index_shard: Level-1 cluster p on rank p mod g, subtrees intact).
    if cfg.get("device_gen"):
        mix = synth.device_mixture(H, c2, d, G1=c1, seed=1000 + cno, device=dev)
        K, V = synth.device_keys(mix, L, seed=1000 + cno, dtype=dt, heads=heads)
        init2 = synth.device_kmeans_init(H, L, c2, seed=2000 + cno, device=dev, heads=heads)
        init1 = synth.device_kmeans_init(H, c2, c1, seed=2100 + cno, device=dev, heads=heads) \
            if c1 else None
        init0 = synth.device_kmeans_init(H, c1, c0, seed=2200 + cno, device=dev, heads=heads) \
            if c0 else None
    else:
        fc = synth.fixed_context(H, L, d, c2, dtype=dt, seed=1000 + cno, G1=c1)
        mix = fc.mix
        K, V = sqz.to_device(fc.K[heads], dev), sqz.to_device(fc.V[heads], dev)
        init2 = torch.from_numpy(synth.kmeans_init(H, L, c2, seed=2000 + cno)[heads]).to(dev)
        init1 = (torch.from_numpy(synth.kmeans_init(H, c2, c1, seed=2100 + cno)[heads]).to(dev)
                 if c1 else None)
        init0 = (torch.from_numpy(synth.kmeans_init(H, c1, c0, seed=2200 + cno)[heads]).to(dev)
                 if c0 else None)
        del fc
    t0 = time.time()
    idx, Kp, Vp, iters = sqz.cluster_keys(K, V, c2, init2, c1, init1, max_iters=kiters,
                                          assign_mode={"auto": sqz.KMEANS_AUTO, "exact": sqz.KMEANS_EXACT,
                                                       "tensor": sqz.KMEANS_TENSOR}[args.kmeans_mode],
                                          c0=c0, init0=init0)
    torch.cuda.synchronize()
    t_index = time.time() - t0
    # host copy of the sampled head (original order) for the oracle parity check
    par_head = 0
    K0 = K[par_head].contiguous().cpu() if rank == 0 else None
    V0 = V[par_head].contiguous().cpu() if rank == 0 else None
    del K, V
    gidx = idx  # the global (unsharded) index: rank 0's parity check reads its tables
    if shard == "clusters":
        idx, Kp_l, Vp_l = sqz.shard_index(idx, Kp, Vp, rank, world)
        torch.cuda.synchronize()
        if rank != 0:
            gidx = None
        del Kp, Vp
        Kp, Vp = Kp_l, Vp_l
        torch.cuda.empty_cache()
    comm = sqz.Comm(rank, world) if shard == "clusters" else None

    # reductions travel on the device with NCCL, on the host with gloo (shared-GPU dry run)
    red_dev = "cpu" if world > 1 and dist.get_backend() == "gloo" else dev

    def allsum(x):
        if world == 1 or shard not in ("heads", "clusters"):
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t)
        return float(t.item())

    # ---- queries: 100 calibration (App. C) + test inputs, user KV ----
    if cfg["mode"] == "decode":
        n_cal, n_inputs = (100, 100) if not cfg.get("device_gen") else (32, 16)
    else:
        n_cal, n_inputs = 4, 4
    if cfg.get("device_gen"):
        if cfg["mode"] == "decode":
            Qc = synth.device_decode_queries(mix, n_cal, seed=3000 + cno, dtype=dt, heads=heads)
            Qt = synth.device_decode_queries(mix, n_inputs * B, seed=4000 + cno, dtype=dt,
                                             heads=heads).view(n_inputs, B, Hl, 1, d)
        else:
            Qc = synth.device_prefill_queries(mix, 1, n_q, seed=3000 + cno, dtype=dt, heads=heads)
            n_inputs = 2
            Qt = synth.device_prefill_queries(mix, n_inputs * B, n_q, seed=4000 + cno, dtype=dt,
                                              heads=heads).view(n_inputs, B, Hl, n_q, d)
        Ku, Vu = synth.device_user_kv(mix, B, n_u, seed=5000 + cno, dtype=dt, heads=heads)
    else:
        if cfg["mode"] == "decode":
            Qc = sqz.to_device(synth.decode_queries(mix, n_cal, seed=3000 + cno, dtype=dt)[:, heads],
                               dev)
            Qt = sqz.to_device(synth.decode_queries(mix, n_inputs * B, seed=4000 + cno,
                                                    dtype=dt)[:, heads], dev).view(n_inputs, B, Hl, 1, d)
        else:
            Qc = sqz.to_device(synth.prefill_queries(mix, n_cal, n_q, seed=3000 + cno,
                                                     dtype=dt)[:, heads], dev)
            Qt = sqz.to_device(synth.prefill_queries(mix, n_inputs * B, n_q, seed=4000 + cno,
                                                     dtype=dt)[:, heads], dev).view(n_inputs, B, Hl, n_q, d)
        Ku, Vu = (sqz.to_device(a[:, heads], dev)
                  for a in synth.user_kv(mix, B, n_u, seed=5000 + cno, dtype=dt))
    # one user-KV cache [2 (K, V), B, H, n_u, d]: the end-to-end step appends a token's K
    # and V rows with ONE device copy
    KVu = torch.stack([Ku, Vu])
    Ku, Vu = KVu[0], KVu[1]
    Ku0 = Ku[:, par_head].contiguous().cpu() if rank == 0 else None
    Vu0 = Vu[:, par_head].contiguous().cpu() if rank == 0 else None
    if shard == "clusters" and rank != 0:
        Ku = Vu = KVu = None  # the user KV partial is computed once, on rank 0
    n_u_r = 0 if Ku is None else n_u
    Bc = Qc.shape[0]
    # ---- calibration of the global thresholds (R12, R13) ----
    # bisection on the all-reduced retained weight (integer sums, exact in fp64):
    # the same T at every N, so the N-GPU run selects what the 1-GPU run selects
    T1 = T0 = 0.0
    if c0:  # three levels: Level 0 keeps 50% of the keys, Level 1 25% (R13 extended)
        s = sqz.centroid_lookup(idx, Qc, scale, 0.0, 0.0, debug=True, comm=comm)
        T0 = calib.distributed_threshold(s.dbg_S0, idx.N0[None], 0.5, allsum(float(
            Bc * idx.N0.sum())), allreduce=allsum)
        s = sqz.centroid_lookup(idx, Qc, scale, 0.0, 0.0, debug=True, comm=comm, T0=T0)
        T1 = calib.distributed_threshold(s.dbg_S1, idx.N1[None], 0.25, allsum(float(
            Bc * idx.N1.sum())), allreduce=allsum)
    elif c1:
        s = sqz.centroid_lookup(idx, Qc, scale, 0.0, 0.0, debug=True, comm=comm)
        T1 = calib.distributed_threshold(s.dbg_S1, idx.N1[None], 0.5, allsum(float(
            Bc * idx.N1.sum())), allreduce=allsum)
    s = sqz.centroid_lookup(idx, Qc, scale, 0.0, T1, debug=True, comm=comm, T0=T0)
    T = calib.distributed_threshold(s.dbg_S, idx.N2[None], cfg["retention"], float(Bc * H * L),
                                    allreduce=allsum)
    del s, Qc
    # ---- per-step work: selection sizes for the algorithmic-byte count ----
    # the batch-shared pass reads the run-length selection (clusters + key_pref) only
    shared_attn = (cfg["mode"] == "decode" and B >= 2 and d == 128 and dt == 1
                   and not args.attn_per_row)
    # single-level prefill reads the run-length selection (cfg3: lookup -6 us, attention +5 us,
    # 285.7 -> 283.8 us per step); hierarchical prefill (cfg5p: 14.49 vs 14.3 ms) and decode
    # (the step: 55.2 vs 51.9 us) keep the expanded key list
    runs = args.sel_runs == "on" or (args.sel_runs == "auto" and cfg["mode"] == "prefill"
                                      and not cfg.get("c1"))
    sel = sqz.Selection.empty(idx, B, n_q, False, dev, key_idx=not (runs or shared_attn))
    esz = 2 if dt == 1 else 4
    ks, kus = [], []
    c2l = idx.c2
    for i in range(n_inputs):
        sqz.centroid_lookup(idx, Qt[i], scale, T, T1, sel=sel, comm=comm, T0=T0)
        ks.append(int(sel.n_keys.sum()))
        # keys in the per-head UNION of the B selections (what the batch-shared pass reads)
        ar = torch.arange(c2l, device=dev)
        ids = torch.where(ar[None, None, :] < sel.n_clusters[:, :, None], sel.clusters,
                          torch.full_like(sel.clusters, c2l)).long()
        um = torch.zeros(B, Hl, c2l + 1, dtype=torch.bool, device=dev)
        um.scatter_(2, ids, True)
        kus.append(int((um[:, :, :c2l].any(0) * idx.N2).sum()))
    torch.cuda.synchronize()
    k_mean = float(np.mean(ks))  # this rank's selected keys per step
    ku_mean = float(np.mean(kus))  # this rank's union keys per step (= k_mean when B = 1)
    k_glob = allsum(k_mean)
    # algorithmic bytes / flops of THIS rank
    c1l, c2l = idx.c1, idx.c2
    lookup_rows = c2l + c1l  # rows scanned per head (hier: L2 restricted, approximated below)
    # lookup bytes: the first level's rows once per head (the batch shares the scan),
    # deeper levels' REALIZED candidate rows per (b, h) (non-NaN debug scores)
    first = {1: c2l, 2: c1l, 3: idx.c0}[idx.levels]
    bytes_lookup = Hl * first * (d * esz + 4)
    if idx.levels >= 2:
        sd = sqz.centroid_lookup(idx, Qt[0], scale, T, T1, debug=True, comm=comm, T0=T0)
        deeper = int((~torch.isnan(sd.dbg_S)).sum())
        if idx.levels == 3:
            deeper += int((~torch.isnan(sd.dbg_S1)).sum())
        bytes_lookup += deeper * (d * esz + 4)
        del sd
    bytes_attn = k_mean * 2 * d * esz + B * Hl * n_u_r * 2 * d * esz + 2 * B * Hl * n_q * d * esz
    bytes_attn_perq = bytes_attn
    if shared_attn:  # NEXT-1: each selected key is read once for all the queries that chose it
        bytes_attn = ku_mean * 2 * d * esz + B * Hl * n_u_r * 2 * d * esz + 2 * B * Hl * n_q * d * esz
    flops_attn = 4.0 * n_q * d * k_mean + (4.0 * d * B * Hl * (n_q * n_u_r - n_q * (n_q - 1) / 2)
                                          if n_u_r else 0.0)
    flops_lookup = 2.0 * B * Hl * n_q * lookup_rows * d
    # cluster-sharded prefill: each rank ends with its head slice (head-slice all-to-all)
    a2a = comm is not None and cfg["mode"] == "prefill"
    Ho = Hl // world if a2a else Hl
    O = torch.empty(B, Ho, n_q, d, dtype=sqz.torch_dtype(dt), device=dev)
    LSE = torch.empty(B, Ho, n_q, dtype=torch.float32, device=dev)
    Op = torch.empty(B, Hl, n_q, d, dtype=torch.float32, device=dev) if comm else None
    Lp = torch.empty(B, Hl, n_q, dtype=torch.float32, device=dev) if comm else None
    # L2 flush between timed steps: a 512 MB write (4x the 126 MB L2).  The write
    # leaves the L2 full of DIRTY lines whose write-back (~126 MB of DRAM writes)
    # would otherwise land inside the next timed step; with --flush write+read a
    # 512 MB read follows (untimed), so the timed step starts from an L2 holding
    # clean, unrelated lines -- the inputs are cold either way.
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    rflush_buf = (torch.ones(128 << 20, dtype=torch.float32, device=dev)
                  if args.flush == "write+read" else None)

    class _Flush:
        @staticmethod
        def zero_():
            flush_buf.zero_()
            if rflush_buf is not None:
                rflush_buf.amax()
    flush = _Flush()
    causal = cfg["mode"] == "prefill"

    def attend_into(q, Oo, Lo, sl=None):
        sl = sel if sl is None else sl
        if comm is None:
            sqz.sparse_attention(q, Kp, Vp, idx, sl, Ku, Vu, scale, causal=causal, O=Oo, LSE=Lo,
                                 per_row=args.attn_per_row)
        else:  # partial over this shard, then the all-gather merge (P:361-363 across GPUs)
            sqz.sparse_attention(q, Kp, Vp, idx, sl, Ku, Vu, scale, causal=causal, partial=True,
                                 out_dtype=sqz.SQZ_F32, O=Op, LSE=Lp, per_row=args.attn_per_row)
            if a2a:  # prefill: each rank merges only its head slice
                sqz.alltoall_merge(comm, Op, Lp, out_dtype=dt, O=Oo, LSE=Lo)
            else:
                sqz.allgather_merge(comm, Op, Lp, out_dtype=dt, O=Oo, LSE=Lo)

    def attend(q):
        attend_into(q, O, LSE)

    # decode through sqz_decode_step (one call: for one single-level query row the
    # lookup hands each row's selection to the attention kernel through flags and
    # attends the user KV itself) unless the fixed context is sharded (the
    # exchange needs the two calls)
    step_applies = cfg["mode"] == "decode" and comm is None and idx.levels == 1 and B == 1
    use_step = step_applies and args.decode_path in ("step", "auto")
    step_ws = None
    if use_step:
        nb = sqz.ctypes.c_size_t(0)
        sqz._check(sqz.lib().sqz_decode_step_workspace(sqz.ctypes.byref(idx.struct()), B, n_u_r,
                                                       sqz.ctypes.byref(nb)))
        step_ws = sqz.workspace(nb.value, dev)

    def step_into(q, Oo, Lo):
        if use_step:
            sqz.decode_step(idx, q, Kp, Vp, Ku, Vu, scale, T, T1, sel=sel, O=Oo, LSE=Lo, ws=step_ws,
                            T0=T0)
        else:
            sqz.centroid_lookup(idx, q, scale, T, T1, sel=sel, comm=comm, T0=T0)
            attend_into(q, Oo, Lo)

    def step(i):
        step_into(Qt[i % n_inputs], O, LSE)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    K_ = args.steps
    # The step is replayed as a CUDA graph (one per test input): the two kernels
    # are chained by programmatic dependent launch and no host launch latency
    # sits between them.  The eager (per-call) figure is reported beside it.
    graphs = [capture_graph(lambda i=i: step(i)) for i in range(n_inputs)] if args.graph else None
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K_)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(K_):
            flush.zero_()
            ev[i][0].record()
            if graphs:
                graphs[i % n_inputs].replay()
            else:
                step(i)
            ev[i][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_step = sum(e[0].elapsed_time(e[1]) for e in ev) / K_  # ms
    eve = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K_)]
    for i in range(K_):
        flush.zero_()
        eve[i][0].record()
        step(i)
        eve[i][1].record()
    torch.cuda.synchronize()
    t_eager = sum(e[0].elapsed_time(e[1]) for e in eve) / K_
    # per-phase attribution (separate pass: the middle event breaks the PDL overlap)
    evp = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K_)]
    for i in range(K_):
        flush.zero_()
        q = Qt[i % n_inputs]
        evp[i][0].record()
        sqz.centroid_lookup(idx, q, scale, T, T1, sel=sel, comm=comm, T0=T0)
        evp[i][1].record()
        attend(q)
        evp[i][2].record()
    torch.cuda.synchronize()
    t_look = sum(e[0].elapsed_time(e[1]) for e in evp) / K_
    t_attn = sum(e[1].elapsed_time(e[2]) for e in evp) / K_
    # ---- end to end through the public API with host buffers ----
    # One pinned host staging buffer per input holds everything the step brings
    # in (the query rows, and the new token's K/V row entering the user cache for
    # decode, the whole user input for prefill), copied in ONE host->device
    # transfer and scattered on the device; O and LSE live in one device buffer
    # read back in ONE device->host transfer (each PCIe copy pays ~2-4 us of
    # latency, so five small copies cost more than the bytes).
    pin = dict(pin_memory=True)
    q_b = Qt[0].numel() * esz
    kv_new = None
    if Ku is not None:
        kv_new = (slice(None), slice(None), slice(n_u - 1, n_u)) if cfg["mode"] == "decode" else \
            (slice(None), slice(None), slice(None))
    kv_b = 0 if kv_new is None else Ku[kv_new].numel() * esz
    h2d = q_b + 2 * kv_b
    hin = torch.empty(n_inputs, h2d, dtype=torch.uint8, **pin)
    for i in range(n_inputs):
        hin[i, :q_b].copy_(Qt[i].contiguous().view(torch.uint8).view(-1).cpu())
        if kv_new is not None:
            hin[i, q_b:q_b + kv_b].copy_(Ku[kv_new].contiguous().view(torch.uint8).view(-1).cpu())
            hin[i, q_b + kv_b:].copy_(Vu[kv_new].contiguous().view(torch.uint8).view(-1).cpu())
    din = torch.empty(h2d, dtype=torch.uint8, device=dev)
    dQ = din[:q_b].view(Qt.dtype).view(Qt[0].shape)
    o_b = O.numel() * O.element_size()
    out_b = o_b + LSE.numel() * 4
    dout = torch.empty(out_b, dtype=torch.uint8, device=dev)
    O_e = dout[:o_b].view(O.dtype).view(O.shape)
    LSE_e = dout[o_b:].view(torch.float32).view(LSE.shape)
    hout = torch.empty(out_b, dtype=torch.uint8, **pin)
    d2h = out_b

    kv_dst = None if kv_new is None else KVu[(slice(None),) + kv_new]  # [2, B, H, rows, d]

    def e2e_step(i):
        din.copy_(hin[i % n_inputs], non_blocking=True)
        if kv_new is not None:  # the staged K rows then V rows, as [2, B, H, rows, d]
            kv_dst.copy_(din[q_b:].view(KVu.dtype).view(kv_dst.shape))
        step_into(dQ, O_e, LSE_e)
        hout.copy_(dout, non_blocking=True)

    e2e_graphs = ([capture_graph(lambda i=i: e2e_step(i)) for i in range(n_inputs)]
                  if args.graph else None)
    ev2 = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K_)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(K_):
        flush.zero_()
        ev2[i][0].record()
        if e2e_graphs:
            e2e_graphs[i % n_inputs].replay()
        else:
            e2e_step(i)
        ev2[i][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_e2e = sum(e[0].elapsed_time(e[1]) for e in ev2) / K_
    # ---- sampled oracle parity of this run's output (after the timed region) ----
    parity = None
    if not args.no_parity:
        q = Qt[0]
        sel_p = sqz.Selection.empty(idx, B, n_q, debug=True, device=dev, key_idx=False)
        sqz.centroid_lookup(idx, q, scale, T, T1, sel=sel_p, comm=comm, T0=T0)
        same_sel = None
        if use_step:
            # the timed path's outputs: O / LSE from sqz_decode_step; its selection must
            # equal the debug lookup's (same arithmetic), whose scores give the band rule
            sel_s = sqz.Selection.empty(idx, B, n_q, False, dev, key_idx=True)
            sqz.decode_step(idx, q, Kp, Vp, Ku, Vu, scale, T, T1, sel=sel_s, O=O, LSE=LSE, ws=step_ws,
                            T0=T0)
            torch.cuda.synchronize()
            nc = sel_s.n_clusters
            same_sel = bool(torch.equal(nc, sel_p.n_clusters) and torch.equal(sel_s.n_keys, sel_p.n_keys)
                            and all(torch.equal(sel_s.clusters[b_, h_, :int(nc[b_, h_])],
                                                sel_p.clusters[b_, h_, :int(nc[b_, h_])])
                                    for b_ in range(B) for h_ in range(Hl)))
            del sel_s
        else:
            attend_into(q, O, LSE, sel_p)
        torch.cuda.synchronize()
        if rank == 0:
            rs = None
            if cfg["mode"] == "prefill":
                rs = np.unique(np.concatenate([[0, n_q - 1], np.linspace(0, n_q - 1, 62)])).astype(np.int32)
            t_p = time.time()
            parity = oracle_parity(sqz, gidx, q, sel_p, O, LSE, T, T1, scale, K0, V0, Ku0, Vu0, idx,
                                   causal, rs, T0=T0)
            parity["oracle_s"] = round(time.time() - t_p, 1)
            parity["path"] = "sqz_decode_step" if use_step else "two calls"
            if same_sel is not None:
                parity["step_selection_equals_lookup"] = same_sel
                parity["ok"] = bool(parity.get("ok")) and same_sel
        del sel_p
    # ---- selection quality (App. A skewness, App. D ideal lookup; after the timed region) ----
    quality = None
    if cfg["mode"] == "decode" and comm is None and rank == 0 and not args.no_parity:
        quality = selection_quality(sqz, idx, Qt, Kp, scale, T, T1, min(n_inputs, 8), B, dev, T0=T0)
    # ---- max over ranks ----
    if world > 1:
        tt = torch.tensor([t_step, t_look, t_attn, t_e2e, t_eager], device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_look, t_attn, t_e2e, t_eager = tt.tolist()
    hbm, bf16, peak_kind = load_peaks()
    # replicas: every rank runs its own step (weak); heads / clusters: the ranks
    # share one step of B sequences (strong)
    tokens = B * n_q * (world if shard in ("none", "replicas") else 1)
    if cfg["mode"] == "decode":
        value = t_step * 1e3 / tokens
        e2e_v = t_e2e * 1e3 / tokens
        step_bytes = bytes_lookup + bytes_attn
        if True:  # the attention kernel of the two-call pass (the same k_attend the step runs)
            ach = bytes_attn / (t_attn * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4),
                    "traffic": traffic_for(args.config, "sparse_attention_shared" if shared_attn
                                           else "sparse_attention"),
                    "kernel": ("k_attend_shared (batch-shared union pass, mma.sync tiles, fused merge); "
                               "bytes = union of the B selections per head" if shared_attn else
                               "sqz_sparse_attention call: k_attend (persistent split-KV over equal key "
                               "ranges) + the row merge (fused ticket, or for short streams k_merge_rows "
                               "behind it, inside the timed call)"),
                    "bytes_if_streamed_per_query": int(bytes_attn_perq),
                    "peak_kind": f"{peak_kind} copy bandwidth",
                    "bytes_per_launch": int(bytes_attn)}
        whole = {"bytes_per_step": int(step_bytes),
                 "achieved_GBps": round(step_bytes / (t_step * 1e-3) / 1e9, 1),
                 "frac_hbm": round(step_bytes / (t_step * 1e-3) / 1e9 / hbm, 4)}
    else:
        value = tokens / (t_step * 1e-3)
        e2e_v = tokens / (t_e2e * 1e-3)
        ach = flops_attn / (t_attn * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": bf16, "unit": "TFLOP/s",
                "frac": round(ach / bf16, 4),
                "traffic": traffic_for(args.config, "sparse_attention"),
                "kernel": "sparse_attention", "peak_kind": f"{peak_kind} bf16 burst",
                "flops_per_launch": int(flops_attn)}
        step_flops = flops_attn + flops_lookup
        whole = {"flops_per_step": int(step_flops),
                 "achieved_TFLOPs": round(step_flops / (t_step * 1e-3) / 1e12, 2)}
    # libsqz kernels per step (NCCL's own kernels not counted)
    levels = idx.levels
    per_select = 1 if cfg["mode"] == "decode" else (2 if dt == 1 and d in (64, 128) else 3)
    if comm is None:
        n_look = levels * per_select
    else:  # stats, then per level: fold + select (+ next level's stats)
        n_look = 1 + levels * (1 + per_select) + (levels - 1)
    # + k_union (batch-shared) or k_merge_rows (per-row persistent decode)
    merge_k = (cfg["mode"] == "decode" and not shared_attn
               and (1 << 17) <= B * Hl * L < (1 << 24))  # attention.cu launch_t
    launches = K_ * (n_look + 1 + (1 if comm else 0) + (1 if shared_attn or merge_k else 0))
    metric, unit, hib = metric_of(cfg)
    line = {
        "metric": metric, "value": round(value, 3), "unit": unit, "n_gpus": world,
        "steps": K_, "warmup": args.warmup, "ms_per_step": round(t_step, 5),
        "higher_is_better": hib, "scaling": "weak" if shard in ("none", "replicas") else "strong",
        "vs_baseline": None,
        "dtype": "bf16" if dt == 1 else "f32", "data": "synthetic (SYN-MIX v1 clustered keys)",
        "config": {"workload": cfg["workload"],
                   "global_batch": B * (world if shard in ("none", "replicas") else 1), "seq_len": L,
                   "n_q": n_q, "n_u": n_u,
                   "parallelism": {"none": "1 GPU", "replicas": f"replicas x{world}",
                                   "heads": f"heads sharded x{world}",
                                   "clusters": f"fixed context sharded by cluster x{world}"}[shard],
                   "l2": {"write": "flushed (512 MB write) between timed steps",
                          "write+read": "flushed between timed steps: 512 MB write, then a 512 MB "
                                        "read of another buffer (untimed), so the step starts from "
                                        "a cold L2 of clean lines"}[args.flush],
                   "T": T, "T1": T1, "T0": T0, "levels": idx.levels,
                   "mean_selected_keys_per_step": k_glob,
                   "mean_union_keys_per_step": allsum(ku_mean),
                   "attention_path": "batch-shared union pass" if shared_attn else "per-(b,h) streams",
                   "retention_realized": k_glob / (B * H * L), "kmeans_iters": list(iters),
                   "kmeans_mode": args.kmeans_mode,
                   "index_build_s": round(t_index, 2)},
        "phases_ms": {"lookup": round(t_look, 5), "sparse_attention": round(t_attn, 5),
                      "phases_of": "the two-call path (sqz_centroid_lookup, sqz_sparse_attention), "
                                   "separate events",
                      "eager_step": round(t_eager, 5), "graph_replay": bool(args.graph),
                      "decode_path": ("sqz_decode_step" if use_step else "two calls")
                      if cfg["mode"] == "decode" else "two calls"},
        "whole_step": whole,
        "roofline": roof,
        "e2e": {"value": round(e2e_v, 3), "unit": unit, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if parity is not None:
        line["parity"] = parity
    if quality is not None:
        line["selection_quality"] = quality
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="one workload; default: cfg2 decode (the headline line) with the cfg3 "
                         "prefill measured in the same run as its `prefill` object")
    ap.add_argument("--no-prefill", action="store_true",
                    help="default run: skip the cfg3 prefill object")
    ap.add_argument("--no-extra", action="store_true",
                    help="default run: skip the cfg4 object (extra_configs)")
    ap.add_argument("--decode-path", default="auto", choices=["auto", "step", "calls"],
                    help="decode: one sqz_decode_step call (flag hand-off from the lookup to the "
                         "attention kernel, user KV attended by the lookup; B = 1 single level) or "
                         "the two calls (lookup, then sparse attention, chained by programmatic "
                         "dependent launch); auto = the step where it applies")
    ap.add_argument("--flush", default="write", choices=["write", "write+read"],
                    help="L2 flush between timed steps (see run_gpu)")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the rank-0 sampled oracle parity check after the timed region")
    ap.add_argument("--kmeans-iters", type=int, default=30)
    ap.add_argument("--kmeans-mode", default="auto", choices=["auto", "exact", "tensor"],
                    help="K-means assignment step: fp32 FFMA (exact), tcgen05 split-bf16 (tensor), "
                         "or tensor for large problems (auto)")
    ap.add_argument("--kmeans-iters-set", type=int, default=None,
                    help="override the per-config Lloyd iteration count (cfg5: 3)")
    ap.add_argument("--retention", type=float, default=None,
                    help="override the config's retention target (1.0 = T = 0, dense)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sel-runs", default="auto", choices=["auto", "on", "off"],
                    help="keep the selection in run-length form (no key_idx expansion in the lookup; "
                         "the attention reads the runs); auto = on for single-level prefill")
    ap.add_argument("--attn-per-row", action="store_true",
                    help="decode with B >= 2: stream each (b,h) selection separately instead of "
                         "the batch-shared union pass (A/B of NEXT-1)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time eager per-call launches instead of CUDA-graph replay")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    with_prefill = args.config is None and not args.no_prefill
    if args.config is None:
        args.config = "cfg2"
    cfg = dict(CONFIGS[args.config])
    if args.retention is not None:
        cfg["retention"] = args.retention
        cfg["workload"] += f" [retention override {args.retention}]"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # dry run of the N-rank code path on ONE GPU (all ranks on device 0, gloo process
    # group): checks the sharding, calibration and max-over-ranks logic before a real
    # multi-GPU run; the numbers of such a run are not measurements
    shared_gpu = os.environ.get("SQZ_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local_rank = 0
    metric, unit, hib = metric_of(cfg)

    if args.impl == "reference":
        if rank != 0:
            return
        value, sample, cores, times = cpu_oracle_run(cfg, steps=args.steps, warmup=args.warmup)
        line = {"impl": "reference", "metric": metric, "value": round(value, 3), "unit": unit,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(float(np.mean(times)) * 1e3, 4), "higher_is_better": hib,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (SYN-MIX v1 clustered keys)",
                "config": {"workload": cfg["workload"], "global_batch": cfg["B"],
                           "seq_len": cfg["L"], "parallelism": "host cores (oracle)"},
                "cpu_baseline": {"value": round(value, 3), "unit": unit, "cores": cores,
                                 "kind": "oracle", "sample": sample},
                "e2e": {"value": round(value, 3), "unit": unit, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_gpu(args, cfg, rank, world, local_rank)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        value, sample, cores, _ = cpu_oracle_run(cfg)
        line["cpu_baseline"] = {"value": round(value, 3), "unit": unit, "cores": cores,
                                "kind": "oracle", "sample": sample}
    if with_prefill:
        # the prefill half of BASELINE's metric (cfg3), same run, same rules
        import torch

        torch.cuda.empty_cache()
        pcfg = dict(CONFIGS["cfg3"])
        if args.retention is not None:
            pcfg["retention"] = args.retention
        pargs = argparse.Namespace(**vars(args))
        pargs.config = "cfg3"
        pl = run_gpu(pargs, pcfg, rank, world, local_rank)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            pv, psample, pcores, _ = cpu_oracle_run(pcfg, seconds=8.0)
            pl["cpu_baseline"] = {"value": round(pv, 3), "unit": pl["unit"], "cores": pcores,
                                  "kind": "oracle", "sample": psample}
        keep = ("metric", "value", "unit", "ms_per_step", "higher_is_better", "dtype", "config",
                "phases_ms", "whole_step", "roofline", "e2e", "gpu_launches", "clocks", "parity",
                "cpu_baseline", "scaling")
        line["prefill"] = {k: pl[k] for k in keep if k in pl}
    if with_prefill and not args.no_extra:
        # the 128K hierarchical batch-8 decode (cfg4: batch-shared attention, tensor-core
        # K-means) in the same run, so the driver's line carries it too
        import torch

        torch.cuda.empty_cache()
        xargs = argparse.Namespace(**vars(args))
        xargs.config = "cfg4"
        xargs.steps = min(args.steps, 30)
        xl = run_gpu(xargs, dict(CONFIGS["cfg4"]), rank, world, local_rank)
        keep = ("metric", "value", "unit", "ms_per_step", "higher_is_better", "dtype", "config",
                "phases_ms", "whole_step", "roofline", "e2e", "gpu_launches", "clocks", "parity",
                "selection_quality", "scaling", "steps")
        line["extra_configs"] = {"cfg4": {k: xl[k] for k in keep if k in xl}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
