"""GPU parity of sqz_selection_diagnostics (App. A skewness, App. D ideal lookup;
NEXT-4) against the fp64 oracle on the same seeded inputs and the GPU's own
selection.  Masses: |delta| <= 2e-5 (fp32 logits and exp vs fp64); counts and
the matched-budget recall: exact except for keys whose fp64 score lies within
1e-5 relative of the decision boundary (the same band rule as the lookup)."""
import zlib

import numpy as np
import pytest

import oracle
from paper_2411_09688_b200 import calib, synth

from helpers import gpu_index, key_mask_from_gpu, oracle_problem

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_09688_b200 import sqz

    sqz.device_check()


CASES = [
    # name, H, L, d, c2, c1, dtype, B, retention, top_frac, T_ideal
    ("bf16_d128", 4, 3000, 128, 97, 0, synth.BF16, 3, 0.3, 0.01, 1e-3),
    ("fp32_d64", 2, 2000, 64, 50, 0, synth.F32, 2, 0.2, 0.05, 1e-4),
    ("hier_bf16", 3, 4000, 128, 200, 40, synth.BF16, 2, 0.1, 0.01, 5e-4),
    ("bf16_T0_full", 2, 1500, 128, 40, 0, synth.BF16, 1, 1.0, 1.0, 0.0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_diagnostics_match_oracle(case):
    from paper_2411_09688_b200 import sqz

    name, H, L, d, c2, c1, dt, B, ret, frac, T_id = case
    P = oracle_problem(H, L, d, c2, c1, dt, seed=zlib.crc32(name.encode()) % 1000, B=B)
    idx = P["idx"]
    scale = 1.0 / np.sqrt(d)
    # thresholds from separate calibration queries (R17)
    Qc = oracle.to_f64(synth.decode_queries(P["fc"].mix, 24, seed=777, dtype=dt))
    T1 = 0.0
    if c1:
        T1 = calib.weighted_threshold(oracle.lookup(Qc, idx, scale, 0.0, 0.0)["Sbar1"], idx.N1[None], 0.5)
    T = 0.0 if ret >= 1.0 else calib.weighted_threshold(
        oracle.lookup(Qc, idx, scale, 0.0, T1)["Sbar2"], idx.N2[None], ret)
    gidx = gpu_index(idx)
    Q = sqz.to_device(P["Q"])
    Kp = sqz.to_device(oracle.permute_kv(P["fc"].K, idx))
    sel = sqz.centroid_lookup(gidx, Q, scale, T, T1)
    out = sqz.selection_diagnostics(gidx, Q, Kp, sel, scale, frac, T_id)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy().astype(np.float64) for k, v in out.items()}
    mask = key_mask_from_gpu(sel, idx, B, H)
    K64 = oracle.to_f64(P["fc"].K)
    Q64 = oracle.to_f64(P["Q"])
    ref = oracle.diagnostics(Q64, K64, mask, scale, frac, T_id)
    k = sel.n_keys.cpu().numpy()
    assert (ref["k"] == k).all()
    for key in ("skew", "mass_sel", "mass_ideal", "mass_T"):
        err = np.abs(g[key] - ref[key]).max()
        assert err <= 2e-5, (key, err)
    assert (g["skew"] <= 1 + 1e-5).all() and (g["mass_ideal"] >= g["mass_sel"] - 2e-5).all()
    for b in range(B):
        for h in range(H):
            z = K64[h] @ Q64[b, h, 0] * scale
            a = np.exp(z - z.max())
            a /= a.sum()
            srt = np.sort(a)[::-1]
            # ideal lookup at threshold: count exact outside the band around T
            if T_id > 0:
                amb = int((np.abs(a - T_id) <= 1e-5 * T_id).sum())
                assert abs(g["n_T"][b, h] - ref["n_T"][b, h]) <= amb
            else:
                assert g["n_T"][b, h] == L
            kk = int(k[b, h])
            if kk == 0:
                assert g["recall"][b, h] == 1.0
                continue
            amb = int((np.abs(a - srt[kk - 1]) <= 1e-5 * srt[kk - 1]).sum())
            assert abs(g["recall"][b, h] - ref["recall"][b, h]) <= (amb + 1e-6) / kk + 1e-6, \
                (b, h, g["recall"][b, h], ref["recall"][b, h], amb)
    if ret >= 1.0:
        assert np.abs(g["recall"] - 1).max() <= 1e-6 and np.abs(g["mass_sel"] - 1).max() <= 2e-5


def test_diagnostics_three_level_index():
    """The diagnostics read the finest-level selection of any hierarchy: a three-level
    index gives the oracle's masses and recall on the GPU's selection."""
    from paper_2411_09688_b200 import sqz

    H, L, d, c2, c1, c0, B = 2, 5000, 128, 200, 40, 6, 2
    fc = synth.fixed_context(H, L, d, c2, dtype=synth.BF16, seed=621, G1=c1)
    g, Kp, Vp, _ = sqz.cluster_keys(sqz.to_device(fc.K), sqz.to_device(fc.V), c2,
                                    torch.from_numpy(synth.kmeans_init(H, L, c2, seed=622)).cuda(), c1,
                                    torch.from_numpy(synth.kmeans_init(H, c2, c1, seed=623)).cuda(),
                                    max_iters=15, c0=c0,
                                    init0=torch.from_numpy(synth.kmeans_init(H, c1, c0, seed=624)).cuda())
    Q = synth.decode_queries(fc.mix, B, seed=625)
    Qd = sqz.to_device(Q)
    scale = 1.0 / np.sqrt(d)
    sel = sqz.centroid_lookup(g, Qd, scale, 2e-5, 1e-4, T0=1e-4)
    out = sqz.selection_diagnostics(g, Qd, Kp, sel, scale, 0.01, 1e-3)
    torch.cuda.synchronize()
    perm, ko = g.perm.cpu().numpy(), g.key_off.cpu().numpy()
    mask = np.zeros((B, H, L), bool)
    cl, n = sel.clusters.cpu().numpy(), sel.n_clusters.cpu().numpy()
    for b in range(B):
        for h in range(H):
            for i in cl[b, h, :n[b, h]]:
                mask[b, h, perm[h][ko[h, i]:ko[h, i + 1]]] = True
    ref = oracle.diagnostics(oracle.to_f64(Q), oracle.to_f64(fc.K), mask, scale, 0.01, 1e-3)
    for key in ("skew", "mass_sel", "mass_ideal", "mass_T"):
        assert np.abs(out[key].cpu().numpy() - ref[key]).max() <= 2e-5, key
