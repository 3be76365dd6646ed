import numpy as np
import torch

from paper_2411_09688_b200 import synth


def test_deterministic_and_shapes():
    a = synth.fixed_context(2, 100, 8, 5, seed=1)
    b = synth.fixed_context(2, 100, 8, 5, seed=1)
    assert np.array_equal(a.K, b.K) and np.array_equal(a.V, b.V)
    assert a.K.shape == (2, 100, 8) and a.K.dtype == np.uint16
    q = synth.decode_queries(a.mix, 3, seed=2)
    assert q.shape == (3, 2, 1, 8)
    p = synth.prefill_queries(a.mix, 1, 17, seed=3)
    assert p.shape == (1, 2, 17, 8)
    ku, vu = synth.user_kv(a.mix, 2, 5)
    assert ku.shape == (2, 2, 5, 8)
    init = synth.kmeans_init(2, 100, 10)
    assert all(len(set(r.tolist())) == 10 for r in init)


def test_bf16_rounding_matches_torch():
    x = np.random.default_rng(0).standard_normal(100000).astype(np.float32) * 7
    ours = synth.storage_to_f32(synth.to_storage(x, synth.BF16))
    t = torch.tensor(x).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(ours, t)
