"""Dense comparators on the same box: torch SDPA (flash) over the
full fixed context + user KV for the cfg2 decode and cfg3 prefill shapes.  The
sparse path's own T = 0 runs come from bench.py --retention 1.0."""
import json

import torch
import torch.nn.functional as F

torch.manual_seed(0)
dev = "cuda"
res = {}
for name, n_q, n_u in (("cfg2_decode", 1, 1024), ("cfg3_prefill", 1024, 1024)):
    H, L, d = 32, 32768, 128
    q = torch.randn(1, H, n_q, d, device=dev, dtype=torch.bfloat16)
    k = torch.randn(1, H, L + n_u, d, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(5):
        F.scaled_dot_product_attention(q, k, v)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        F.scaled_dot_product_attention(q, k, v)  # non-causal over L + n_u: an upper bound
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    res[name] = {"torch_sdpa_us": round(ts[len(ts) // 2] * 1e3, 2),
                 "note": "F.scaled_dot_product_attention bf16, dense over L + n_u keys, non-causal, L2 flushed"}
print(json.dumps(res))
