"""Floor of the bench's timing method: CUDA-event pairs around an (almost) empty
step, eager vs CUDA-graph replay, after the 512 MB write flush."""
import torch

x = torch.zeros(16, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn, n=30, fl=True):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        if fl:
            flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)[2:-2]
    return sum(v) / len(v)


def graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


one = lambda: x.add_(1)
two = lambda: (x.add_(1), x.add_(1))
g1, g2 = graph(one), graph(two)
for fl in (True, False):
    print(f"flush={fl}: nothing {t(lambda: None, fl=fl):.2f} us | eager 1 kernel {t(one, fl=fl):.2f} | "
          f"eager 2 {t(two, fl=fl):.2f} | graph 1 {t(g1.replay, fl=fl):.2f} | graph 2 {t(g2.replay, fl=fl):.2f}")
