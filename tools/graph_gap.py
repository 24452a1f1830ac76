"""How long does one dependent kernel boundary cost inside a replayed CUDA
graph?  A chain of K tiny dependent kernels (torch in-place adds on a 4-element
tensor) captured once, replayed, timed with events: per-kernel time ~ the
launch-to-launch latency the Stage-1 iteration graph pays ~35 times."""
import torch

x = torch.zeros(4, device="cuda")
s = torch.cuda.Stream()
for K in (1, 10, 40, 80):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for _ in range(3):
            x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(K):
                x.add_(1)
    torch.cuda.synchronize()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 200 * 1000
    print(f"K={K}: {t:.2f} us per graph, {t / K:.2f} us per kernel")
