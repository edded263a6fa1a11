"""Per-launch floors under CUDA-graph replay (dev aid): an empty kernel, an
8 MB copy, a 64 MB copy -- rotating over copies larger than L2 in total."""
import torch

def graph_time(fn, steps=200):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    fn(0)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(steps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / steps

t = torch.zeros(1, device="cuda")
print("empty kernel   %.2f us" % graph_time(lambda i: t.add_(1)))
for mb in (8, 64):
    n = mb * 2**20 // 4 // 2
    R = max(2, 3 * 126 // mb + 1)
    xs = [torch.rand(n, device="cuda") for _ in range(R)]
    ys = [torch.empty(n, device="cuda") for _ in range(R)]
    us = graph_time(lambda i: ys[i % R].copy_(xs[i % R]))
    print("copy %3d MB     %.2f us  %.0f GB/s" % (mb, us, mb * 2**20 / us / 1e3))

# write-only floor at CCSD(T)'s output size (729 MiB, larger than L2)
y = torch.empty(24 ** 6, device="cuda")
us = graph_time(lambda i: y.fill_(float(i)), steps=50)
print("fill 729 MiB   %.2f us  %.0f GB/s" % (us, y.numel() * 4 / us / 1e3))
x = torch.rand(24 ** 6 // 2, device="cuda")
y2 = torch.empty(24 ** 6 // 2, device="cuda")
us = graph_time(lambda i: y2.copy_(x), steps=50)
print("copy 2x365 MiB %.2f us  %.0f GB/s" % (us, 2 * x.numel() * 4 / us / 1e3))
