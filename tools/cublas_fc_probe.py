"""cuBLAS FP32 (no TF32) on the ResNet-50 FC shape 16x2048 @ 2048x1000 under
CUDA-graph replay with rotating inputs (context for skinny_cluster)."""
import torch

torch.backends.cuda.matmul.allow_tf32 = False
R = 48
As = [torch.randn(16, 2048, device="cuda") for _ in range(R)]
Bs = [torch.randn(2048, 1000, device="cuda") for _ in range(R)]
Cs = [torch.empty(16, 1000, device="cuda") for _ in range(R)]
for i in range(R):
    torch.matmul(As[i], Bs[i], out=Cs[i])
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
steps = 200
with torch.cuda.graph(g, stream=s):
    for i in range(steps):
        torch.matmul(As[i % R], Bs[i % R], out=Cs[i % R])
g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
g.replay()
b.record()
b.synchronize()
us = a.elapsed_time(b) * 1e3 / steps
print(f"cuBLAS FP32 16x2048x1000: {us:.2f} us/launch, {8204288 / us / 1e3:.0f} GB/s")
