"""Device copy bandwidth of this box (1 GiB bf16 copy, as MEASURED_PEAKS does) next to the stencil."""
import torch
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda").uniform_()
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
print(f"copy 2 GiB read+write: {2 * a.numel() * 2 / best / 1e9:.1f} GB/s")
