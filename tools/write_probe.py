"""Write-only HBM bandwidth (development aid): fill_ and cudaMemset of a
764 MB buffer (CCSD(T)'s output size), CUDA-event timed after warm-up."""
import torch

n = 764411904 // 4
x = torch.empty(n, dtype=torch.float32, device="cuda")
row = torch.rand(576, device="cuda")
for name, fn in (("fill_", lambda: x.fill_(1.0)), ("zero_", lambda: x.zero_()),
                 ("copy_ of a broadcast random 576-float row", lambda: x.view(-1, 576).copy_(row.expand(n // 576, 576)))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"{name}: {ms:.4f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
