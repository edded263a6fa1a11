"""cuBLAS reference points on this box (context for the FFMA / TF32 rooflines)."""
import torch

n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for tf32 in (False, True):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        c = a @ b
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"cuBLAS {'TF32' if tf32 else 'FP32'} 8192^3: {ms:.3f} ms  {2 * n**3 / ms / 1e9:.1f} TFLOP/s")
