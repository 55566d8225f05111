"""cuBLAS TF32 (and bf16) throughput on this box: the practical peaks for the TF32 roofline."""
import torch

torch.backends.cuda.matmul.allow_tf32 = True
for dt, name in ((torch.float32, "tf32"), (torch.bfloat16, "bf16")):
    a = torch.randn(8192, 8192, device="cuda").to(dt)
    b = torch.randn(8192, 8192, device="cuda").to(dt)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        s.record()
        a @ b
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"cuBLAS {name} 8192^3: {2 * 8192 ** 3 / best / 1e9:.1f} TFLOP/s (best of 10)")
