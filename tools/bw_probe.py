"""HBM probe: achieved GB/s of torch's copy (1R+1W) and add (2R+1W) at 2^28 fp32,
the ceilings a 1-read and a 2-read streaming kernel can expect."""
import torch


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


n = 1 << 28
x = torch.rand(n, device="cuda")
y = torch.rand(n, device="cuda")
z = torch.empty(n, device="cuda")
ms = timeit(lambda: z.copy_(x))
print(f"copy 1R1W: {ms:.4f} ms {8 * n / ms / 1e6:.1f} GB/s")
ms = timeit(lambda: torch.add(x, y, out=z))
print(f"add  2R1W: {ms:.4f} ms {12 * n / ms / 1e6:.1f} GB/s")
ms = timeit(lambda: torch.mul(x, 2.0, out=z))
print(f"mul  1R1W: {ms:.4f} ms {8 * n / ms / 1e6:.1f} GB/s")
ms = timeit(lambda: torch.addcmul(x, y, x, out=z))
print(f"addcmul 2R1W: {ms:.4f} ms {12 * n / ms / 1e6:.1f} GB/s")
