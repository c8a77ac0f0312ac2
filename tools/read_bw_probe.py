"""Experiment: read-only vs copy HBM bandwidth on this box (torch kernels, CUDA events)."""
import torch

x = torch.empty(2 ** 30, dtype=torch.float32, device="cuda").normal_()  # 4 GiB
y = torch.empty_like(x)
s = torch.empty((), device="cuda")


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


nb = x.numel() * 4
print("copy GB/s (r+w)", round(2 * nb / t(lambda: y.copy_(x)) / 1e6, 1))
print("sum  GB/s (read)", round(nb / t(lambda: torch.sum(x)) / 1e6, 1))
print("amax GB/s (read)", round(nb / t(lambda: torch.amax(x)) / 1e6, 1))
