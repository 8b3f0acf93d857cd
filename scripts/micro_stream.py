"""Streaming reference points on this GPU (not part of the product): torch elementwise kernels with
the update kernel's byte pattern (2 reads + 1 write of 52 MB vectors) and a plain copy."""
import torch
N = 6489990
d = torch.randn(N, dtype=torch.float64, device="cuda")
h = torch.randn(N, dtype=torch.float64, device="cuda")
x = torch.randn(N, dtype=torch.float64, device="cuda")
big = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")


def t(fn, nbytes, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(reps):
        big.zero_()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / reps
    return ms * 1e3, nbytes / (ms * 1e-3) / 1e9


print("copy      %.1f us %.0f GB/s" % t(lambda: x.copy_(h), 16 * N))
print("d += a*h  %.1f us %.0f GB/s" % t(lambda: d.add_(h, alpha=1e-3), 24 * N))
print("d += h+x  %.1f us %.0f GB/s" % t(lambda: d.add_(h).add_(x), 48 * N))
hh = torch.randn(3 * N, dtype=torch.float64, device="cuda")
dd = torch.randn(3 * N, dtype=torch.float64, device="cuda")
print("3N d+=a*h %.1f us %.0f GB/s" % t(lambda: dd.add_(hh, alpha=1e-3), 24 * 3 * N))
