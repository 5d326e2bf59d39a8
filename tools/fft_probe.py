"""Time the summed-periodogram autocovariance variants on bench-shaped samples."""
import sys
import time

import torch

n, m, d = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (900, 16384, 100)
S = torch.randn(n, m, d, dtype=torch.float64, device="cuda")
mean = S.mean(dim=0)
size = 1 << (2 * n - 1).bit_length()


def v_dim0(chunk_elems):
    power = torch.zeros((size // 2 + 1, d), dtype=torch.float64, device="cuda")
    chunk = max(1, chunk_elems // (size * d))
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        f = torch.fft.rfft(S[:, lo:hi, :] - mean[lo:hi], n=size, dim=0)
        power += torch.view_as_real(f).square().sum(dim=(1, 3))
    return torch.fft.irfft(power, n=size, dim=0)[:n] / n


def v_last(chunk_elems):
    power = torch.zeros((d, size // 2 + 1), dtype=torch.float64, device="cuda")
    chunk = max(1, chunk_elems // (size * d))
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        c = (S[:, lo:hi, :] - mean[lo:hi]).permute(1, 2, 0)      # [chains, d, n] view
        f = torch.fft.rfft(c, n=size, dim=2)                      # copies to contiguous
        power += (f.real.square() + f.imag.square()).sum(dim=0)
    return (torch.fft.irfft(power, n=size, dim=1)[:, :n] / n).T


for name, fn in [("dim0", v_dim0), ("last", v_last)]:
    for ce in (1 << 26, 1 << 27, 1 << 28):
        fn(ce)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(ce)
        torch.cuda.synchronize()
        print(f"{name} chunk 2^{ce.bit_length() - 1}: {1e3 * (time.perf_counter() - t0):.1f} ms")
a, b = v_dim0(1 << 27), v_last(1 << 27)
print("max rel diff", float(((a - b).abs() / b.abs().clamp_min(1e-300)).max()))
