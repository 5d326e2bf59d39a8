"""Variants of analysis.acov_all (the all-lags autocovariance by FFT) on a
C3-sized sample array: time each with CUDA events and compare to the current
path.  Usage: python tools/acov_probe.py [n m d]"""
import math
import sys

import torch

n_all, m, d = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1000, 16384, 100)
burn = n_all // 10
n = n_all - burn
g = torch.Generator(device="cuda").manual_seed(0)
S = torch.randn((n_all, m, d), dtype=torch.float64, device="cuda", generator=g)
mean = S[burn:].mean(dim=0)


def current(size, chunk_elems=1 << 27, power_mode="sq"):
    power = torch.zeros((d, size // 2 + 1), dtype=torch.float64, device="cuda")
    chunk = max(1, chunk_elems // (size * d))
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        c = (S[burn:, lo:hi, :] - mean[lo:hi]).permute(1, 2, 0)
        f = torch.fft.rfft(c, n=size, dim=2)
        if power_mode == "sq":
            power += (f.real.square() + f.imag.square()).sum(dim=0)
        else:
            r = torch.view_as_real(f)
            power += (r * r).sum(dim=(0, 3))
    return (torch.fft.irfft(power, n=size, dim=1)[:, :n] / n)


def timed(fn, *a, **k):
    fn(*a, **k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn(*a, **k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


p2 = 1 << int(math.ceil(math.log2(2 * n)))
t0, ref = timed(current, p2)
print(f"current size={p2}: {t0:.1f} ms")
for label, kw in [("size=2n (mixed radix)", dict(size=2 * n)),
                  ("chunk 2^28", dict(size=p2, chunk_elems=1 << 28)),
                  ("chunk 2^26", dict(size=p2, chunk_elems=1 << 26)),
                  ("view_as_real power", dict(size=p2, power_mode="var")),
                  ("2n + chunk 2^28", dict(size=2 * n, chunk_elems=1 << 28))]:
    t, out = timed(current, **kw)
    err = float(((out - ref).abs() / ref.abs().clamp_min(1e-300).max()).max())
    print(f"{label}: {t:.1f} ms  max err rel to max {err:.2e}")
