"""Device-to-host copy bandwidth into pinned memory (the e2e legs' bound):
contiguous, and pitched 2D copies of chain-part column blocks."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_17405_b200 import _lib  # noqa: E402

n, m, d = 1000, 65536, 10
src = torch.randn(n, m, d, dtype=torch.float64, device="cuda")
dst = torch.empty(n, m, d, dtype=torch.float64, pin_memory=True)
nbytes = src.numel() * 8
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"contiguous D2H {nbytes / 1e9:.2f} GB: {1e3 * dt:.1f} ms, {nbytes / dt / 1e9:.1f} GB/s", flush=True)
lib = _lib.lib()
for parts in (4, 12):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pitch = m * d * 8
        for h in range(parts):
            lo, hi = m * h // parts, m * (h + 1) // parts
            _lib.check(lib.fsmc_copy_to_host_2d(dst.data_ptr() + lo * d * 8, src.data_ptr() + lo * d * 8,
                                                pitch, (hi - lo) * d * 8, n, _lib.stream_ptr()), "copy")
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{parts} pitched column blocks: {1e3 * dt:.1f} ms, {nbytes / dt / 1e9:.1f} GB/s", flush=True)
# the same copy split over several streams (copy engines)
for ns in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            lo, hi = n * i // ns, n * (i + 1) // ns
            with torch.cuda.stream(s):
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{ns} streams: {1e3 * dt:.1f} ms, {nbytes / dt / 1e9:.1f} GB/s", flush=True)
