"""Counter-based splittable random streams (drop-in for ``fsm_mcmc.prng``).

Keys are host metadata (an immutable ``(seed, stream, counter)`` triple,
``prng.py:37-47``) and ``split`` is exact 64-bit integer arithmetic
(``prng.py:84-94``).  Every *draw* is made by the device generator
(``csrc/prng.cuh`` through ``fsmc_prng_fill``), the same code the samplers
use, so a value returned here is bit-identical to what a chain consumes.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _lib

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_MIX_A = 0xBF58476D1CE4E5B9
_MIX_B = 0x94D049BB133111EB

__all__ = ["RngKey", "key", "split", "uniform", "normal", "normal_vec", "uniform_block",
           "bits_block", "normal_block"]


class RngKey(NamedTuple):
    """Immutable position in a random stream (prng.py:37-42)."""

    seed: int
    stream: int
    counter: int


def key(seed: int, stream: int = 0, counter: int = 0) -> RngKey:
    """prng.py:45-47: all fields reduced to 64-bit unsigned range."""
    return RngKey(seed & _MASK64, stream & _MASK64, counter & _MASK64)


def _mix64(x: int) -> int:
    x &= _MASK64
    x = ((x ^ (x >> 30)) * _MIX_A) & _MASK64
    x = ((x ^ (x >> 27)) * _MIX_B) & _MASK64
    return x ^ (x >> 31)


def split(k: RngKey, n_streams: int) -> list[RngKey]:
    """prng.py:84-94: child streams mix64(parent*G + i + 1), counters reset."""
    if n_streams < 1:
        raise ValueError(f"n_streams must be >= 1, got {n_streams}")
    base = (k.stream * _GOLDEN) & _MASK64
    return [RngKey(k.seed, _mix64(base + i + 1), 0) for i in range(n_streams)]


def _fill(k: RngKey, count: int, kind: int) -> torch.Tensor:
    dtype = torch.int64 if kind == 0 else torch.float64
    out = torch.empty(count, dtype=dtype, device="cuda")
    _lib.check(_lib.lib().fsmc_prng_fill(k.seed, k.stream, k.counter, count, kind,
                                         out.data_ptr(), _lib.stream_ptr()), "fsmc_prng_fill")
    return out


def _advance(k: RngKey, count: int) -> RngKey:
    return RngKey(k.seed, k.stream, (k.counter + count) & _MASK64)


def uniform(k: RngKey) -> tuple[float, RngKey]:
    """One uniform in [0, 1); advances the counter by 1 (prng.py:97-100)."""
    return float(_fill(k, 1, 1).item()), _advance(k, 1)


def normal(k: RngKey) -> tuple[float, RngKey]:
    """One standard normal, ndtri((bits53 + 0.5) 2^-53) (prng.py:103-111)."""
    return float(_fill(k, 1, 2).item()), _advance(k, 1)


def normal_vec(k: RngKey, dim: int, chol_factor: np.ndarray | None = None
               ) -> tuple[np.ndarray, RngKey]:
    """``L @ z`` for a standard normal z; consumes ``dim`` counters (prng.py:114-136)."""
    if dim < 1:
        raise ValueError(f"dim must be >= 1, got {dim}")
    if chol_factor is not None:
        L = np.asarray(chol_factor, dtype=float)
        if L.shape != (dim, dim):
            raise ValueError(f"chol_factor has shape {L.shape}, expected {(dim, dim)}")
        if np.any(np.triu(L, 1) != 0.0) or np.any(np.diag(L) <= 0.0):
            raise ValueError("chol_factor must be lower-triangular with positive diagonal")
    z = _fill(k, dim, 2)
    if chol_factor is not None:
        z = torch.as_tensor(L, device="cuda") @ z
    return z.cpu().numpy(), _advance(k, dim)


def uniform_block(k: RngKey, count: int) -> tuple[np.ndarray, RngKey]:
    """``count`` uniforms from consecutive counters (prng.py:139-153)."""
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    return _fill(k, count, 1).cpu().numpy(), _advance(k, count)


def normal_block(k: RngKey, count: int) -> tuple[torch.Tensor, RngKey]:
    """Device tensor of ``count`` normals from consecutive counters."""
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    return _fill(k, count, 2), _advance(k, count)


def bits_block(k: RngKey, count: int) -> tuple[np.ndarray, RngKey]:
    """The raw 64-bit words ``_bits(seed, stream, counter + i)`` (prng.py:58-81)."""
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    return _fill(k, count, 0).cpu().numpy().view(np.uint64), _advance(k, count)
