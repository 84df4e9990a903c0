"""Seeded synthetic workload streams, vectorised with numpy.

The same splitmix64 stream as HeadMatrix::random (head.cpp:89-107) is used
for every input, so the workload is portable and reproducible:
  W      = HeadMatrix::random(V, d, 0x5EED)    (generated on the device)
  hidden = rows of HeadMatrix::random(steps*B, d, 0x41DD)
  T      = first n distinct ids of splitmix64(0x57A7) mod V
  prompt = L ids of splitmix64(0x9A0 + request) mod V
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
SEED_W, SEED_H, SEED_T, SEED_P = 0x5EED, 0x41DD, 0x57A7, 0x9A0


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix_stream(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Outputs start..start+n-1 of the splitmix64 sequence seeded with seed."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        return _mix(np.uint64(seed) + k * GAMMA)


def head_random(rows: int, dim: int, seed: int, first: int = 0) -> np.ndarray:
    """HeadMatrix::random values (fp32), elements [first, first+rows*dim)."""
    z = splitmix_stream(seed, rows * dim, first)
    r = (z >> np.uint64(40)).astype(np.float32)
    return (r * np.float32(2.0 ** -23) - np.float32(1.0)).astype(np.float32).reshape(rows, dim)


def round_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    r = ((u + np.uint32(0x7FFF) + lsb) >> np.uint32(16)) << np.uint32(16)
    return r.astype(np.uint32).view(np.float32)


def static_ids(V: int, n: int, seed: int = SEED_T) -> np.ndarray:
    """First n distinct ids of splitmix64(seed) mod V, in draw order."""
    out, seen, start = [], set(), 0
    while len(out) < n:
        chunk = (splitmix_stream(seed, 4 * n, start) % np.uint64(V)).astype(np.int64)
        start += 4 * n
        for i in chunk:
            if i not in seen:
                seen.add(int(i))
                out.append(int(i))
                if len(out) == n:
                    break
    return np.array(out, np.uint32)


def prompt_ids(V: int, L: int, request: int, seed: int = SEED_P) -> np.ndarray:
    return (splitmix_stream(seed + request, L) % np.uint64(V)).astype(np.uint32)


def words_of(ids: np.ndarray, V: int) -> np.ndarray:
    w = np.zeros((V + 63) // 64, np.uint64)
    ids = np.asarray(ids, np.uint64)
    np.bitwise_or.at(w, (ids // np.uint64(64)).astype(np.int64),
                     np.left_shift(np.uint64(1), ids % np.uint64(64)))
    return w
