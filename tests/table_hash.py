"""Checksums of C tables for full-size parity (test infrastructure).

The config-4 table (L=1000, S=4000: 501,501 rows of 4,001 fp64 values, 16 GB)
cannot be stored as a fixture, so `scripts/make_golden_cfg4.py` (oracle only)
records checksums of it and the GPU test recomputes them from the product's
exported rows.  No method arithmetic is here: only a hash of fp64 bit patterns.

row hash      h(s,t) = sum_m bits(C[s,t,m]) * K[m]            (mod 2^64)
per-s hash    H_s    = sum_{t=s..n} h(s,t) * K2[t]            (mod 2^64)
per-d hash    G_d    = sum_{s=1..n-d} h(s,s+d) * K2[s]        (mod 2^64)

K, K2 are odd splitmix64 outputs, so a change of any single value of a row
changes h, and a change of a single h changes its H_s and G_d: a mismatch is
located to the cell (s, s+d) where both differ.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix_stream(seed: int, count: int) -> np.ndarray:
    """count outputs of splitmix64 from `seed` (vectorised; uint64 wrap-around)."""
    with np.errstate(over="ignore"):
        st = np.uint64(seed) + np.arange(1, count + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        z = st
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def row_keys(width: int) -> np.ndarray:
    return splitmix_stream(0x5EED0001, width) | np.uint64(1)


def cell_keys(n: int) -> np.ndarray:
    """K2[i] for i = 0..n (index = stage)."""
    return splitmix_stream(0x5EED0002, n + 1) | np.uint64(1)


def row_hashes(rows: np.ndarray) -> np.ndarray:
    """rows: (R, W) float64 -> (R,) uint64 row hashes."""
    bits = np.ascontiguousarray(rows).view(np.uint64)
    K = row_keys(bits.shape[1])
    with np.errstate(over="ignore"):
        return (bits * K[None, :]).sum(axis=1, dtype=np.uint64)


def cell_index(n: int, s: int, t: int) -> int:
    r = s - 1
    return r * n - r * (r - 1) // 2 + (t - s)


class TableHasher:
    """Accumulates H_s / G_d from row hashes fed in any order."""

    def __init__(self, n: int):
        self.n = n
        self.K2 = cell_keys(n)
        self.H = np.zeros(n + 1, dtype=np.uint64)  # index s (1..n)
        self.G = np.zeros(n, dtype=np.uint64)  # index d (0..n-1)
        self.rows = 0

    def add(self, s: np.ndarray, t: np.ndarray, h: np.ndarray):
        s = np.asarray(s, dtype=np.int64)
        t = np.asarray(t, dtype=np.int64)
        with np.errstate(over="ignore"):
            np.add.at(self.H, s, h * self.K2[t])
            np.add.at(self.G, t - s, h * self.K2[s])
        self.rows += len(h)

    def complete(self) -> bool:
        return self.rows == self.n * (self.n + 1) // 2


def all_cells(n: int):
    """(s, t) arrays of every cell in the canonical (s-major) order."""
    s = np.repeat(np.arange(1, n + 1, dtype=np.int64), np.arange(n, 0, -1))
    first = np.concatenate([[0], np.cumsum(np.arange(n, 0, -1))[:-1]])
    t = s + (np.arange(len(s)) - np.repeat(first, np.arange(n, 0, -1)))
    return s, t


def hash_canonical_table(C: np.ndarray, n: int, chunk: int = 8192) -> TableHasher:
    """Hash a whole canonical-layout table (cells, S+1) held in host memory."""
    hs = TableHasher(n)
    s_all, t_all = all_cells(n)
    for lo in range(0, C.shape[0], chunk):
        hi = min(lo + chunk, C.shape[0])
        hs.add(s_all[lo:hi], t_all[lo:hi], row_hashes(C[lo:hi]))
    return hs


def write_hex(f, name: str, values):
    f.write(f"list:{name} {len(values)}\n")
    for v in values:
        f.write(f"{int(v):016x}\n")


def read_golden(path: str) -> dict:
    """Parse the golden file: 'key value' scalars and 'name count' + count hex lines."""
    out = {}
    with open(path) as f:
        lines = [ln.rstrip("\n") for ln in f if not ln.startswith("#")]
    i = 0
    while i < len(lines):
        parts = lines[i].split()
        i += 1
        if not parts:
            continue
        key = parts[0]
        if key.startswith("list:"):
            cnt = int(parts[1])
            out[key[5:]] = [int(x, 16) for x in lines[i: i + cnt]]
            i += cnt
        else:
            out[key] = parts[1] if len(parts) == 2 else parts[1:]
    return out
