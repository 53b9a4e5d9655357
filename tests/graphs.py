"""Seeded synthetic inputs shared by the oracle tests and the GPU parity tests.

This module holds no arithmetic of the method (no BFS, no CSR, no generator):
it only writes down small hand-built edge lists and seeded random edge lists
as int32 [m, 2] arrays.  Both sides (oracle and CUDA path) build their own
CSR from these tuples.
"""
from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _e(pairs) -> np.ndarray:
    a = np.asarray(list(pairs), dtype=np.int32)
    return a.reshape(-1, 2)


def load_golden_edges(name: str) -> np.ndarray:
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#") or not line[0].isdigit():
                continue
            parts = line.split()
            if len(parts) == 2:
                rows.append((int(parts[0]), int(parts[1])))
    return _e(rows)


def load_golden_table(name: str) -> dict:
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            out[key] = [int(x) for x in vals]
    return out


def g1():
    return 6, load_golden_edges("g1.txt")


def path(n):
    return n, _e((i, i + 1) for i in range(n - 1))


def cycle(n):
    return n, _e((i, (i + 1) % n) for i in range(n))


def star(n):
    """centre 0, leaves 1..n-1"""
    return n, _e((0, i) for i in range(1, n))


def clique(n):
    return n, _e((i, j) for i in range(n) for j in range(i + 1, n))


def complete_bipartite(a, b):
    return a + b, _e((i, a + j) for i in range(a) for j in range(b))


def hypercube(dim):
    n = 1 << dim
    return n, _e((v, v ^ (1 << k)) for v in range(n) for k in range(dim) if v < v ^ (1 << k))


def grid(r, c):
    pairs = []
    for i in range(r):
        for j in range(c):
            v = i * c + j
            if j + 1 < c:
                pairs.append((v, v + 1))
            if i + 1 < r:
                pairs.append((v, v + c))
    return r * c, _e(pairs)


def heap_tree(n):
    """binary heap: parent of i is (i-1)//2"""
    return n, _e(((i - 1) // 2, i) for i in range(1, n))


def random_edges(n, m, seed, self_loops=True):
    rng = np.random.default_rng(seed)
    uv = rng.integers(0, n, size=(m, 2), dtype=np.int64).astype(np.int32)
    if not self_loops:
        keep = uv[:, 0] != uv[:, 1]
        uv = uv[keep]
    return n, uv


def skewed_edges(n, m, seed):
    """power-law-ish endpoints (a few hubs, many leaves) for ragged degree mixes"""
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, n + 1) ** 1.1
    w /= w.sum()
    perm = rng.permutation(n)
    u = perm[rng.choice(n, size=m, p=w)]
    v = rng.integers(0, n, size=m)
    return n, np.stack([u, v], 1).astype(np.int32)


def disjoint_union(*graphs):
    off = 0
    parts = []
    for n, uv in graphs:
        parts.append(uv + off)
        off += n
    return off, np.concatenate(parts) if parts else _e([])
