"""Edge-list ingestion for real graphs (SPEC S:110-118 `load_edge_list`).

Host-side parsing only: the result feeds `Graph.from_edges` (bfs_graph_create_edges), which
builds the CSR on the device.  Two formats:

- text: one "u v" pair per line (whitespace separated, extra columns ignored, '#' or '%'
  starts a comment, blank lines skipped);
- binary: little-endian int32 or int64 (u, v) pairs, no header.

Vertex IDs are relabeled densely in order of first appearance ("dense relabeled vertex
IDs, stable mapping emitted alongside"); n = number of distinct endpoints, or `n_hint` when the
caller declares a larger vertex count (isolated padding).  An unparseable text line raises
ValueError naming its line number; an empty file is an empty graph.
"""
from __future__ import annotations

import numpy as np


def _parse_text(path: str) -> np.ndarray:
    pairs = []
    with open(path, "r") as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s or s[0] in "#%":
                continue
            parts = s.split()
            if len(parts) < 2:
                raise ValueError(f"{path}:{ln}: expected 'u v', got {line.rstrip()!r}")
            try:
                pairs.append((int(parts[0]), int(parts[1])))
            except ValueError:
                raise ValueError(f"{path}:{ln}: not an integer pair: {line.rstrip()!r}") from None
    return np.asarray(pairs, dtype=np.int64).reshape(-1, 2)


def load_edge_list(path: str, fmt: str = "text", n_hint: int | None = None):
    """-> (uv int32[m, 2] dense labels, n, original_ids int64[n]) ; original_ids[i] is the file ID of label i."""
    if fmt == "text":
        raw = _parse_text(path)
    elif fmt in ("bin32", "bin64"):
        raw = np.fromfile(path, dtype=np.int32 if fmt == "bin32" else np.int64).astype(np.int64)
        if raw.size % 2:
            raise ValueError(f"{path}: odd number of integers in a pair file")
        raw = raw.reshape(-1, 2)
    else:
        raise ValueError(f"unknown edge-list format {fmt!r}")
    if raw.size == 0:
        n = int(n_hint or 0)
        return np.zeros((0, 2), np.int32), n, np.arange(n, dtype=np.int64)
    flat = raw.reshape(-1)
    # first-appearance order: unique with return_index, then sort the uniques by first index
    uniq, first, inv = np.unique(flat, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    labels = rank[inv].reshape(-1, 2)
    n = int(uniq.size)
    if n_hint is not None:
        if n_hint < n:
            raise ValueError(f"declared vertex count {n_hint} < {n} distinct endpoints")
        n = int(n_hint)
    if n > np.iinfo(np.int32).max:
        raise ValueError("more than 2^31-1 vertices")
    ids = np.full(n, -1, np.int64)
    ids[: uniq.size] = uniq[order]
    return labels.astype(np.int32), n, ids
