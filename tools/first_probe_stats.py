"""For each level of a few K29 searches: the share of the vertices discovered at depth
d+1 whose FIRST neighbour (row order = highest degree) sits at depth d (a first-probe
parent), per direction.  Sizing aid for the tile-mode finish pass.

    python tools/first_probe_stats.py --roots 6
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_04359_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="k29")
ap.add_argument("--roots", type=int, default=6)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
n = g.n
off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
pkg.bfs_graph_export_csr(g.h, off, None)
deg = off[1:] - off[:-1]
act = deg > 0
first = torch.full((n,), -1, dtype=torch.int64, device="cuda")
idx = torch.nonzero(act).squeeze(1)
# first neighbour of every active row, read row by row through export_row is too slow:
# gather adj[off[v]] with a device copy of the adjacency in chunks
arcs = int(off[-1])
adj = torch.empty(arcs, dtype=torch.int32, device="cuda")
pkg.bfs_graph_export_csr(g.h, None, adj)
first[idx] = adj[off[idx]].long()
label = torch.empty(n, dtype=torch.int32, device="cuda")
pkg.bfs_graph_export_labels(g.h, label)
g.set_policy(mode=0, alpha=30, beta=1000, level_times=True)
parent = torch.empty(n, dtype=torch.int32, device="cuda")
depth = torch.empty(n, dtype=torch.int32, device="cuda")
for r in g.sample_roots(cfg["scale"], cfg["seed"], a.roots):
    pkg.bfs_run(g.h, int(r), parent, depth)
    run, levels = g.stats(tuples=False)
    di = torch.empty_like(depth)
    di[label.long()] = depth
    rows = []
    for lv in levels:
        d = lv["level"]
        new = (di == d + 1)
        cnt = int(new.sum())
        if cnt == 0:
            continue
        fd = di[first[new].clamp(min=0)]
        hit = int((fd == d).sum())
        rows.append(("TB"[lv["direction"]], lv["frontier"], cnt, round(hit / cnt, 4)))
    print(int(r), rows, flush=True)
