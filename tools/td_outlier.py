"""Frontier composition of the hub top-down level for given K29 roots: degree
classes of the frontier, its largest rows and their share of m_f (why two roots with
the same F and m_f differ in tile-mode time).

    python tools/td_outlier.py 86254516 452924735 ...
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_04359_b200 as pkg  # noqa: E402

cfg = bench.CONFIGS["k29"]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
n = g.n
off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
pkg.bfs_graph_export_csr(g.h, off, None)
deg = off[1:] - off[:-1]
label = torch.empty(n, dtype=torch.int32, device="cuda")
pkg.bfs_graph_export_labels(g.h, label)
g.set_policy(mode=0, alpha=30, beta=1000, level_times=True)
parent = torch.empty(n, dtype=torch.int32, device="cuda")
depth = torch.empty(n, dtype=torch.int32, device="cuda")
for r in [int(x) for x in sys.argv[1:]]:
    pkg.bfs_run(g.h, r, parent, depth)
    run, levels = g.stats(tuples=False)
    di = torch.empty_like(depth)
    di[label.long()] = depth
    for lv in levels:
        if lv["direction"] != 0 or lv["m_f"] < (1 << 24):
            continue
        fr = torch.nonzero(di == lv["level"]).flatten()
        fd = deg[fr]
        top = torch.topk(fd, min(8, fd.numel()))
        out = {"root": r, "level": lv["level"], "F": lv["frontier"], "m_f": lv["m_f"], "ms": round(lv["ms"], 3),
               "kernel_ms": round(lv["kernel_ms"], 3), "max_label": int(fr.max()), "top_degrees": top.values.tolist(),
               "top_labels": fr[top.indices].tolist()}
        for H in (4096, 16384, 65536, 1 << 20):
            m = fd >= H
            out[f"F>={H}"] = int(m.sum())
            out[f"mf>={H}"] = int(fd[m].sum())
        print(json.dumps(out), flush=True)
