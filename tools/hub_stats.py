"""Per-level frontier statistics of K29 searches, for sizing the tiled top-down step:
degree histogram of the reindexed graph (vertices with degree >= H), and per level
the frontier size, m_f, and the share of m_f from frontier vertices of degree >= H.

    python tools/hub_stats.py --config k29 --roots 8
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
ap.add_argument("--roots", type=int, default=8)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
n = g.n
off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
pkg.bfs_graph_export_csr(g.h, off, None)
deg = (off[1:] - off[:-1])
label = torch.empty(n, dtype=torch.int32, device="cuda")
pkg.bfs_graph_export_labels(g.h, label)
res = {"n": n, "arcs": int(off[-1]), "n_active": int((deg > 0).sum()), "heavy": {}}
for H in (256, 1024, 4096, 16384, 65536):
    m = deg >= H
    res["heavy"][H] = {"count": int(m.sum()), "arcs": int(deg[m].sum())}
print(json.dumps(res), flush=True)
roots = g.sample_roots(cfg["scale"], cfg["seed"], a.roots)
g.set_policy(mode=0, alpha=30, beta=1000, level_times=True)
per = []
parent = torch.empty(n, dtype=torch.int32, device="cuda")
depth = torch.empty(n, dtype=torch.int32, device="cuda")
for r in roots:
    pkg.bfs_run(g.h, int(r), parent, depth)
    run, levels = g.stats(tuples=False)
    di = torch.empty_like(depth)
    di[label.long()] = depth          # depth by internal label
    rows = []
    for lv in levels:
        d = lv["level"]
        fr = di == d
        row = {"dir": lv["direction"], "F": lv["frontier"], "m_f": lv["m_f"], "D": lv["discovered"],
               "insp": lv["inspections"], "ms": round(lv["kernel_ms"], 4)}
        for H in (1024, 4096, 16384):
            hm = fr & (deg >= H)
            row[f"F{H}"] = int(hm.sum())
            row[f"mf{H}"] = int(deg[hm].sum())
        rows.append(row)
    per.append({"root": int(r), "ms": round(run["ms_total"], 4), "levels": rows})
    print(json.dumps(per[-1]), flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump({"graph": res, "roots": per}, f, indent=1)
