"""Per-root device time and per-level kernel times of K29 searches (A/B helper).

    python tools/level_times.py --roots 64 [--reps 2]
prints one JSON line: total ms over the roots, per-root ms, and the top-down levels'
kernel ms with m_f >= 2^24 (the tile-mode levels).
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
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--alpha", type=int, default=30)
ap.add_argument("--tag", default="")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
g.set_policy(mode=0, alpha=a.alpha, beta=1000, level_times=True)
parent = torch.empty(g.n, dtype=torch.int32, device="cuda")
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
per, td, bu = [], [], []
for r in g.sample_roots(cfg["scale"], cfg["seed"], a.roots):
    best = None
    for _ in range(a.reps):
        pkg.bfs_run(g.h, int(r), parent, depth)
        run, lv = g.stats(tuples=False)
        if best is None or run["ms_total"] < best[0]:
            best = (run["ms_total"], lv)
    per.append(round(best[0], 4))
    td += [round(x["kernel_ms"], 4) for x in best[1] if x["direction"] == 0 and x["m_f"] >= 1 << 24]
    bu += [round(x["kernel_ms"], 4) for x in best[1] if x["direction"] == 1]
print(json.dumps({"tag": a.tag, "total_ms": round(sum(per), 3), "hmean_ms": round(len(per) / sum(1 / x for x in per), 4),
                  "tile_td_ms": round(sum(td), 3), "bu_ms": round(sum(bu), 3), "per_root": per}), flush=True)
