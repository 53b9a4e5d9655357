"""Run-to-run variance of K29 searches: every sampled root R times (graph loop, level
times on); prints per root the min/max search ms and, for the slowest repetition,
the level that differs most from the fastest one.

    python tools/td_variance.py --reps 6
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
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--no-output", action="store_true", help="searches without the output pass (null outputs)")
a = ap.parse_args()
cfg = bench.CONFIGS["k29"]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
g.set_policy(mode=0, alpha=30, beta=1000, level_times=True)
roots = g.sample_roots(cfg["scale"], cfg["seed"], a.roots)
parent = torch.empty(g.n, dtype=torch.int32, device="cuda")
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
res = {int(r): [] for r in roots}
for rep in range(a.reps):
    for r in roots:
        if a.no_output:
            pkg.bfs_run(g.h, int(r), None, None)
        else:
            pkg.bfs_run(g.h, int(r), parent, depth)
        run, levels = g.stats(tuples=False)
        res[int(r)].append((run["ms_total"], [(lv["direction"], round(lv["ms"], 3), round(lv["kernel_ms"], 3)) for lv in levels]))
out = []
for r, runs in res.items():
    ts = [x[0] for x in runs]
    lo, hi = min(range(len(ts)), key=lambda i: ts[i]), max(range(len(ts)), key=lambda i: ts[i])
    worst = max(range(len(runs[lo][1])), key=lambda d: runs[hi][1][d][1] - runs[lo][1][d][1]) if runs[lo][1] else -1
    out.append({"root": r, "min_ms": round(ts[lo], 3), "max_ms": round(ts[hi], 3), "spread": round(ts[hi] / ts[lo], 3),
                "level": worst, "fast": runs[lo][1][worst] if worst >= 0 else None, "slow": runs[hi][1][worst] if worst >= 0 else None})
out.sort(key=lambda x: -x["spread"])
for x in out[:12]:
    print(json.dumps(x))
print(json.dumps({"roots": len(out), "spread>1.2": sum(x["spread"] > 1.2 for x in out)}))
