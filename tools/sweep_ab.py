"""Direction-switch tuning sweep: one graph, 64 roots per
(alpha, beta) setting, harmonic-mean GTEPS from the library's device timers."""
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
ap.add_argument("--config", default="k26")
ap.add_argument("--alphas", default="5,10,15,30,60")
ap.add_argument("--betas", default="2,6,18,24")
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--reindex", type=int, default=0)
ap.add_argument("--rows", type=int, default=1)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"],
                        opts=pkg.default_opts(reindex_by_degree=bool(a.reindex), sort_rows=a.rows))
print("build_ms", g.build_ms, flush=True)
roots = g.sample_roots(cfg["scale"], cfg["seed"], a.roots)
parent = torch.empty(g.n, dtype=torch.int32, device="cuda")
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
edges = {}
res = []
for alpha in [int(x) for x in a.alphas.split(",")]:
    for beta in [int(x) for x in a.betas.split(",")]:
        g.set_policy(mode=0, alpha=alpha, beta=beta)
        rates = []
        for r in roots:
            pkg.bfs_run(g.h, int(r), parent, depth)
            run, _ = g.stats(tuples=True)
            rates.append(run["component_edge_tuples"] / (run["ms_total"] * 1e-3) / 1e9)
        res.append({"alpha": alpha, "beta": beta, "gteps": bench.hmean(rates)})
        print(json.dumps(res[-1]), flush=True)
best = max(res, key=lambda x: x["gteps"])
print("best", json.dumps(best))
