"""Sweep a library tuning knob read from the environment at each bfs_run (e.g.
BFS_HUB_BITS): one graph, 64 roots per value (run twice, second pass kept),
harmonic-mean GTEPS from the library's device timers.

    python tools/sweep_env.py --var BFS_HUB_BITS --values 0,8192,32768 [--config k29]
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
ap.add_argument("--var", required=True)
ap.add_argument("--values", required=True)
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--alpha", type=int, default=30)
ap.add_argument("--beta", type=int, default=1000)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
print("build_ms", g.build_ms, flush=True)
roots = g.sample_roots(cfg["scale"], cfg["seed"], a.roots)
parent = torch.empty(g.n, dtype=torch.int32, device="cuda")
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
g.set_policy(mode=0, alpha=a.alpha, beta=a.beta)
edges = {}
for rep in range(2):
    for val in a.values.split(","):
        os.environ[a.var] = val
        rates = []
        parts = [0.0, 0.0, 0.0]   # init, level loop, output pass (device ms, summed)
        for r in roots:
            pkg.bfs_run(g.h, int(r), parent, depth)
            run, _ = g.stats(tuples=int(r) not in edges)
            if int(r) not in edges:
                edges[int(r)] = run["component_edge_tuples"]
            rates.append(edges[int(r)] / (run["ms_total"] * 1e-3) / 1e9)
            parts[0] += run["ms_init"]
            parts[1] += run["ms_compute"]
            parts[2] += run["ms_total"] - run["ms_init"] - run["ms_compute"]
        if rep == 1:
            k = len(roots)
            print(json.dumps({a.var: val, "gteps": round(bench.hmean(rates), 2),
                              "ms_init": round(parts[0] / k, 4), "ms_loop": round(parts[1] / k, 4),
                              "ms_output": round(parts[2] / k, 4)}), flush=True)
