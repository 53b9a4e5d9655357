"""Fig. 4-left analogue: per-level device time of the classic
top-down-only BFS vs direction-optimized BFS (and the paper's section 3.3 rule) on the
same roots of one graph, from the library's per-step device stamps.

    python tools/fig4_levels.py --config k29 --roots 4
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_04359_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="k26")
ap.add_argument("--roots", type=int, default=4)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
roots = g.sample_roots(cfg["scale"], cfg["seed"], a.roots)
pols = {"TD-only": dict(mode=1), "DO a30/b1000": dict(mode=0, alpha=30, beta=1000),
        "paper 0.05/3": dict(mode=3, alpha=500, beta=3)}
print(f"# {cfg['name']}, per-level device ms (direction T/B, frontier size), total ms and GTEPS per search")
for r in roots:
    print(f"root {int(r)}")
    for name, pol in pols.items():
        g.set_policy(level_times=True, **pol)
        g.run(int(r))                      # warm
        g.run(int(r))
        run, levels = g.stats()
        cells = " ".join(f"{'TB'[lv['direction']]}{lv['frontier']}:{lv['ms']:.3f}" for lv in levels)
        print(f"  {name:13s} total {run['ms_total']:8.3f} ms  {run['component_edge_tuples'] / run['ms_total'] / 1e6:8.1f} GTEPS  | {cells}")
g.close()
