"""Small driver for ncu captures: build one config's graph, run R roots.

    ncu ... python tools/profile_run.py --config k26 --roots 2
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
ap.add_argument("--roots", type=int, default=2)
ap.add_argument("--skip", type=int, default=0, help="roots to skip (sampled order)")
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--root", type=int, default=-1, help="run this root (original label) instead of sampled ones")
ap.add_argument("--reindex", type=int, default=0)
ap.add_argument("--alpha", type=int, default=30)
ap.add_argument("--beta", type=int, default=1000)
ap.add_argument("--reps", type=int, default=1, help="run the root list this many times")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"],
                        opts=pkg.default_opts(reindex_by_degree=bool(a.reindex)))
print("build_ms", g.build_ms, flush=True)
roots = [a.root] if a.root >= 0 else g.sample_roots(cfg["scale"], cfg["seed"], a.skip + a.roots)[a.skip:]
roots = list(roots) * a.reps
g.set_policy(mode=a.mode, alpha=a.alpha, beta=a.beta, level_times=True)
for r in roots:
    p, d = g.run(int(r))
    run, levels = g.stats()
    print(int(r), round(run["ms_total"], 4), [(lv["direction"], lv["frontier"], round(lv["kernel_ms"], 4)) for lv in levels])
torch.cuda.synchronize()
