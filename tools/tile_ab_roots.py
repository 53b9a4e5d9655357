"""Per-root A/B of the tiled top-down step in one process (BFS_TILE_MIN is read per
search): every sampled root with tile mode on and off, levels of the roots that differ.

    python tools/tile_ab_roots.py --config k29 --roots 64
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
ap.add_argument("--config", default="k29")
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--alpha", type=int, default=30)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=pkg.default_opts(reindex_by_degree=True))
print("tiles", pkg.bfs_graph_tiles(g.h), flush=True)
g.set_policy(mode=0, alpha=a.alpha, beta=1000, level_times=True)
parent = torch.empty(g.n, dtype=torch.int32, device="cuda")
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
default_min = os.environ.get("BFS_TILE_MIN")


def run(r, on):
    if on:
        if default_min is None:
            os.environ.pop("BFS_TILE_MIN", None)
        else:
            os.environ["BFS_TILE_MIN"] = default_min
    else:
        os.environ["BFS_TILE_MIN"] = str(1 << 62)
    best = None
    for _ in range(a.reps):
        pkg.bfs_run(g.h, int(r), parent, depth)
        run_, lv = g.stats(tuples=False)
        if best is None or run_["ms_total"] < best[0]:
            best = (run_["ms_total"], [("TB"[x["direction"]], x["frontier"], round(x["ms"], 3)) for x in lv])
    return best


tot_on = tot_off = 0.0
for r in g.sample_roots(cfg["scale"], cfg["seed"], a.roots):
    on, off = run(r, True), run(r, False)
    tot_on += on[0]
    tot_off += off[0]
    flag = "  <-- slower" if on[0] > off[0] * 1.03 else ""
    print(int(r), round(on[0], 3), round(off[0], 3), flag, flush=True)
    if flag or on[0] < off[0] * 0.9:
        print("    on ", on[1])
        print("    off", off[1])
print("total", round(tot_on, 2), round(tot_off, 2))
