"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel path (build, sort classes incl. merge, reindex, degree
rows, TD/BU/conversions, output passes, device-driven graph loop and host loop,
persistent and one-cluster searches, the one-kernel small top-down step, tile mode,
multi-partition local transport with claim lists and with bitmap pushes).
SANITIZE_SKIP_GRAPH=1 leaves out the conditional loop graph (racecheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_04359_b200 as pkg  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
for opts in (pkg.default_opts(), pkg.default_opts(reindex_by_degree=True), pkg.default_opts(sort_rows=2),
             pkg.default_opts(False, False, False, 1)):
    g = pkg.Graph.kronecker(11, 16, 3, opts=opts)
    loops = ["host", "persistent", "cluster"] + ([] if os.environ.get("SANITIZE_SKIP_GRAPH") else ["graph"])
    for pol in [dict(mode=0, loop=lp) for lp in loops] + [dict(mode=1, loop="host"), dict(mode=2, bu_from_level=0, loop="host"),
                dict(mode=3, alpha=500, beta=2, loop="host"), dict(mode=1, loop=loops[-1])]:
        g.set_policy(**pol)
        for r in g.sample_roots(11, 3, 3):
            g.run(int(r))
            g.stats()
    g.close()
# tile mode on a small reindexed graph (tiny tiles, low heavy threshold, every top-down step)
os.environ.update(BFS_TILE_H="8", BFS_TILE_WORDS="4", BFS_TILE_COUNT="37", BFS_TILE_MIN="1", BFS_TD_SMALL="-1")
g = pkg.Graph.kronecker(11, 16, 3, opts=pkg.default_opts(reindex_by_degree=True))
assert pkg.bfs_graph_tiles(g.h)["tiles"] > 0
for lp in ["host"] + ([] if os.environ.get("SANITIZE_SKIP_GRAPH") else ["graph"]):
    for mode in (0, 1):
        g.set_policy(mode=mode, loop=lp)
        for r in g.sample_roots(11, 3, 2):
            g.run(int(r))
g.close()
for k in ("BFS_TILE_H", "BFS_TILE_WORDS", "BFS_TILE_COUNT", "BFS_TILE_MIN", "BFS_TD_SMALL"):
    del os.environ[k]
# a hub row longer than the shared-memory sort (merge path)
n = 1 << 16
uv = np.concatenate([np.stack([np.zeros(40000, np.int64), rng.integers(0, n, 40000)], 1),
                     rng.integers(0, n, size=(20000, 2))]).astype(np.int32)
g = pkg.Graph.from_edges(uv, n)
g.run(0)
h = np.empty(n, np.int32)
pkg.bfs_run(g.h, 0, h, None)
g.close()
# multi-partition with the degree reindex and the final aggregation (local transport)
comms_r = pkg.bfs_comm_create_local(2, 0)
gr = pkg.run_ranks(lambda r: pkg.Graph.kronecker(10, 16, 2, comm=comms_r[r], stream=torch.cuda.Stream(),
                                                 opts=pkg.default_opts(reindex_by_degree=True)), 2)
def go_r(r):
    torch.cuda.set_device(0)
    gr[r].run(5)
    return gr[r].stats()
pkg.run_ranks(go_r, 2)
for x in gr:
    x.close()
# multi-partition (local transport), claim lists and bitmap pushes
os.environ["BFS_TD_BITMAP_MIN"] = "1"
comms_b = pkg.bfs_comm_create_local(2, 0)
gb = pkg.run_ranks(lambda r: pkg.Graph.kronecker(10, 16, 2, comm=comms_b[r], stream=torch.cuda.Stream()), 2)
def go_b(r):
    torch.cuda.set_device(0)
    gb[r].set_policy(mode=1)
    gb[r].run(5)
    return gb[r].stats()
pkg.run_ranks(go_b, 2)
for x in gb:
    x.close()
del os.environ["BFS_TD_BITMAP_MIN"]
comms = pkg.bfs_comm_create_local(3, 0)
gs = pkg.run_ranks(lambda r: pkg.Graph.kronecker(10, 16, 2, comm=comms[r], stream=torch.cuda.Stream()), 3)
def go(r):
    torch.cuda.set_device(0)
    gs[r].run(5)
    return gs[r].stats()
pkg.run_ranks(go, 3)
for x in gs:
    x.close()
print("sanitize workload done")
