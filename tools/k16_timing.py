"""Small-graph level-loop comparison (K16 by default): device time per search for every
level loop, with and without the degree reindex.

    python tools/k16_timing.py [scale]
"""
import os
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1503_04359_b200 as pkg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
torch.cuda.set_device(0)
for reindex in (True, False):
    g = pkg.Graph.kronecker(scale, 16, 1, opts=pkg.default_opts(reindex_by_degree=reindex))
    roots = g.sample_roots(scale, 1, 64)
    p = torch.empty(g.n, dtype=torch.int32, device='cuda')
    d = torch.empty_like(p)
    edges = {}
    for r in roots:
        pkg.bfs_run(g.h, int(r), p, d)
        edges[int(r)] = pkg.bfs_component_tuples(g.h)
    for loop, env in (("persistent", None), ("graph", None), ("host", None), ("cluster", "16"), ("cluster", "8")):
        if env:
            os.environ["BFS_CLUSTER"] = env
        g.set_policy(mode=0, alpha=30, beta=1000, loop=loop)
        for r in roots:
            pkg.bfs_run(g.h, int(r), p, d)
        tot = ini = comp = 0
        rates = []
        for r in roots:
            pkg.bfs_run(g.h, int(r), p, d)
            run, lv = g.stats(tuples=False)
            tot += run['ms_total']
            ini += run['ms_init']
            comp += run['ms_compute']
            rates.append(edges[int(r)] / (run['ms_total'] * 1e-3) / 1e9)
        k = len(roots)
        hm = len(rates) / sum(1 / x for x in rates)
        print(f"s{scale} reindex={reindex} {loop:10s} {env or '':3s} total {tot/k*1000:7.1f} us  init {ini/k*1000:6.1f}  "
              f"loop {comp/k*1000:6.1f}  rest {(tot-ini-comp)/k*1000:6.1f}  hmean {hm:7.2f} GTEPS", flush=True)
    g.close()
