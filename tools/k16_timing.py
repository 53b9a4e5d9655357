import sys; sys.path.insert(0, '.')
import torch, paper_1503_04359_b200 as pkg, bench
torch.cuda.set_device(0)
for reindex in (True, False):
    g = pkg.Graph.kronecker(16, 16, 1, opts=pkg.default_opts(reindex_by_degree=reindex))
    roots = g.sample_roots(16, 1, 16)
    p = torch.empty(g.n, dtype=torch.int32, device='cuda'); d = torch.empty_like(p)
    for loop in ("persistent", "graph", "host"):
        g.set_policy(mode=0, alpha=30, beta=1000, loop=loop)
        for r in roots: pkg.bfs_run(g.h, int(r), p, d)
        tot = ini = comp = 0
        for r in roots:
            pkg.bfs_run(g.h, int(r), p, d)
            run, lv = g.stats(tuples=False)
            tot += run['ms_total']; ini += run['ms_init']; comp += run['ms_compute']
        k = len(roots)
        print(f"reindex={reindex} {loop:10s} total {tot/k*1000:7.1f} us  init {ini/k*1000:6.1f}  loop {comp/k*1000:6.1f}  rest {(tot-ini-comp)/k*1000:6.1f}")
    g.close()
