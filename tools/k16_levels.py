import sys, os
sys.path.insert(0, '.')
import torch, paper_1503_04359_b200 as pkg
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(16, 16, 1, opts=pkg.default_opts(reindex_by_degree=True))
roots = g.sample_roots(16, 1, 8)
p = torch.empty(g.n, dtype=torch.int32, device='cuda'); d = torch.empty_like(p)
for loop in ("cluster", "persistent"):
    g.set_policy(mode=0, alpha=30, beta=1000, loop=loop, level_times=True)
    for r in roots:
        pkg.bfs_run(g.h, int(r), p, d); pkg.bfs_run(g.h, int(r), p, d)
        run, lv = g.stats(tuples=False)
        print(loop, int(r), round(run["ms_total"]*1000,1), [("TB"[x["direction"]], x["frontier"], x["m_f"], x["inspections"], round(x["ms"]*1000,1)) for x in lv])
