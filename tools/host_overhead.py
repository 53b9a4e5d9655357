"""Host-side cost of one bfs_run on a small graph: wall time of the call vs the
library's device time (ms_total), and the event-bracketed time bench.py measures."""
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1503_04359_b200 as pkg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(scale, 16, 1, opts=pkg.default_opts(reindex_by_degree=True))
roots = g.sample_roots(scale, 1, 64)
p = torch.empty(g.n, dtype=torch.int32, device='cuda')
d = torch.empty_like(p)
s = g.stream
for lt in (True, False):
    g.set_policy(mode=0, alpha=30, beta=1000, level_times=lt)
    for r in roots:
        pkg.bfs_run(g.h, int(r), p, d, check=False)
    wall = dev = ev = 0.0
    for r in roots:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        pkg.bfs_run(g.h, int(r), p, d, check=False)
        t1 = time.perf_counter()
        e1.record(s)
        e1.synchronize()
        run, _ = g.stats(tuples=False)
        wall += (t1 - t0) * 1e6
        dev += run["ms_total"] * 1e3
        ev += e0.elapsed_time(e1) * 1e3
    k = len(roots)
    print(f"level_times={lt}: host wall {wall / k:.1f} us, device ms_total {dev / k:.1f} us, events {ev / k:.1f} us")
t0 = time.perf_counter()
for _ in range(1000):
    pkg.lib().bfs_abi_version()
print(f"empty ctypes call {(time.perf_counter() - t0) * 1e3:.2f} us")
