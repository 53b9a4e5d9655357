"""Full-size parity, in the launch configuration bench.py times (BASELINE.json
configs K26 and K29: Kronecker, edgefactor 16, section 3.4 degree reindex with
rows by decreasing neighbour degree, alpha 30 / beta 24).

The serial oracle cannot build these graphs in test time, so the checks use what
it CAN compute one by one plus properties that hold at any size:
  * generator: sampled edge ranges, oracle Philox generator vs the GPU, bit-exact;
  * CSR (internal labels; the label map is checked to be a permutation that
    orders vertices by non-increasing degree): every sampled oracle edge {u, v}
    is present in the GPU row of its lower-degree endpoint (self-loops dropped),
    sampled rows are duplicate-free and in the degree order;
  * BFS: V1 and V5 on every vertex, V3 (depth[parent] = depth - 1) on every
    reached vertex, V2 (tree edge exists) on sampled vertices against the checked
    rows, V4 (no edge spans more than one level) on sampled oracle edges, and the
    per-step discovered counts equal the depth histogram.
By the validator theorem V1-V5 imply exact depths.
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pkg = pytest.importorskip("paper_1503_04359_b200")
from paper_1503_04359_b200 import build as pkg_build  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = {"k26": (26, 16, 1, oracle.KRON_ABC, 40e9), "k29": (29, 16, 1, oracle.KRON_ABC, 150e9)}


@pytest.fixture(scope="module", autouse=True)
def _dev():
    pkg_build.build()
    torch.cuda.set_device(0)


@pytest.mark.timeout(1500)
@pytest.mark.parametrize("name", sorted(CASES))
def test_fullscale_properties(name):
    scale, ef, seed, abc, need = CASES[name]
    if torch.cuda.mem_get_info()[0] < need:
        pytest.skip("not enough device memory")
    rng = np.random.default_rng(scale)
    M = ef << scale
    n = 1 << scale

    # generator: 16 random ranges of 4096 edges, bit-exact
    buf = torch.empty((4096, 2), dtype=torch.int32, device="cuda")
    samples = []
    for k, first in enumerate(rng.integers(0, M - 4096, 128)):
        want = oracle.kron_edges(scale, ef, seed, abc, first=int(first), count=4096)
        if k < 16:
            pkg.bfs_kronecker_edges(scale, ef, seed, abc, int(first), 4096, buf)
            assert np.array_equal(buf.cpu().numpy(), want)
        samples.append(want)
    edges = np.concatenate(samples)   # 512K oracle edges for the V4 check

    g = pkg.Graph.kronecker(scale, ef, seed, abc, opts=pkg.default_opts(reindex_by_degree=True))
    g.set_policy(mode=0, alpha=30, beta=1000)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    pkg.bfs_graph_export_labels(g.h, lab)
    label = lab.cpu().numpy()
    del lab
    assert np.array_equal(np.sort(label), np.arange(n, dtype=np.int32))       # a permutation

    def row(v):  # row of ORIGINAL vertex v, as original labels
        return ilabel[pkg.bfs_graph_export_row(g.h, int(label[v]), cap=1 << 24)]

    ilabel = np.empty(n, np.int32)
    ilabel[label] = np.arange(n, dtype=np.int32)

    # CSR: sampled edges present in the row of the lower-degree endpoint
    deg_cache = {}

    def deg(v):
        if v not in deg_cache:
            deg_cache[v] = len(row(v))
        return deg_cache[v]

    checked_rows = {}
    for u, v in edges[rng.choice(len(edges), 400, replace=False)]:
        if u == v:
            continue
        a, b = (u, v) if deg(u) <= deg(v) else (v, u)
        r = checked_rows.setdefault(int(a), row(a))
        assert b in r, (a, b)
    for a, r in checked_rows.items():
        assert len(np.unique(r)) == len(r) and a not in r                    # dedup, no self-loops
        d = np.array([deg(int(x)) for x in r[:64]])
        assert np.all(d[:-1] >= d[1:])                                         # decreasing degree
        assert np.all(np.diff(label[r]) > 0)                                   # ties by (internal) ID
    # internal order = degree order on sampled vertices
    smp = np.sort(rng.choice(n, 200, replace=False))
    ds = np.array([deg(int(ilabel[x])) for x in smp])
    assert np.all(ds[:-1] >= ds[1:])

    roots = g.sample_roots(scale, seed, 2)
    depth_h = torch.empty(n, dtype=torch.int32).pin_memory()
    parent_h = torch.empty(n, dtype=torch.int32).pin_memory()
    for r in roots:
        r = int(r)
        pkg.bfs_run(g.h, r, parent_h, depth_h)
        run, levels = g.stats()
        d = depth_h.numpy()
        p = parent_h.numpy()
        # V1, V5
        assert d[r] == 0 and p[r] == r and int((d == 0).sum()) == 1
        assert np.array_equal(d < 0, p < 0) and d.min() >= -1
        reached = d >= 0
        assert run["reached"] == int(reached.sum())
        # V3 on every reached vertex
        vv = np.nonzero(reached)[0]
        vv = vv[vv != r]
        assert np.all(d[p[vv]] == d[vv] - 1)
        # per-step discovered counts = depth histogram
        hist = np.bincount(d[reached])
        assert [lv["discovered"] for lv in levels][:-1] == hist[1:].tolist()
        assert levels[0]["frontier"] == 1
        # V2 on sampled reached vertices (rows of low-degree vertices only)
        for v in rng.choice(vv, 300, replace=False):
            if deg(int(v)) <= 1 << 16:
                assert p[v] in row(v), v
        # V4 on sampled oracle edges
        a, b = edges[:, 0], edges[:, 1]
        ra, rb = d[a] >= 0, d[b] >= 0
        assert np.array_equal(ra, rb)
        assert np.all(np.abs(d[a][ra].astype(np.int64) - d[b][ra]) <= 1)
    g.close()
