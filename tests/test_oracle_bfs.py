"""Pins for the serial oracle BFS (oracle/oracle.c orc_bfs).

Depth is the hop distance from the root, a quantity with independent
definitions: brute force over every labelled graph on up to 6 vertices
(Floyd-Warshall by boolean matrix powers), closed forms on structured graphs,
the SPEC's G1 examples, and scipy's unweighted shortest paths.
"""
import itertools

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.csgraph as csg

import oracle
from tests import graphs


def _check_tree(g, root, depth, parent):
    assert depth[root] == 0 and parent[root] == root
    for v in range(g.n):
        if depth[v] < 0:
            assert parent[v] == -1
        elif v != root:
            assert parent[v] in g.row(v).tolist()
            assert depth[parent[v]] == depth[v] - 1


def _all_pairs_hops(adjm: np.ndarray) -> np.ndarray:
    """Floyd-Warshall over a stack of boolean adjacency matrices [G, n, n]."""
    G, n, _ = adjm.shape
    INF = 10 ** 6
    d = np.where(adjm, 1, INF).astype(np.int64)
    idx = np.arange(n)
    d[:, idx, idx] = 0
    for k in range(n):
        d = np.minimum(d, d[:, :, k:k + 1] + d[:, k:k + 1, :])
    d[d >= INF] = -1
    return d


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_brute_force_all_small_graphs(n):
    pairs = list(itertools.combinations(range(n), 2))
    G = 1 << len(pairs)
    masks = np.arange(G)
    adjm = np.zeros((G, n, n), bool)
    for k, (a, b) in enumerate(pairs):
        bit = ((masks >> k) & 1).astype(bool)
        adjm[:, a, b] = bit
        adjm[:, b, a] = bit
    dist = _all_pairs_hops(adjm)
    for gi in range(G):
        uv = np.array([p for k, p in enumerate(pairs) if (gi >> k) & 1], np.int32).reshape(-1, 2)
        g = oracle.build_csr(n, uv)
        for root in range(n):
            depth, parent = oracle.bfs(g, root)
            assert depth.tolist() == dist[gi, root].tolist(), (gi, root)
            if n <= 4 or root == 0:
                _check_tree(g, root, depth, parent)


def test_spec_g1():
    n, uv = graphs.g1()
    g = oracle.build_csr(n, uv)
    d, p = oracle.bfs(g, 0)
    assert d.tolist() == [0, 1, 1, 1, 2, 3]
    assert p.tolist() == [0, 0, 0, 0, 3, 4]
    d, p = oracle.bfs(g, 5)
    assert d.tolist() == [3, 4, 4, 2, 1, 0]
    _check_tree(g, 5, d, p)


def test_edgeless_and_isolated_root():
    g = oracle.build_csr(4, np.zeros((0, 2), np.int32))
    d, p = oracle.bfs(g, 2)
    assert d.tolist() == [-1, -1, 0, -1] and p.tolist() == [-1, -1, 2, -1]
    n, uv = graphs.path(5)
    g = oracle.build_csr(7, uv)                                  # vertices 5, 6 isolated
    d, p = oracle.bfs(g, 6)
    assert (d >= 0).sum() == 1 and d[6] == 0 and p[6] == 6


def test_root_out_of_range():
    g = oracle.build_csr(3, [[0, 1]])
    with pytest.raises(IndexError):
        oracle.bfs(g, 3)
    with pytest.raises(IndexError):
        oracle.bfs(g, -1)


def _depths(n_uv, root, **kw):
    n, uv = n_uv
    g = oracle.build_csr(n, uv, **kw)
    d, p = oracle.bfs(g, root)
    _check_tree(g, root, d, p)
    return d


@pytest.mark.parametrize("n,r", [(1, 0), (9, 0), (9, 4), (50, 17)])
def test_path(n, r):
    assert _depths(graphs.path(n), r).tolist() == [abs(i - r) for i in range(n)]


@pytest.mark.parametrize("n,r", [(3, 0), (8, 3), (51, 10)])
def test_cycle(n, r):
    want = [min(abs(i - r), n - abs(i - r)) for i in range(n)]
    assert _depths(graphs.cycle(n), r).tolist() == want


def test_star():
    n = 20
    assert _depths(graphs.star(n), 0).tolist() == [0] + [1] * (n - 1)
    want = [1] + [2] * (n - 1)
    want[5] = 0
    assert _depths(graphs.star(n), 5).tolist() == want


def test_clique_and_bipartite():
    assert _depths(graphs.clique(12), 4).tolist() == [1] * 4 + [0] + [1] * 7
    a, b = 4, 7
    d = _depths(graphs.complete_bipartite(a, b), 1)
    assert d.tolist() == [2, 0, 2, 2] + [1] * b
    d = _depths(graphs.complete_bipartite(a, b), a + 2)
    assert d.tolist() == [1] * a + [2, 2, 0, 2, 2, 2, 2]


@pytest.mark.parametrize("dim,r", [(1, 0), (4, 0), (7, 45)])
def test_hypercube(dim, r):
    n = 1 << dim
    assert _depths(graphs.hypercube(dim), r).tolist() == [bin(i ^ r).count("1") for i in range(n)]


def test_grid():
    R, C = 7, 11
    r0, c0 = 3, 2
    d = _depths(graphs.grid(R, C), r0 * C + c0)
    assert d.tolist() == [abs(i // C - r0) + abs(i % C - c0) for i in range(R * C)]


def test_heap_tree():
    n = 100
    d = _depths(graphs.heap_tree(n), 0)
    assert d.tolist() == [int(np.floor(np.log2(i + 1))) for i in range(n)]


def test_disjoint_union_unreached():
    n, uv = graphs.disjoint_union(graphs.path(6), graphs.cycle(5), graphs.star(4))
    d = _depths((n, uv), 7)
    assert d[:6].tolist() == [-1] * 6 and d[11:].tolist() == [-1] * 4
    assert d[6:11].tolist() == [1, 0, 1, 2, 2]


def test_self_loops_and_multi_edges_change_nothing():
    n, uv = graphs.grid(5, 6)
    extra = np.concatenate([uv, uv[::3], np.array([[v, v] for v in range(0, n, 4)], np.int32)])
    for r in (0, 13):
        base = _depths((n, uv), r)
        assert np.array_equal(_depths((n, extra), r), base)
        assert np.array_equal(_depths((n, extra), r, dedup=True, drop_self_loops=True, sort_rows=True), base)


def test_matches_scipy_on_kronecker_s14():
    uv, g = oracle.kron_graph(14, 16, 5)
    A = sp.csr_matrix((np.ones(g.arcs), g.adj, g.offsets), shape=(g.n, g.n))
    roots = oracle.sample_roots(g, 14, 5, 6)
    D = csg.shortest_path(A, unweighted=True, indices=roots, directed=False)
    for i, r in enumerate(roots):
        d, p = oracle.bfs(g, int(r))
        want = np.where(np.isinf(D[i]), -1, D[i]).astype(np.int64)
        assert np.array_equal(d.astype(np.int64), want)
        _check_tree(g, int(r), d, p)
