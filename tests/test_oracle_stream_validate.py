"""Pins for the streaming Graph500 validator (oracle/oracle.c orc_stream_validate_*;
SURVEY section 8(c4)).

It is pinned against things other than itself:
  * the CSR validator orc_validate (itself pinned by the SPEC mutations in
    test_oracle_validate.py): the same set of failing rules on correct outputs, on the
    SPEC's mutations and on random corruptions;
  * the depth-exactness theorem it is used for (V1-V5 => depth = hop distance):
    random spanning trees pass V1, V2, V3 and V5 by construction, and the validator
    must accept exactly those whose depths are the BFS distances of the scipy
    breadth-first order;
  * the harness's range partition: several threads and chunk sizes give one verdict.
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

import oracle
from tests import graphs
from tests import stream_harness as H


def _stream_rules(n, uv, roots, depths, parents, chunk=1 << 22, threads=None):
    d8, pr = H.pack(depths, parents)
    res = H.validate(n, np.asarray(roots, np.int64), d8, pr, uv=uv, chunk=chunk, threads=threads)
    return [set(H.failing_rules(res, r)) for r in range(len(roots))]


def _csr_rules(n, uv, root, depth, parent):
    g = oracle.build_csr(n, uv)      # every tuple as two arcs: the same edge set
    return {k for k in oracle.validate(g, root, depth, parent) if k != "V6_exact_depth"}


def _kron(scale=10, seed=3):
    return 1 << scale, oracle.kron_edges(scale, 16, seed)


def test_correct_outputs_pass_many_roots():
    n, uv = _kron()
    g = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    roots = oracle.sample_roots(g, 10, 3, 16)
    outs = [oracle.bfs(g, int(r)) for r in roots]
    got = _stream_rules(n, uv, roots, [o[0] for o in outs], [o[1] for o in outs])
    assert got == [set()] * len(roots)


def test_isolated_root_and_disconnected_graph():
    n, uv = graphs.disjoint_union(graphs.path(4), graphs.star(5))
    n2 = n + 2                       # two isolated vertices
    g = oracle.build_csr(n2, uv)
    roots = [0, 5, n2 - 1]
    outs = [oracle.bfs(g, r) for r in roots]
    assert _stream_rules(n2, uv, roots, [o[0] for o in outs], [o[1] for o in outs]) == [set()] * 3


def test_spec_mutations_match_csr_validator():
    n, uv = graphs.g1()
    g = oracle.build_csr(n, uv)
    d, p = oracle.bfs(g, 0)
    p1 = p.copy()
    p1[4] = 5
    d2, p2 = d.copy(), p.copy()
    d2[5], p2[5] = -1, -1
    for dd, pp in ((d, p1), (d2, p2)):
        want = _csr_rules(n, uv, 0, dd, pp)
        assert want
        assert _stream_rules(n, uv, [0], [dd], [pp]) == [want]
    assert _stream_rules(n, uv, [0], [d], [p1]) == [{"V3_parent_depth"}]
    assert "V4_edge_span" in _stream_rules(n, uv, [0], [d2], [p2])[0]


@pytest.mark.parametrize("seed", range(6))
def test_random_corruptions_match_csr_validator(seed):
    """Each search gets one random corruption (or none); the failing rule sets of the
    two validators must agree search by search."""
    rng = np.random.default_rng(seed)
    n, uv = graphs.skewed_edges(300, 1500, seed)
    uv = np.concatenate([uv, np.array([[5, 5], [7, 7]], np.int32)])      # self-loops too
    g = oracle.build_csr(n, uv)
    roots = [int(x) for x in rng.choice(n, 12, replace=False)]
    depths, parents = [], []
    for r in roots:
        d, p = oracle.bfs(g, r)
        d, p = d.copy(), p.copy()
        v = int(rng.integers(n))
        kind = int(rng.integers(8))
        if kind == 1:
            p[v] = int(rng.integers(n))
        elif kind == 2:
            d[v] = int(rng.integers(-1, 6))
        elif kind == 3:
            d[v], p[v] = -1, -1
        elif kind == 4:
            p[r] = int(rng.integers(n))
        elif kind == 5:
            d[v] = 0
        elif kind == 6:
            p[v] = v
        elif kind == 7:
            d[v], p[v] = int(rng.integers(1, 4)), int(rng.integers(n))
        depths.append(d)
        parents.append(p)
    got = _stream_rules(n, uv, roots, depths, parents, chunk=257)
    want = [_csr_rules(n, uv, r, d, p) for r, d, p in zip(roots, depths, parents)]
    assert got == want


def _random_spanning_tree(n, adj, root, rng, fifo):
    """A random tree of the root's component with tree depths: random search order
    (not a BFS tree in general), or FIFO order with random neighbour choice (a BFS
    tree with random ties)."""
    depth = np.full(n, -1, np.int32)
    parent = np.full(n, -1, np.int32)
    depth[root], parent[root] = 0, root
    frontier = [root]
    while frontier:
        i = 0 if fifo else int(rng.integers(len(frontier)))
        u = frontier[i]
        nbrs = [v for v in adj[u] if depth[v] < 0]
        if not nbrs:
            frontier.pop(i)
            continue
        v = nbrs[int(rng.integers(len(nbrs)))]
        depth[v], parent[v] = depth[u] + 1, u
        frontier.append(v)
    return depth, parent


@pytest.mark.parametrize("seed", range(8))
def test_theorem_accepts_exactly_bfs_depths(seed):
    """V1-V5 => depth == hop distance: among random spanning trees (which
    satisfy V1, V2, V3, V5 by construction) the validator accepts a tree iff its depths
    equal scipy's unweighted shortest-path distances."""
    rng = np.random.default_rng(100 + seed)
    n = 12
    m = int(rng.integers(n, 3 * n))
    uv = rng.integers(0, n, size=(m, 2)).astype(np.int32)
    adj = [[] for _ in range(n)]
    for a, b in uv.tolist():
        adj[a].append(b)
        adj[b].append(a)
    A = sp.coo_matrix((np.ones(2 * m), (np.r_[uv[:, 0], uv[:, 1]], np.r_[uv[:, 1], uv[:, 0]])), shape=(n, n)).tocsr()
    dist = shortest_path(A, unweighted=True, directed=False)
    accepted = rejected = 0
    for t in range(40):
        root = int(rng.integers(n))
        d, p = _random_spanning_tree(n, adj, root, rng, fifo=t % 3 == 0)
        exact = np.where(np.isinf(dist[root]), -1, dist[root]).astype(np.int32)
        ok = _stream_rules(n, uv, [root], [d], [p]) == [set()]
        assert ok == bool(np.array_equal(d, exact)), (root, d, exact)
        accepted += ok
        rejected += not ok
    assert accepted and rejected      # both outcomes exercised


def test_thread_and_chunk_partition_do_not_change_the_verdict():
    n, uv = _kron(11, 5)
    g = oracle.build_csr(n, uv)
    roots = oracle.sample_roots(g, 11, 5, 4)
    outs = [oracle.bfs(g, int(r)) for r in roots]
    depths = [o[0].copy() for o in outs]
    parents = [o[1].copy() for o in outs]
    parents[1][int(np.flatnonzero(depths[1] > 1)[0])] = int(roots[1])   # V2/V3 for search 1
    depths[3][int(np.flatnonzero(depths[3] > 0)[-1])] += 2                # V3/V4 for search 3
    d8, pr = H.pack(depths, parents)
    ref = H.validate(n, roots, d8, pr, uv=uv, chunk=uv.shape[0], threads=1)
    for threads, chunk in ((2, 1000), (8, 4097), (3, 1 << 20)):
        res = H.validate(n, roots, d8, pr, uv=uv, chunk=chunk, threads=threads)
        assert np.array_equal(res["fails"], ref["fails"]) and np.array_equal(res["first"], ref["first"])
    gen = H.validate(n, roots, d8, pr, gen=(11, 16, 5, oracle.KRON_ABC), chunk=3001)
    assert np.array_equal(gen["fails"], ref["fails"]) and np.array_equal(gen["first"], ref["first"])
    assert ref["fails"][0].sum() == 0 and ref["fails"][2].sum() == 0
    assert ref["fails"][1].sum() > 0 and ref["fails"][3].sum() > 0


def test_parallel_generation_equals_serial():
    uv = H.generate_edges(12, 16, 9, oracle.KRON_ABC, threads=4, chunk=999)
    assert np.array_equal(uv, oracle.kron_edges(12, 16, 9))
