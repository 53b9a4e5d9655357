"""Pins for the oracle CSR build and the section 3.4 reindex (oracle/oracle.c).

SPEC examples, Graph invariants
and scipy.sparse's independent CSR construction fix the expected values.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from tests import graphs


def test_spec_examples():
    g = oracle.build_csr(2, [[0, 1]])
    assert g.offsets.tolist() == [0, 1, 2] and g.adj.tolist() == [1, 0]
    n, uv = graphs.g1()
    g = oracle.build_csr(n, uv)
    assert g.offsets.tolist() == [0, 3, 4, 5, 7, 9, 10]
    assert g.degree(0) == 3 and g.degree(5) == 1
    g = oracle.build_csr(3, np.zeros((0, 2), np.int32))
    assert g.offsets.tolist() == [0, 0, 0, 0] and g.arcs == 0 and g.degree(1) == 0


def test_encounter_order_and_self_loop_doubling():
    # rows in encounter order; a self-loop contributes two identical arcs
    g = oracle.build_csr(3, [[2, 0], [1, 1], [0, 1]])
    assert g.row(0).tolist() == [2, 1]
    assert g.row(1).tolist() == [1, 1, 0]
    assert g.row(2).tolist() == [0]


def test_malformed_input_names_tuple():
    with pytest.raises(oracle.MalformedInput, match=r"tuple 1 = \(2, 5\)"):
        oracle.build_csr(5, [[0, 1], [2, 5]])


def _row_multisets(g):
    return [sorted(g.row(v).tolist()) for v in range(g.n)]


@pytest.mark.parametrize("seed", range(6))
def test_invariants_random(seed):
    n, uv = graphs.random_edges(40, 150, seed)
    g = oracle.build_csr(n, uv)
    off = g.offsets
    assert off[0] == 0 and np.all(np.diff(off) >= 0) and off[-1] == g.adj.size
    assert g.adj.min() >= 0 and g.adj.max() < n
    assert g.degree().sum() == 2 * uv.shape[0]
    A = np.zeros((n, n), np.int64)
    for v in range(n):
        for x in g.row(v):
            A[v, x] += 1
    assert np.array_equal(A, A.T)
    # S:65 round trip: each tuple {u,v} (u != v) appears once as u->v and once as v->u
    M = np.zeros((n, n), np.int64)
    for u, v in uv:
        M[u, v] += 1
        M[v, u] += 1
    assert np.array_equal(A, M)


@pytest.mark.parametrize("seed", range(4))
def test_matches_scipy_sparse(seed):
    n, uv = graphs.skewed_edges(300, 3000, seed)
    rows = np.concatenate([uv[:, 0], uv[:, 1]])
    cols = np.concatenate([uv[:, 1], uv[:, 0]])
    S = sp.coo_matrix((np.ones(rows.size, np.int64), (rows, cols)), shape=(n, n)).tocsr()
    S.sum_duplicates()
    S.sort_indices()
    # multigraph: row multisets == scipy's summed counts expanded
    g = oracle.build_csr(n, uv, sort_rows=True)
    for v in range(n):
        lo, hi = S.indptr[v], S.indptr[v + 1]
        want = np.repeat(S.indices[lo:hi], S.data[lo:hi]).tolist()
        assert g.row(v).tolist() == want
    # dedup + drop self-loops: rows == scipy's distinct off-diagonal pattern
    gd = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    S.setdiag(0)
    S.eliminate_zeros()
    assert gd.offsets.tolist() == S.indptr.tolist()
    assert gd.adj.tolist() == S.indices.tolist()


def test_dedup_without_sort_keeps_first_occurrence():
    g = oracle.build_csr(4, [[0, 3], [0, 1], [0, 3], [2, 2]], dedup=True, drop_self_loops=True)
    assert g.row(0).tolist() == [3, 1]
    assert g.row(2).tolist() == []
    assert g.row(3).tolist() == [0]


def test_reindex_spec_examples():
    n, uv = graphs.g1()
    g = oracle.build_csr(n, uv, sort_rows=True)
    new, pos = oracle.degree_reindex(g, 1)
    # degrees 3,1,1,2,2,1 -> order (deg desc, id asc) = 0,3,4,1,2,5 (S:183 ties keep ID order)
    assert pos.tolist() == [0, 3, 4, 1, 2, 5]
    assert new.tolist() == pos.tolist()
    r = oracle.relabel_csr(g, new, pos)
    # vertex 4's list {3,5} -> [3, 5] (degrees 2 > 1), in new labels [1, 5]
    assert r.row(new[4]).tolist() == [new[3], new[5]]
    assert r.row(new[1]).tolist() == [new[0]]                  # S:193 singleton


def test_reindex_round_robin_partitions():
    n, uv = graphs.skewed_edges(64, 400, 1)
    g = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    new, pos = oracle.degree_reindex(g, 4)
    assert sorted(new.tolist()) == list(range(n))
    deg = g.degree()
    # partition of position k is k % 4; inside a partition degree is non-increasing in local ID
    for part in range(4):
        members = sorted((int(new[v]), int(deg[v])) for v in range(n) if new[v] // 16 == part)
        assert all(members[i][1] >= members[i + 1][1] for i in range(len(members) - 1))
        assert {int(pos[v]) % 4 for v in range(n) if new[v] // 16 == part} == {part}


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("seed", range(2))
def test_reindex_partition_local(p, seed):
    """P:158 'after partitioning ... permutation of local IDs': pinned by the properties that
    determine the labelling uniquely -- a permutation that keeps every vertex in its block,
    with degree non-increasing and, among equal degrees, original ID increasing in the new
    label inside each block -- and by p = 1 being the global reindex."""
    n, uv = graphs.skewed_edges(128, 900, seed)
    g = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    new, pos = oracle.degree_reindex_local(g, p)
    per = n // p
    deg = g.degree()
    assert sorted(new.tolist()) == list(range(n))
    assert np.array_equal(new // per, np.arange(n) // per)               # ownership preserved
    for b in range(p):
        members = sorted((int(new[v]), -int(deg[v]), v) for v in range(b * per, (b + 1) * per))
        keys = [(m[1], m[2]) for m in members]                             # in new-label order
        assert keys == sorted(keys)                                        # degree desc, then ID asc
    gnew, gpos = oracle.degree_reindex(g, 1)
    assert np.array_equal(pos, gpos)                                       # rows: global degree order
    if p == 1:
        assert np.array_equal(new, gnew)
    r = oracle.relabel_csr(g, new, pos)
    rdeg = r.degree()
    assert np.array_equal(rdeg[new], deg)
    for root in (0, int(np.argmax(deg))):                                  # S:200 levels unchanged
        assert np.array_equal(oracle.bfs(r, int(new[root]))[0][new], oracle.bfs(g, root)[0])


@pytest.mark.parametrize("seed", range(3))
def test_relabel_preserves_structure(seed):
    n, uv = graphs.skewed_edges(200, 1500, seed)
    g = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    new, pos = oracle.degree_reindex(g, 1)
    r = oracle.relabel_csr(g, new, pos)
    deg = g.degree()
    rdeg = r.degree()
    assert np.array_equal(rdeg[new], deg)                   # S:185 degree sequence invariant
    for v in range(n):                                      # rows sorted by neighbour degree desc
        row = r.row(v)
        assert all(rdeg[row[i]] >= rdeg[row[i + 1]] for i in range(len(row) - 1))
    # S:200 BFS levels identical before and after relabeling
    for root in (0, 7, 123):
        d0, _ = oracle.bfs(g, root)
        d1, _ = oracle.bfs(r, int(new[root]))
        assert np.array_equal(d1[new], d0)


def test_sort_rows_by_degree_spec():
    n, uv = graphs.g1()
    g = oracle.sort_rows_by_degree(oracle.build_csr(n, uv, sort_rows=True))
    assert g.row(4).tolist() == [3, 5]        # degrees 2 > 1
    assert g.row(1).tolist() == [0]           # S:193 singleton
    assert g.row(0).tolist() == [3, 1, 2]     # degree 2 first, then the degree-1 tie by ID


@pytest.mark.parametrize("seed", range(3))
def test_sort_rows_by_degree_properties(seed):
    n, uv = graphs.skewed_edges(300, 2500, seed)
    base = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    g = oracle.sort_rows_by_degree(base)
    deg = base.degree()
    for v in range(n):
        row = g.row(v).tolist()
        assert sorted(row) == base.row(v).tolist()                          # multiset unchanged
        keys = [(-deg[x], x) for x in row]
        assert keys == sorted(keys)                                          # S:194 + ID tie-break
    for root in (0, int(np.argmax(deg))):                                    # S:200 levels unchanged
        assert np.array_equal(oracle.bfs(g, root)[0], oracle.bfs(base, root)[0])
