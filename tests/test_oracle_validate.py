"""Pins for the oracle validator (oracle/oracle.c orc_validate).

Correct outputs must pass; each class of injected corruption must
be rejected by the rule that defines it; an alternative valid BFS tree built
independently in the test must pass V1-V5.
"""
import numpy as np
import pytest

import oracle
from tests import graphs


def _g1():
    n, uv = graphs.g1()
    g = oracle.build_csr(n, uv)
    d, p = oracle.bfs(g, 0)
    return g, d, p


def test_correct_output_passes():
    g, d, p = _g1()
    assert oracle.validate(g, 0, d, p, ref_depth=d) == {}


def test_spec_mutation_parent_altered():
    # parents[4] altered to 5 -> levels[5]=3 != levels[4]-1 = 1 (rule 3); 5-4 is an edge
    g, d, p = _g1()
    p = p.copy()
    p[4] = 5
    bad = oracle.validate(g, 0, d, p, ref_depth=d)
    assert "V3_parent_depth" in bad and bad["V3_parent_depth"][1] == 4
    assert "V2_tree_edge" not in bad


def test_spec_mutation_false_unreached():
    # vertex 5 marked unreached -> fails against the oracle / edge-span rule
    g, d, p = _g1()
    d, p = d.copy(), p.copy()
    d[5] = -1
    p[5] = -1
    bad = oracle.validate(g, 0, d, p, ref_depth=oracle.bfs(g, 0)[0])
    assert "V6_exact_depth" in bad and "V4_edge_span" in bad


def test_mutation_non_edge_parent():
    g, d, p = _g1()
    p = p.copy()
    p[5] = 3            # depth[3] = 1 but depth[5] = 3 and 3-5 is not an edge
    bad = oracle.validate(g, 0, d, p)
    assert "V2_tree_edge" in bad and "V3_parent_depth" in bad


def test_mutation_wrong_depth_consistent_tree():
    # shift a whole subtree one level deeper: parent chain consistent only if edges span > 1
    n, uv = graphs.cycle(6)
    g = oracle.build_csr(n, uv)
    d, p = oracle.bfs(g, 0)
    d2 = d.copy()
    d2[3] = 4
    bad = oracle.validate(g, 0, d2, p, ref_depth=d)
    assert "V3_parent_depth" in bad and "V6_exact_depth" in bad


def test_mutation_false_reached_and_root():
    n, uv = graphs.disjoint_union(graphs.path(3), graphs.path(2))
    g = oracle.build_csr(n, uv)
    d, p = oracle.bfs(g, 0)
    d2, p2 = d.copy(), p.copy()
    d2[3], p2[3] = 1, 0          # claims a vertex of the other component
    bad = oracle.validate(g, 0, d2, p2)
    assert "V2_tree_edge" in bad and "V4_edge_span" in bad
    d3, p3 = d.copy(), p.copy()
    p3[0] = 1
    assert "V1_root" in oracle.validate(g, 0, d3, p3)
    d4, p4 = d.copy(), p.copy()
    p4[4] = 3                    # parent set but depth unreached
    assert "V5_unreached" in oracle.validate(g, 0, d4, p4)


@pytest.mark.parametrize("seed", range(5))
def test_alternative_valid_tree_passes(seed):
    """Any neighbour one level up is a valid parent: pick the LAST such neighbour
    (the FIFO oracle picks the first discovered) and the validator must accept it."""
    n, uv = graphs.skewed_edges(400, 2500, seed)
    g = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    root = int(np.argmax(g.degree()))
    d, p = oracle.bfs(g, root)
    alt = p.copy()
    for v in range(n):
        if d[v] > 0:
            cands = [x for x in g.row(v).tolist() if d[x] == d[v] - 1]
            alt[v] = cands[-1]
    assert oracle.validate(g, root, d, alt, ref_depth=d) == {}
