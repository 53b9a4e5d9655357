"""Pins for the direction-optimized BFS emulator (oracle/oracle.c orc_do_emulate).

The emulator derives counters, directions, inspections and bottom-up parents
from the oracle depth.  Pinned by (i) the hand trace of G1 in
tests/golden/g1_do_trace.txt and (ii) a literal, independent step-by-step
simulation of Algorithm 1 written here with Python sets, whose live
counters must agree exactly with the emulator's derived ones.
"""
import numpy as np
import pytest

import oracle
from tests import graphs


def test_g1_hand_trace():
    want = graphs.load_golden_table("g1_do_trace.txt")
    n, uv = graphs.g1()
    g = oracle.build_csr(n, uv, sort_rows=True)
    d, _ = oracle.bfs(g, 0)
    td = oracle.do_emulate(g, d, policy=1)
    assert td["n_f"].tolist() == want["n_f"]
    assert td["m_f"].tolist() == want["m_f"]
    assert td["m_u"].tolist() == want["m_u"]
    assert td["insp"].tolist() == want["td_insp"] and td["insp"].sum() == 10
    assert td["dir"].tolist() == [0, 0, 0, 0]
    auto = oracle.do_emulate(g, d, alpha=15, beta=18, policy=0, want_bu_parent=True)
    assert auto["dir"].tolist() == want["auto_dir"]
    assert auto["insp"].tolist() == want["auto_insp"]
    bp = auto["bu_parent"].copy()
    bp[0] = 0
    assert bp.tolist() == want["auto_parent"]


def simulate_alg1(g, root, alpha, beta, policy, bu_from=0, coord_hi=None):
    """Algorithm 1 on one partition, literally, with Python sets.
    Returns per-step lists and the parent array; the direction rule is applied
    to counters measured live on the simulated frontier.  Policy 3 is the paper's
    section 3.3 rule: the coordinator (vertices < coord_hi) compares
    its own frontier degree sum with a static fraction alpha/10000 of all arcs;
    after beta bottom-up steps the search returns top-down for good."""
    n = g.n
    adj = [g.row(v).tolist() for v in range(n)]
    deg = [len(a) for a in adj]
    arcs = sum(deg)
    visited = {root}
    parent = [-1] * n
    parent[root] = root
    frontier = {root}
    mode = 0
    seen_deg = 0
    prev_nf = None
    coord_hi = n if coord_hi is None else coord_hi
    bu_steps, returned = 0, False
    out = {k: [] for k in ("dir", "n_f", "m_f", "m_u", "discovered", "insp")}
    d = 0
    while True:
        n_f = len(frontier)
        m_f = sum(deg[v] for v in frontier)
        seen_deg += m_f
        m_u = arcs - seen_deg
        if policy == 1:
            mode = 0
        elif policy == 2:
            mode = 1 if d >= bu_from else 0
        elif policy == 3:
            if mode == 0:
                coord = sum(deg[v] for v in frontier if v < coord_hi)
                if not returned and coord * 10000 >= alpha * arcs:
                    mode = 1
            elif bu_steps >= beta:
                mode, returned = 0, True
            if mode == 1:
                bu_steps += 1
        else:
            if mode == 0:
                if m_f * alpha > m_u:
                    mode = 1
            else:
                if n_f * beta < n and n_f < prev_nf:
                    mode = 0
        nxt = set()
        insp = 0
        if mode == 0:                                   # TOP-DOWN
            for vtx in sorted(frontier):
                for nbr in adj[vtx]:
                    insp += 1
                    if nbr not in visited:
                        nxt.add(nbr)
                        parent[nbr] = vtx
                        visited.add(nbr)
        else:                                           # BOTTOM-UP
            for vtx in range(n):
                if vtx not in visited:
                    for nbr in adj[vtx]:
                        insp += 1
                        if nbr in frontier:             # DESIGN.md R1
                            nxt.add(vtx)
                            parent[vtx] = nbr
                            break
            visited |= nxt
        for k, val in (("dir", mode), ("n_f", n_f), ("m_f", m_f), ("m_u", m_u),
                       ("discovered", len(nxt)), ("insp", insp)):
            out[k].append(val)
        prev_nf = n_f
        frontier = nxt
        d += 1
        if not frontier:
            break
    return out, parent


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("policy,alpha,beta,bu_from", [(0, 15, 18, 0), (0, 2, 4, 0), (1, 15, 18, 0),
                                                       (2, 15, 18, 1), (2, 15, 18, 0), (0, 100, 2, 0),
                                                       (3, 500, 3, 0), (3, 50, 1, 0), (3, 2000, 2, 0)])
@pytest.mark.parametrize("coord_frac", [1.0, 0.5])
def test_emulator_equals_literal_simulation(seed, policy, alpha, beta, bu_from, coord_frac):
    if coord_frac != 1.0 and policy != 3:
        pytest.skip("coordinator share only matters for policy 3")
    n, uv = graphs.skewed_edges(300, 1200, seed)
    g = oracle.build_csr(n, uv, dedup=seed % 2 == 0, drop_self_loops=seed % 2 == 0, sort_rows=True)
    roots = [int(np.argmax(g.degree())), int(np.nonzero(g.degree())[0][seed])]
    coord_hi = int(n * coord_frac)
    for root in roots:
        depth, _ = oracle.bfs(g, root)
        sim, sim_parent = simulate_alg1(g, root, alpha, beta, policy, bu_from, coord_hi)
        emu = oracle.do_emulate(g, depth, alpha, beta, policy, bu_from, want_bu_parent=True, coord_hi=coord_hi)
        for k in ("dir", "n_f", "m_f", "m_u", "discovered", "insp"):
            assert emu[k].tolist() == sim[k], (k, root)
        # bottom-up parents are the first frontier neighbour in stored order
        for v in range(n):
            if emu["bu_parent"][v] >= 0:
                assert sim_parent[v] == emu["bu_parent"][v]


def test_invariants_kronecker():
    uv, g = oracle.kron_graph(12, 16, 2)
    for root in oracle.sample_roots(g, 12, 2, 4):
        depth, _ = oracle.bfs(g, int(root))
        e = oracle.do_emulate(g, depth)
        assert e["n_f"].sum() == (depth >= 0).sum()                       # S:313 frontier conservation
        assert e["discovered"][-1] == 0 and np.all(e["discovered"][:-1] > 0)
        td = oracle.do_emulate(g, depth, policy=1)
        assert np.array_equal(td["insp"], td["m_f"])
        assert e["insp"].sum() <= td["insp"].sum()                        # DO explores fewer edges


def test_isolated_root_single_step():
    g = oracle.build_csr(4, [[0, 1]])
    d, _ = oracle.bfs(g, 3)
    e = oracle.do_emulate(g, d)
    assert e["n_f"].tolist() == [1] and e["discovered"].tolist() == [0] and e["insp"].tolist() == [0]


def test_paper_rule_hand_trace_g1():
    """Policy 3 on SPEC G1 from root 0, traced by hand: arcs = 10 and
    m_f = 3/4/2/1 at d = 0..3 (tests/golden/g1_do_trace.txt).  TD -> BU iff
    m_fc * 10000 >= alpha * arcs; S:297's threshold example (degree sum 1 -> TD,
    5 -> BU at 10 arcs) holds for a fraction of 0.5, i.e. alpha = 5000 (R23)."""
    g = oracle.build_csr(6, [[0, 1], [0, 2], [0, 3], [3, 4], [4, 5]], sort_rows=True)
    d, _ = oracle.bfs(g, 0)
    dirs = lambda **kw: oracle.do_emulate(g, d, policy=3, **kw)["dir"].tolist()  # noqa: E731
    assert dirs(alpha=3000, beta=2) == [1, 1, 0, 0]     # 3e4 >= 3e4: BU at once, 2 BU steps
    assert dirs(alpha=3001, beta=1) == [0, 1, 0, 0]     # 3e4 < 30010; 4e4 >= 30010; 1 BU step
    assert dirs(alpha=500, beta=3) == [1, 1, 1, 0]      # SPEC default 0.05, 3 steps
    assert dirs(alpha=500, beta=9) == [1, 1, 1, 1]      # the search ends first
    assert dirs(alpha=3001, beta=1, coord_hi=1) == [0, 0, 0, 0]   # coordinator owns only vertex 0
    assert dirs(alpha=5001, beta=1, coord_hi=1) == [0, 0, 0, 0]
    # S:297 threshold arithmetic with a 1-arc-sum vs 5-arc-sum frontier at 10 arcs, fraction 0.5
    assert not (1 * 10000 >= 5000 * 10) and (5 * 10000 >= 5000 * 10)
    # never re-enters BU after returning: a path graph has tiny frontiers
    path = oracle.build_csr(8, [[i, i + 1] for i in range(7)], sort_rows=True)
    dp, _ = oracle.bfs(path, 0)
    pd = oracle.do_emulate(path, dp, policy=3, alpha=1, beta=2)["dir"].tolist()
    assert pd == [1, 1] + [0] * (len(pd) - 2)
