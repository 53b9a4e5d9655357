"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element, on the same seeded inputs.

Bars: generator tuples, CSR offsets/adjacency, depth,
roots, counters and inspection counts are bit-exact; parents may differ from
the oracle's FIFO tree and must pass the Graph500 validator, except for
vertices discovered by bottom-up steps, whose parent is unique (first frontier
neighbour in row order) and must equal the emulator's.
"""
import numpy as np
import pytest

import oracle
from tests import graphs

torch = pytest.importorskip("torch")
pkg = pytest.importorskip("paper_1503_04359_b200")
from paper_1503_04359_b200 import build as pkg_build  # noqa: E402

pytestmark = pytest.mark.gpu

POLICIES = [dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=1), dict(mode=2, bu_from_level=0),
            dict(mode=0, alpha=2, beta=4), dict(mode=0, alpha=100, beta=2),
            dict(mode=3, alpha=500, beta=3), dict(mode=3, alpha=50, beta=1),
            # every level loop (auto picks the persistent kernel for these small graphs)
            dict(mode=0, loop="host"), dict(mode=3, alpha=500, beta=3, loop="host"),
            dict(mode=0, loop="graph"), dict(mode=2, bu_from_level=1, loop="graph"),
            dict(mode=3, alpha=500, beta=3, loop="graph"), dict(mode=1, loop="graph"),
            dict(mode=0, loop="cluster"), dict(mode=2, bu_from_level=1, loop="cluster"),
            dict(mode=3, alpha=500, beta=3, loop="cluster")]


@pytest.fixture(scope="module", autouse=True)
def _dev():
    pkg_build.build()
    torch.cuda.set_device(0)


def _gpu_csr(g):
    off, adj = g.export_csr()
    return off.cpu().numpy(), adj.cpu().numpy()


def _check_run(g, ref, root, policy, uv=None):
    g.set_policy(**policy)
    parent, depth = g.run(int(root))
    d = depth.cpu().numpy()
    p = parent.cpu().numpy()
    want, _ = oracle.bfs(ref, int(root))
    assert np.array_equal(d, want), f"depth mismatch root={root} policy={policy}: " \
                                    f"{np.nonzero(d != want)[0][:10]}"
    bad = oracle.validate(ref, int(root), d, p, ref_depth=want)
    assert not bad, bad
    emu = oracle.do_emulate(ref, want, alpha=policy.get("alpha", 15), beta=policy.get("beta", 18),
                            policy=policy.get("mode", 0), bu_from=policy.get("bu_from_level", 0),
                            want_bu_parent=True)
    run, levels = g.stats()
    assert run["levels"] == len(emu["insp"])
    for key, lk in (("dir", "direction"), ("n_f", "frontier"), ("discovered", "discovered"), ("m_f", "m_f"),
                    ("m_u", "m_u"), ("insp", "inspections")):
        assert [lv[lk] for lv in levels] == emu[key].tolist(), (key, root, policy)
    bu = emu["bu_parent"] >= 0
    assert np.array_equal(p[bu], emu["bu_parent"][bu]), "bottom-up parent is not the first frontier neighbour"
    assert run["reached"] == int((want >= 0).sum())
    if uv is not None:
        assert run["component_edge_tuples"] == oracle.component_tuples(uv, want)
    return run, levels


# ------------------------------------------------------------------ generator
@pytest.mark.parametrize("scale,ef,seed,abc", [(1, 1, 42, oracle.KRON_ABC), (10, 16, 7, oracle.KRON_ABC),
                                               (16, 16, 1, oracle.KRON_ABC), (13, 8, 3, oracle.ER_ABC),
                                               (20, 1, 5, oracle.KRON_ABC)])
def test_generator_bit_exact(scale, ef, seed, abc):
    m = ef << scale
    uv = torch.empty((m, 2), dtype=torch.int32, device="cuda")
    pkg.bfs_kronecker_edges(scale, ef, seed, abc, 0, m, uv)
    want = oracle.kron_edges(scale, ef, seed, abc)
    assert np.array_equal(uv.cpu().numpy(), want)


def test_generator_range_offsets():
    scale, ef, seed = 12, 16, 9
    uv = torch.empty((777, 2), dtype=torch.int32, device="cuda")
    pkg.bfs_kronecker_edges(scale, ef, seed, oracle.KRON_ABC, 5000, 777, uv)
    assert np.array_equal(uv.cpu().numpy(), oracle.kron_edges(scale, ef, seed, first=5000, count=777))


# ------------------------------------------------------------------ CSR
@pytest.mark.parametrize("dedup,loops,sort", [(1, 1, 1), (0, 0, 1), (1, 0, 1), (0, 1, 1)])
def test_csr_kronecker_bit_exact(dedup, loops, sort):
    scale = 14
    opts = pkg.default_opts(dedup, loops, False, sort)
    g = pkg.Graph.kronecker(scale, 16, 3, opts=opts)
    off, adj = _gpu_csr(g)
    uv = oracle.kron_edges(scale, 16, 3)
    ref = oracle.build_csr(1 << scale, uv, dedup=bool(dedup), drop_self_loops=bool(loops), sort_rows=True)
    assert np.array_equal(off, ref.offsets)
    assert np.array_equal(adj, ref.adj)
    g.close()


def test_csr_unsorted_row_multisets():
    n, uv = graphs.skewed_edges(5000, 60000, 2)
    g = pkg.Graph.from_edges(torch.from_numpy(uv), n, opts=pkg.default_opts(False, False, False, False))
    off, adj = _gpu_csr(g)
    ref = oracle.build_csr(n, uv, sort_rows=True)
    assert np.array_equal(off, ref.offsets)
    for v in range(0, n, 7):
        assert sorted(adj[off[v]:off[v + 1]].tolist()) == ref.row(v).tolist()
    g.close()


def test_csr_big_rows_merge_path():
    """rows longer than the 32768-element shared-memory sort go through the merge passes"""
    rng = np.random.default_rng(11)
    n = 1 << 20
    hub_edges = np.stack([np.zeros(200000, np.int64), rng.integers(0, n, 200000)], 1)
    hub2 = np.stack([np.full(70000, 5), rng.integers(0, n, 70000)], 1)
    rest = rng.integers(0, n, size=(300000, 2))
    uv = np.concatenate([hub_edges, hub2, rest]).astype(np.int32)
    for opts in ((1, 1, 0, 1), (0, 0, 0, 1)):
        g = pkg.Graph.from_edges(torch.from_numpy(uv).cuda(), n, opts=pkg.default_opts(*opts))
        off, adj = _gpu_csr(g)
        ref = oracle.build_csr(n, uv, dedup=bool(opts[0]), drop_self_loops=bool(opts[1]), sort_rows=True)
        assert np.array_equal(off, ref.offsets) and np.array_equal(adj, ref.adj)
        g.close()


def test_csr_input_path():
    n, uv = graphs.skewed_edges(3000, 20000, 4)
    ref = oracle.build_csr(n, uv)
    g = pkg.Graph.from_csr(ref.offsets, ref.adj, n)
    off, adj = _gpu_csr(g)
    want = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    assert np.array_equal(off, want.offsets) and np.array_equal(adj, want.adj)
    g.close()


def test_malformed_inputs():
    with pytest.raises(pkg.BfsError, match="MALFORMED.*tuple 1 = \\(2, 5\\)"):
        pkg.Graph.from_edges(np.array([[0, 1], [2, 5]], np.int32), 5)
    with pytest.raises(pkg.BfsError, match="CAPACITY"):
        pkg.Graph.kronecker(31)


# ------------------------------------------------------------------ BFS
FIXTURES = {
    "g1": graphs.g1(), "path": graphs.path(40), "cycle": graphs.cycle(33), "star": graphs.star(70),
    "clique": graphs.clique(20), "bip": graphs.complete_bipartite(5, 9), "cube": graphs.hypercube(7),
    "grid": graphs.grid(13, 17), "heap": graphs.heap_tree(300),
    "union": graphs.disjoint_union(graphs.path(6), graphs.cycle(5), graphs.star(40), graphs.clique(7)),
    "skewed": graphs.skewed_edges(3000, 20000, 1), "random": graphs.random_edges(2000, 9000, 3),
}


@pytest.mark.parametrize("name", sorted(FIXTURES))
@pytest.mark.parametrize("pi", range(len(POLICIES)))
def test_fixtures_all_policies(name, pi):
    n, uv = FIXTURES[name]
    g = pkg.Graph.from_edges(uv, n)
    ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    for root in sorted({0, n // 2, n - 1, int(np.argmax(ref.degree()))}):
        _check_run(g, ref, root, POLICIES[pi], uv)
    g.close()


def test_g1_golden_trace():
    want = graphs.load_golden_table("g1_do_trace.txt")
    n, uv = graphs.g1()
    g = pkg.Graph.from_edges(uv, n)
    g.set_policy(mode=0)
    parent, depth = g.run(0)
    assert depth.cpu().tolist() == [0, 1, 1, 1, 2, 3]
    assert parent.cpu().tolist() == want["auto_parent"]
    _, levels = g.stats()
    assert [lv["inspections"] for lv in levels] == want["auto_insp"]
    g.set_policy(mode=1)
    g.run(0)
    _, levels = g.stats()
    assert [lv["inspections"] for lv in levels] == want["td_insp"]
    g.close()


def test_isolated_root_and_out_of_range():
    g = pkg.Graph.from_edges(np.array([[0, 1], [1, 2]], np.int32), 6)
    parent, depth = g.run(4)
    assert depth.cpu().tolist() == [-1, -1, -1, -1, 0, -1]
    assert parent.cpu().tolist() == [-1, -1, -1, -1, 4, -1]
    run, levels = g.stats()
    assert run["levels"] == 1 and run["reached"] == 1 and run["component_edge_tuples"] == 0
    with pytest.raises(pkg.BfsError, match="OUT_OF_RANGE"):
        g.run(6)
    g.close()


def test_self_loops_and_multi_edges_kept():
    n, uv = graphs.grid(9, 9)
    uv2 = np.concatenate([uv, uv[::2], np.array([[v, v] for v in range(0, n, 3)], np.int32)])
    g = pkg.Graph.from_edges(uv2, n, opts=pkg.default_opts(False, False, False, True))
    ref = oracle.build_csr(n, uv2, sort_rows=True)
    for pol in POLICIES:
        _check_run(g, ref, 40, pol, uv2)
    g.close()


@pytest.mark.parametrize("abc,seed", [(oracle.KRON_ABC, 1), (oracle.ER_ABC, 2)])
def test_s16_64_roots(abc, seed):
    scale = 16
    g = pkg.Graph.kronecker(scale, 16, seed, abc)
    uv, ref = oracle.kron_graph(scale, 16, seed, abc)
    off, adj = _gpu_csr(g)
    assert np.array_equal(off, ref.offsets) and np.array_equal(adj, ref.adj)
    roots = g.sample_roots(scale, seed, 64)
    assert np.array_equal(roots, oracle.sample_roots(ref, scale, seed, 64))
    for i, r in enumerate(roots):
        _check_run(g, ref, r, POLICIES[i % 3] if i < 12 else POLICIES[0], uv)
    g.close()


def test_host_output_buffers():
    """the end-to-end path: outputs in (pinned or pageable) host memory"""
    scale = 13
    g = pkg.Graph.kronecker(scale, 16, 4)
    uv, ref = oracle.kron_graph(scale, 16, 4)
    r = int(g.sample_roots(scale, 4, 1)[0])
    d = np.empty(1 << scale, np.int32)
    p = torch.empty(1 << scale, dtype=torch.int32).pin_memory()
    pkg.bfs_run(g.h, r, p, d)
    want, _ = oracle.bfs(ref, r)
    assert np.array_equal(d, want)
    assert not oracle.validate(ref, r, d, p.numpy(), ref_depth=want)
    g.close()


@pytest.mark.parametrize("reindex", [False, True])
@pytest.mark.parametrize("loop", ["host", "graph", "persistent", "cluster"])
def test_pinned_host_outputs(reindex, loop):
    """pinned host outputs (the e2e leg of bench.py): every entry is overwritten
    (buffers start as garbage), depth == oracle, parents valid, in every level loop
    and with and without the degree reindex"""
    scale = 14
    g = pkg.Graph.kronecker(scale, 16, 9, opts=pkg.default_opts(reindex_by_degree=reindex))
    g.set_policy(loop=loop)
    uv, ref = oracle.kron_graph(scale, 16, 9)
    n = 1 << scale
    p = torch.full((n,), 0x5a5a5a5a, dtype=torch.int32).pin_memory()
    d = torch.full((n,), 0x5a5a5a5a, dtype=torch.int32).pin_memory()
    for r in g.sample_roots(scale, 9, 3):
        p.fill_(0x5a5a5a5a)
        d.fill_(0x5a5a5a5a)
        pkg.bfs_run(g.h, int(r), p, d)
        want, _ = oracle.bfs(ref, int(r))
        assert np.array_equal(d.numpy(), want)
        assert not oracle.validate(ref, int(r), d.numpy(), p.numpy(), ref_depth=want)
        # depth only / parent only
        d.fill_(0x5a5a5a5a)
        pkg.bfs_run(g.h, int(r), None, d)
        assert np.array_equal(d.numpy(), want)
    g.close()


def test_repeated_runs_and_stream():
    s = torch.cuda.Stream()
    scale = 14
    g = pkg.Graph.kronecker(scale, 16, 6, stream=s)
    uv, ref = oracle.kron_graph(scale, 16, 6)
    roots = g.sample_roots(scale, 6, 5)
    for _ in range(2):
        for r in roots:
            with torch.cuda.stream(s):
                parent, depth = g.run(int(r))
            s.synchronize()
            want, _ = oracle.bfs(ref, int(r))
            assert np.array_equal(depth.cpu().numpy(), want)
    g.close()


def test_deep_search_falls_back_to_host_loop():
    """A path of 5000 vertices needs 5000 steps: more than the device loops' record
    capacity (4096), so the search is rerun host-driven; outputs and counters exact."""
    n, uv = graphs.path(5000)
    ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    g = pkg.Graph.from_edges(uv, n)
    for pol in (dict(mode=0), dict(mode=1), dict(mode=0, loop="graph")):
        run, levels = _check_run(g, ref, 0, pol, uv)
        assert run["levels"] == 5000
    g.close()


@pytest.mark.parametrize("reindex", [False, True])
def test_all_loops_agree_kronecker(reindex):
    """Persistent kernel, loop graph and host loop give identical outputs and step records."""
    uv, ref = oracle.kron_graph(14, 16, 11)
    g = pkg.Graph.kronecker(14, 16, 11, opts=pkg.default_opts(reindex_by_degree=reindex))
    for r in g.sample_roots(14, 11, 6):
        out = []
        for loop in ("persistent", "graph", "host", "cluster"):
            g.set_policy(mode=0, alpha=30, beta=24, loop=loop, level_times=True)
            parent, depth = g.run(int(r))
            run, levels = g.stats()
            out.append((parent.cpu().numpy(), depth.cpu().numpy(), run, levels))
            assert all(lv["kernel_ms"] >= 0 and lv["ms"] > 0 for lv in levels)
        want, _ = oracle.bfs(ref, int(r)) if not reindex else (None, None)
        for o in out[1:]:
            assert np.array_equal(out[0][1], o[1])
            for k in ("direction", "frontier", "discovered", "m_f", "m_u", "inspections", "scanned"):
                assert [lv[k] for lv in out[0][3]] == [lv[k] for lv in o[3]], k
            assert out[0][2]["reached"] == o[2]["reached"]
            assert out[0][2]["component_edge_tuples"] == o[2]["component_edge_tuples"]
        if want is not None:
            assert np.array_equal(out[0][1], want)
            assert not oracle.validate(ref, int(r), out[0][1], out[0][0], ref_depth=want)
    g.close()


def test_edge_list_file_ingestion(tmp_path):
    """f4: an edge list read from a text file builds the same graph as the oracle's."""
    from paper_1503_04359_b200.edgelist import load_edge_list
    n0, e = graphs.skewed_edges(3000, 20000, 9)
    e = np.asarray(e).reshape(-1, 2) * 7 + 11          # sparse file IDs, relabeled densely
    p = tmp_path / "g.txt"
    p.write_text("# skewed test graph\n" + "".join(f"{u} {v}\n" for u, v in e))
    uv, n, ids = load_edge_list(str(p))
    ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    g = pkg.Graph.from_edges(uv, n)
    for root in (0, int(np.argmax(ref.degree()))):
        _check_run(g, ref, root, dict(mode=0), uv)
    g.close()


def _check_outputs(g, ref, root, policy):
    """depth == oracle, parents valid, reached count -- label-order independent checks."""
    g.set_policy(**policy)
    parent, depth = g.run(int(root))
    d = depth.cpu().numpy()
    p = parent.cpu().numpy()
    want, _ = oracle.bfs(ref, int(root))
    assert np.array_equal(d, want), (root, policy, np.nonzero(d != want)[0][:8])
    assert not oracle.validate(ref, int(root), d, p, ref_depth=want)
    run, levels = g.stats()
    assert run["reached"] == int((want >= 0).sum())
    assert sum(lv["frontier"] for lv in levels) == run["reached"]


def _degenerate_cases():
    rng = np.random.default_rng(5)
    e0 = np.zeros((0, 2), np.int32)
    loops = np.array([[v, v] for v in range(0, 50, 2)], np.int32)
    n_hub, hub = graphs.star(5000)                       # a row longer than every shared-memory path
    hub = np.concatenate([hub, rng.integers(1, n_hub, size=(3000, 2)).astype(np.int32)])
    n_u, uni = graphs.disjoint_union(graphs.path(7), graphs.clique(5), graphs.star(33))
    return {
        "single": (1, e0), "edgeless": (1000, e0), "self_loops_only": (50, loops),
        "ragged33": graphs.path(33), "ragged1025": graphs.random_edges(1025, 4000, 7),
        "ragged4097": graphs.random_edges(4097, 30000, 8), "hub5000": (n_hub, hub),
        "isolated_tail": (n_u + 77, uni),                # 77 isolated vertices after the components
    }


@pytest.mark.parametrize("loop", ["persistent", "graph", "host", "cluster"])
@pytest.mark.parametrize("reindex", [False, True])
def test_degenerate_and_ragged_graphs(loop, reindex):
    """Empty, edgeless, self-loop-only and ragged-size graphs, a long hub row, isolated roots:
    every level loop, with and without the degree reindex (isolated vertices last)."""
    for name, (n, uv) in _degenerate_cases().items():
        g = pkg.Graph.from_edges(uv, n, opts=pkg.default_opts(reindex_by_degree=reindex))
        ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
        deg = ref.degree()
        roots = {0, n - 1, int(np.argmax(deg))}
        if (deg == 0).any():
            roots.add(int(np.nonzero(deg == 0)[0][-1]))   # an isolated root
        for root in sorted(roots):
            for pol in (dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=0)):
                _check_outputs(g, ref, root, dict(loop=loop, **pol))
        g.close()


@pytest.mark.parametrize("loop", ["graph", "host"])
def test_claim_only_topdown_steps(loop, monkeypatch):
    """Large top-down steps run claim-only + k_td_finish (winners read back in vertex order).
    Forcing it on every top-down step (BFS_TD_CLAIM_MIN=1) must change nothing observable."""
    monkeypatch.setenv("BFS_TD_CLAIM_MIN", "1")
    monkeypatch.setenv("BFS_TD_SMALL", "-1")   # small steps would take the one-kernel path
    for name in ("g1", "union", "skewed", "random", "grid"):
        n, uv = FIXTURES[name]
        g = pkg.Graph.from_edges(uv, n)
        ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
        for root in sorted({0, n - 1, int(np.argmax(ref.degree()))}):
            for pol in (dict(mode=0), dict(mode=1), dict(mode=3, alpha=500, beta=2)):
                _check_run(g, ref, root, dict(loop=loop, **pol), uv)
        g.close()
    uv, ref = oracle.kron_graph(14, 16, 9)
    g = pkg.Graph.kronecker(14, 16, 9, opts=pkg.default_opts(reindex_by_degree=True))
    for r in g.sample_roots(14, 9, 4):
        _check_outputs(g, ref, int(r), dict(loop=loop, mode=1))
        _check_outputs(g, ref, int(r), dict(loop=loop, mode=0, alpha=30, beta=1000))
    g.close()


@pytest.mark.parametrize("small", ["-1", str(1 << 40)])
def test_small_topdown_kernel(small, monkeypatch):
    """Top-down steps with m_f <= BFS_TD_SMALL run as one kernel on the device loop
    (k_td_small: warp per frontier vertex, from the queue or straight from the bitmap
    after a bottom-up step).  Forcing it on every top-down step, hub roots included, and
    disabling it must both leave every output and counter exact."""
    monkeypatch.setenv("BFS_TD_SMALL", small)
    for name in ("g1", "union", "skewed", "grid"):
        n, uv = FIXTURES[name]
        g = pkg.Graph.from_edges(uv, n)
        ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
        for root in sorted({0, n - 1, int(np.argmax(ref.degree()))}):
            for pol in (dict(mode=0), dict(mode=1), dict(mode=3, alpha=500, beta=2), dict(mode=2, bu_from_level=1)):
                _check_run(g, ref, root, dict(loop="graph", **pol), uv)
        g.close()
    uv, ref = oracle.kron_graph(14, 16, 9)
    g = pkg.Graph.kronecker(14, 16, 9, opts=pkg.default_opts(reindex_by_degree=True))
    for r in list(g.sample_roots(14, 9, 3)) + [int(np.argmax(ref.degree()))]:
        _check_outputs(g, ref, int(r), dict(loop="graph", mode=1))
        _check_outputs(g, ref, int(r), dict(loop="graph", mode=0, alpha=30, beta=1000))
    g.close()


def test_persistent_grid_not_coresident_falls_back(monkeypatch):
    """The persistent search is a cooperative launch (its grid barrier needs every CTA
    resident).  A grid that cannot be co-resident must fail the launch, and the search
    must then run as the loop graph with identical results -- never hang."""
    uv, ref = oracle.kron_graph(12, 16, 4)
    g = pkg.Graph.kronecker(12, 16, 4)
    roots = [int(r) for r in g.sample_roots(12, 4, 3)]
    monkeypatch.setenv("BFS_PERSIST_GRID", str(1 << 20))
    for r in roots:
        _check_run(g, ref, r, dict(mode=0, loop="persistent"), uv)
    monkeypatch.delenv("BFS_PERSIST_GRID")
    for r in roots:
        _check_run(g, ref, r, dict(mode=0, loop="persistent"), uv)
    g.close()


@pytest.mark.parametrize("reindex,rows", [(False, 1), (True, 1), (False, 2), (False, 0)])
def test_device_validator_matches_oracle_validator(reindex, rows):
    """bfs_validate (the bench's self-check) flags exactly the rules the oracle's CSR
    validator flags: on the GPU's own outputs (none) and on corrupted copies."""
    rng = np.random.default_rng(5 + rows)
    uv, _ = oracle.kron_graph(12, 16, 6)
    ref = oracle.build_csr(1 << 12, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    g = pkg.Graph.kronecker(12, 16, 6, opts=pkg.default_opts(reindex_by_degree=reindex, sort_rows=rows))
    for r in g.sample_roots(12, 6, 4):
        r = int(r)
        parent, depth = g.run(r)
        assert pkg.bfs_validate(g.h, r, parent, depth) == {}
        d0, p0 = depth.cpu().numpy(), parent.cpu().numpy()
        for kind in range(6):
            d, p = d0.copy(), p0.copy()
            v = int(rng.choice(np.flatnonzero(d0 > 1)))
            if kind == 0:
                p[v] = r                          # V2 + V3
            elif kind == 1:
                d[v], p[v] = -1, -1               # V4
            elif kind == 2:
                p[r] = v                          # V1
            elif kind == 3:
                d[v] += 1                         # V3 / V4
            elif kind == 4:
                p[v] = -1                         # V5
            else:
                d[v] = 0                          # V1 + V3 + V4
            want = {k for k in oracle.validate(ref, r, d, p) if k != "V6_exact_depth"}
            got = set(pkg.bfs_validate(g.h, r, torch.from_numpy(p).cuda(), torch.from_numpy(d).cuda()))
            assert got == want, (kind, got, want)
            assert set(pkg.bfs_validate(g.h, r, p, d)) == want          # host buffers
    g.close()


@pytest.mark.parametrize("nb4", ["2", "1", "0"])
@pytest.mark.parametrize("loop", ["graph", "host"])
def test_bottomup_second_probe_blocks(nb4, loop, monkeypatch):
    """Bottom-up rows that miss on the first arc probe arcs 1..4 from the dense nb4 block
    (phase 3a'' of k_bu_batch, planes of 4 arcs) and continue in the CSR after the last plane; BFS_BU_NB4=0 takes the
    CSR from arc 1.  Both must give the emulator's counters, inspections and first
    frontier neighbours (every fixture has rows of degree 2..6 around the block edge)."""
    monkeypatch.setenv("BFS_BU_NB4", nb4)
    for name in ("skewed", "random", "grid", "cube", "union", "clique"):
        n, uv = FIXTURES[name]
        g = pkg.Graph.from_edges(uv, n)
        ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
        for root in sorted({0, n - 1, int(np.argmax(ref.degree()))}):
            for pol in (dict(mode=1), dict(mode=2, bu_from_level=1), dict(mode=0, alpha=2, beta=4)):
                _check_run(g, ref, root, dict(loop=loop, **pol), uv)
        g.close()
    uv, ref = oracle.kron_graph(14, 16, 5)
    g = pkg.Graph.kronecker(14, 16, 5, opts=pkg.default_opts(reindex_by_degree=True))
    for r in g.sample_roots(14, 5, 4):
        _check_outputs(g, ref, int(r), dict(loop=loop, mode=1))
        _check_outputs(g, ref, int(r), dict(loop=loop, mode=0, alpha=30, beta=1000))
    g.close()
