"""Multi-partition parity on one GPU: p rank endpoints of a local communicator,
each driven from its own host thread through the same C ABI calls, kernels and
host logic as the one-process-per-GPU NCCL path (only the transport differs).
The concatenated owned slices must match the oracle exactly as on one GPU, and
the global per-step counters must equal the emulator's on every rank."""
import numpy as np
import pytest

import oracle
from tests import graphs

torch = pytest.importorskip("torch")
pkg = pytest.importorskip("paper_1503_04359_b200")
from paper_1503_04359_b200 import build as pkg_build  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    pkg_build.build()
    torch.cuda.set_device(0)


def _build(p, make):
    comms = pkg.bfs_comm_create_local(p, 0)

    def mk(r):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        return make(comms[r], s)

    gs = pkg.run_ranks(mk, p)
    return comms, gs


def _run_all(gs, root, policy):
    p = len(gs)

    def go(r):
        torch.cuda.set_device(0)
        g = gs[r]
        g.set_policy(**policy)
        with torch.cuda.stream(g.stream):
            parent, depth = g.run(int(root))
        g.stream.synchronize()
        run, levels = g.stats()
        return parent.cpu().numpy(), depth.cpu().numpy(), run, levels

    res = pkg.run_ranks(go, p)
    parent = np.concatenate([x[0] for x in res])
    depth = np.concatenate([x[1] for x in res])
    return parent, depth, [x[2] for x in res], [x[3] for x in res]


def _check(gs, ref, root, policy, uv=None):
    parent, depth, runs, levels = _run_all(gs, root, policy)
    want, _ = oracle.bfs(ref, int(root))
    assert np.array_equal(depth, want), np.nonzero(depth != want)[0][:10]
    assert not oracle.validate(ref, int(root), depth, parent, ref_depth=want)
    emu = oracle.do_emulate(ref, want, alpha=policy.get("alpha", 15), beta=policy.get("beta", 18),
                            policy=policy.get("mode", 0), bu_from=policy.get("bu_from_level", 0),
                            want_bu_parent=True, coord_hi=gs[0].local_end)   # coordinator = partition 0
    for lv in levels:   # every rank reports the same global counters
        for key, lk in (("dir", "direction"), ("n_f", "frontier"), ("discovered", "discovered"),
                        ("m_f", "m_f"), ("m_u", "m_u"), ("insp", "inspections")):
            assert [x[lk] for x in lv] == emu[key].tolist(), key
    bu = emu["bu_parent"] >= 0
    assert np.array_equal(parent[bu], emu["bu_parent"][bu])
    for run in runs:
        assert run["reached"] == int((want >= 0).sum())
        if uv is not None:
            assert run["component_edge_tuples"] == oracle.component_tuples(uv, want)
    return runs, levels


def _close(comms, gs):
    for g in gs:
        g.close()
    for c in comms:
        pkg.bfs_comm_destroy(c)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_partition_ranges_tile(p):
    n = 1000
    rs = [pkg.bfs_partition_range(n, p, r) for r in range(p)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    for (a, b), (c, d) in zip(rs, rs[1:]):
        assert b == c and a % 32 == 0


def test_g1_two_partitions():
    """push OR-merges claims into the owner; pull overwrites frontier views."""
    n, uv = graphs.g1()
    ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    comms, gs = _build(2, lambda c, s: pkg.Graph.from_edges(uv, n, comm=c, stream=s))
    for pol in (dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=0)):
        for root in range(n):
            _check(gs, ref, root, pol, uv)
    _close(comms, gs)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("abc", [oracle.KRON_ABC, oracle.ER_ABC])
def test_kronecker_s14(p, abc):
    scale, seed = 14, 7
    uv, ref = oracle.kron_graph(scale, 16, seed, abc)
    comms, gs = _build(p, lambda c, s: pkg.Graph.kronecker(scale, 16, seed, abc, comm=c, stream=s))
    # every rank holds exactly the oracle rows of its range
    for g in gs:
        off, adj = g.export_csr()
        lo, hi = g.local_begin, g.local_end
        assert np.array_equal(off.cpu().numpy(), ref.offsets[lo:hi + 1] - ref.offsets[lo])
        assert np.array_equal(adj.cpu().numpy(), ref.adj[ref.offsets[lo]:ref.offsets[hi]])
    roots = pkg.run_ranks(lambda r: gs[r].sample_roots(scale, seed, 6), p)
    assert all(np.array_equal(roots[0], x) for x in roots)
    assert np.array_equal(roots[0], oracle.sample_roots(ref, scale, seed, 6))
    pols = [dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=1), dict(mode=0, alpha=2, beta=4),
            dict(mode=3, alpha=500, beta=3), dict(mode=3, alpha=100, beta=2)]
    slice_bytes = pkg.bfs_partition_range(ref.n, p, 0)[1] // 8
    sparse_pulls = 0
    for i, r in enumerate(roots[0]):
        runs, levels = _check(gs, ref, r, pols[i % len(pols)], uv)
        if p > 1:
            # the run's bytes = the levels' + the final parent-log aggregation (bitmap pushes)
            lv_bytes = sum(x["nvlink_bytes"] for x in levels[0])
            assert lv_bytes <= runs[0]["nvlink_bytes"]
            if runs[0]["ms_aggregate"] == 0:
                assert lv_bytes == runs[0]["nvlink_bytes"]
            # bottom-up pulls: bitmap slices when dense, vertex lists when sparse
            for lv in levels[0]:
                if lv["direction"] == 1 and 4 * lv["frontier"] < slice_bytes * (p - 1):
                    sparse_pulls += 1
                    assert lv["nvlink_bytes"] < slice_bytes * (p - 1)
    if p > 1:
        assert sparse_pulls > 0
    _close(comms, gs)


@pytest.mark.parametrize("p", [2, 5])
def test_fixtures_multi(p):
    for name, (n, uv) in {"union": graphs.disjoint_union(graphs.path(40), graphs.star(90), graphs.clique(9)),
                          "skewed": graphs.skewed_edges(4000, 30000, 5), "grid": graphs.grid(20, 31)}.items():
        ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
        comms, gs = _build(p, lambda c, s: pkg.Graph.from_edges(uv, n, comm=c, stream=s))
        for root in sorted({0, n - 1, int(np.argmax(ref.degree()))}):
            for pol in (dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=0), dict(mode=3, alpha=300, beta=2)):
                _check(gs, ref, root, pol, uv)
        _close(comms, gs)


@pytest.mark.parametrize("p", [2, 4])
def test_degree_row_order_multi(p):
    scale, seed = 13, 3
    uv, base = oracle.kron_graph(scale, 16, seed)
    ref = oracle.sort_rows_by_degree(base)
    opts = pkg.default_opts(sort_rows=2)
    comms, gs = _build(p, lambda c, s: pkg.Graph.kronecker(scale, 16, seed, comm=c, stream=s, opts=opts))
    for g in gs:
        off, adj = g.export_csr()
        lo, hi = g.local_begin, g.local_end
        assert np.array_equal(adj.cpu().numpy(), ref.adj[ref.offsets[lo]:ref.offsets[hi]])
    roots = oracle.sample_roots(ref, scale, seed, 4)
    for r in roots:
        _check(gs, ref, r, dict(mode=0), uv)
    _close(comms, gs)


def test_nccl_bootstrap_single_rank():
    """The NCCL backend (dlopen of torch's libnccl, unique id, CommInitRank) on the one GPU
    a box has: a one-rank communicator builds the graph and searches like no communicator."""
    import torch
    torch.cuda.set_device(0)
    uid = pkg.bfs_comm_unique_id()
    assert len(uid) == 128 and any(uid)
    comm = pkg.bfs_comm_create(1, 0, uid, 0)
    scale, seed = 12, 4
    uv, ref = oracle.kron_graph(scale, 16, seed)
    g = pkg.Graph.kronecker(scale, 16, seed, comm=comm)
    assert (g.local_begin, g.local_end) == (0, ref.n)
    for r in g.sample_roots(scale, seed, 3):
        parent, depth = g.run(int(r))
        want, _ = oracle.bfs(ref, int(r))
        assert np.array_equal(depth.cpu().numpy(), want)
        assert not oracle.validate(ref, int(r), depth.cpu().numpy(), parent.cpu().numpy(), ref_depth=want)
    g.close()
    pkg.bfs_comm_destroy(comm)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_degree_reindex_multi(p):
    """Degree reindex on p ranks ("after partitioning ... permutation of local IDs"):
    the oracle's degree_reindex_local(g, p) -- block partition of the original labels, then
    (degree desc, ID asc) local IDs -- rows in global degree order; every rank's outputs
    are its own original labels, produced locally (no aggregation exchange)."""
    scale, seed = 14, 5
    uv, ref = oracle.kron_graph(scale, 16, seed)
    lab, pos = oracle.degree_reindex_local(ref, p)
    rel = oracle.relabel_csr(ref, lab, pos)
    inv = np.empty_like(lab)
    inv[lab] = np.arange(ref.n)
    opts = pkg.default_opts(reindex_by_degree=True)
    comms, gs = _build(p, lambda c, s: pkg.Graph.kronecker(scale, 16, seed, comm=c, stream=s, opts=opts))
    for g in gs:   # every rank holds exactly the oracle's relabeled rows of its range
        off, adj = g.export_csr()
        lo, hi = g.local_begin, g.local_end
        assert np.array_equal(off.cpu().numpy(), rel.offsets[lo:hi + 1] - rel.offsets[lo])
        assert np.array_equal(adj.cpu().numpy(), rel.adj[rel.offsets[lo]:rel.offsets[hi]])
    roots = pkg.run_ranks(lambda r: gs[r].sample_roots(scale, seed, 6), p)
    assert np.array_equal(roots[0], oracle.sample_roots(ref, scale, seed, 6))
    nb = gs[0].local_end
    pols = [dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=1), dict(mode=3, alpha=500, beta=3)]
    for i, r in enumerate(roots[0]):
        pol = pols[i % len(pols)]
        parent, depth, runs, levels = _run_all(gs, r, pol)
        want, _ = oracle.bfs(ref, int(r))
        assert np.array_equal(depth, want), np.nonzero(depth != want)[0][:10]
        assert not oracle.validate(ref, int(r), depth, parent, ref_depth=want)
        want_int = np.empty_like(want)
        want_int[lab] = want
        emu = oracle.do_emulate(rel, want_int, alpha=pol.get("alpha", 15), beta=pol.get("beta", 18),
                                policy=pol["mode"], bu_from=pol.get("bu_from_level", 0), want_bu_parent=True,
                                coord_hi=nb)
        for lv in levels:
            for key, lk in (("dir", "direction"), ("n_f", "frontier"), ("discovered", "discovered"),
                            ("m_f", "m_f"), ("m_u", "m_u"), ("insp", "inspections")):
                assert [x[lk] for x in lv] == emu[key].tolist(), key
        bu = np.nonzero(emu["bu_parent"] >= 0)[0]            # internal labels found bottom-up
        assert np.array_equal(parent[inv[bu]], inv[emu["bu_parent"][bu]])
        for run in runs:
            assert run["reached"] == int((want >= 0).sum())
            assert run["component_edge_tuples"] == oracle.component_tuples(uv, want)
            # outputs are local; only bitmap-pushed levels leave parent logs to aggregate
            bitmap = any(x["direction"] == 0 and x["m_f"] >= ref.n // 64 for x in levels[0])
            assert (run["ms_aggregate"] > 0) == bitmap
    _close(comms, gs)


def test_degree_reindex_multi_needs_exact_deal():
    comms = pkg.bfs_comm_create_local(3, 0)
    with pytest.raises(pkg.BfsError, match="divisible"):
        pkg.run_ranks(lambda r: pkg.Graph.kronecker(10, 16, 1, comm=comms[r],
                                                    opts=pkg.default_opts(reindex_by_degree=True)), 3)
    for c in comms:
        pkg.bfs_comm_destroy(c)


@pytest.mark.parametrize("p", [2, 3, 8])
@pytest.mark.parametrize("bitmap_min", ["1", "20000"])
def test_bitmap_push(p, bitmap_min, monkeypatch):
    """Dense top-down levels push per-peer outbox BITMAPS (Alg. 2 NextFrontier[P]) and defer
    the parents to a final aggregation of (vertex, parent, level) logs: forced on every
    top-down step (BFS_TD_BITMAP_MIN=1) or on the dense ones only, with and without the degree
    reindex, the outputs, parents and counters must match the oracle exactly as in list mode."""
    monkeypatch.setenv("BFS_TD_BITMAP_MIN", bitmap_min)
    scale, seed = 14, 4
    uv, ref = oracle.kron_graph(scale, 16, seed)
    comms, gs = _build(p, lambda c, s: pkg.Graph.kronecker(scale, 16, seed, comm=c, stream=s))
    roots = pkg.run_ranks(lambda r: gs[r].sample_roots(scale, seed, 5), p)[0]
    pols = [dict(mode=1), dict(mode=0), dict(mode=2, bu_from_level=2), dict(mode=0, alpha=2, beta=4),
            dict(mode=3, alpha=500, beta=2)]
    slice_bytes = pkg.bfs_partition_range(ref.n, p, 0)[1] // 8
    bitmap_levels = 0
    for i, r in enumerate(roots):
        runs, levels = _check(gs, ref, r, pols[i % len(pols)], uv)
        for lv in levels[0]:
            if lv["direction"] == 0 and lv["m_f"] >= int(bitmap_min):
                bitmap_levels += 1
                assert lv["nvlink_bytes"] == slice_bytes * (p - 1)
        if any(lv["direction"] == 0 and lv["m_f"] >= int(bitmap_min) for lv in levels[0]):
            assert runs[0]["ms_aggregate"] > 0
    assert bitmap_levels > 0
    _close(comms, gs)
    if p in (2, 8):   # degree-reindexed ranks (partition-local labels)
        lab, pos = oracle.degree_reindex_local(ref, p)
        comms, gs = _build(p, lambda c, s: pkg.Graph.kronecker(scale, 16, seed, comm=c, stream=s,
                                                              opts=pkg.default_opts(reindex_by_degree=True)))
        for r in roots[:3]:
            parent, depth, runs, levels = _run_all(gs, r, dict(mode=1))
            want, _ = oracle.bfs(ref, int(r))
            assert np.array_equal(depth, want)
            assert not oracle.validate(ref, int(r), depth, parent, ref_depth=want)
        _close(comms, gs)
