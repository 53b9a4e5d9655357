"""Section 3.4 degree reindex on the GPU against the oracle.

The internal CSR must equal the oracle's relabeled CSR bit-exactly (labels by
degree descending / ID ascending, rows by neighbour position); bfs_run still
takes and returns original labels, so depth must equal the oracle's on the
original graph, parents must validate on the original graph, and the per-step
counters and inspections must equal the emulator run on the relabeled graph.
"""
import numpy as np
import pytest

import oracle
from tests import graphs

torch = pytest.importorskip("torch")
pkg = pytest.importorskip("paper_1503_04359_b200")
from paper_1503_04359_b200 import build as pkg_build  # noqa: E402

pytestmark = pytest.mark.gpu
REIDX = dict(dedup=True, drop_self_loops=True, reindex_by_degree=True, sort_rows=True)


@pytest.fixture(scope="module", autouse=True)
def _dev():
    pkg_build.build()
    torch.cuda.set_device(0)


def _labels(g):
    lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
    pkg.bfs_graph_export_labels(g.h, lab)
    return lab.cpu().numpy()


def _check(g, ref, rel, new, root, policy, uv):
    g.set_policy(**policy)
    parent, depth = g.run(int(root))
    d = depth.cpu().numpy()
    p = parent.cpu().numpy()
    want, _ = oracle.bfs(ref, int(root))
    assert np.array_equal(d, want)
    assert not oracle.validate(ref, int(root), d, p, ref_depth=want)
    want_int = np.empty_like(want)
    want_int[new] = want
    emu = oracle.do_emulate(rel, want_int, alpha=policy.get("alpha", 15), beta=policy.get("beta", 18),
                            policy=policy.get("mode", 0), bu_from=policy.get("bu_from_level", 0), want_bu_parent=True)
    run, levels = g.stats()
    for key, lk in (("dir", "direction"), ("n_f", "frontier"), ("discovered", "discovered"), ("m_f", "m_f"),
                    ("m_u", "m_u"), ("insp", "inspections")):
        assert [lv[lk] for lv in levels] == emu[key].tolist(), key
    inv = np.empty_like(new)
    inv[new] = np.arange(len(new))
    bp = emu["bu_parent"]
    for vi in np.nonzero(bp >= 0)[0]:
        assert p[inv[vi]] == inv[bp[vi]]
    assert run["component_edge_tuples"] == oracle.component_tuples(uv, want)


@pytest.mark.parametrize("scale,abc,seed", [(12, oracle.KRON_ABC, 3), (14, oracle.KRON_ABC, 1),
                                            (12, oracle.ER_ABC, 2)])
def test_kronecker_reindex(scale, abc, seed):
    g = pkg.Graph.kronecker(scale, 16, seed, abc, opts=pkg.default_opts(**REIDX))
    uv, ref = oracle.kron_graph(scale, 16, seed, abc)
    new, pos = oracle.degree_reindex(ref, 1)
    rel = oracle.relabel_csr(ref, new, pos)
    assert np.array_equal(_labels(g), new)
    off, adj = g.export_csr()
    assert np.array_equal(off.cpu().numpy(), rel.offsets)
    assert np.array_equal(adj.cpu().numpy(), rel.adj)
    roots = g.sample_roots(scale, seed, 8)
    assert np.array_equal(roots, oracle.sample_roots(ref, scale, seed, 8))
    pols = [dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=1)]
    for i, r in enumerate(roots):
        _check(g, ref, rel, new, r, pols[i % 3], uv)
    g.close()


def test_edges_reindex_and_host_outputs():
    n, uv = graphs.skewed_edges(3000, 25000, 8)
    g = pkg.Graph.from_edges(uv, n, opts=pkg.default_opts(**REIDX))
    ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    new, pos = oracle.degree_reindex(ref, 1)
    rel = oracle.relabel_csr(ref, new, pos)
    off, adj = g.export_csr()
    assert np.array_equal(off.cpu().numpy(), rel.offsets) and np.array_equal(adj.cpu().numpy(), rel.adj)
    for root in (0, int(np.argmax(ref.degree())), n - 1):
        _check(g, ref, rel, new, root, dict(mode=0), uv)
        d = np.empty(n, np.int32)
        p = np.empty(n, np.int32)
        pkg.bfs_run(g.h, root, p, d)
        want, _ = oracle.bfs(ref, root)
        assert np.array_equal(d, want) and not oracle.validate(ref, root, d, p, ref_depth=want)
    g.close()


def test_radix_order_large_ties():
    """many equal degrees: the stable sort must keep ascending IDs inside a degree class"""
    n, uv = graphs.random_edges(1 << 16, 1 << 16, 4, self_loops=False)
    g = pkg.Graph.from_edges(uv, n, opts=pkg.default_opts(**REIDX))
    ref = oracle.build_csr(n, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    new, _ = oracle.degree_reindex(ref, 1)
    assert np.array_equal(_labels(g), new)
    g.close()


DEGROWS = dict(dedup=True, drop_self_loops=True, reindex_by_degree=False, sort_rows=2)


@pytest.mark.parametrize("scale,abc,seed", [(14, oracle.KRON_ABC, 2), (12, oracle.ER_ABC, 5)])
def test_degree_row_order(scale, abc, seed):
    """sort_rows=2: rows by decreasing neighbour degree, labels unchanged"""
    g = pkg.Graph.kronecker(scale, 16, seed, abc, opts=pkg.default_opts(**DEGROWS))
    uv, base = oracle.kron_graph(scale, 16, seed, abc)
    ref = oracle.sort_rows_by_degree(base)
    off, adj = g.export_csr()
    assert np.array_equal(off.cpu().numpy(), ref.offsets) and np.array_equal(adj.cpu().numpy(), ref.adj)
    ident = np.arange(ref.n)
    for i, r in enumerate(g.sample_roots(scale, seed, 6)):
        _check(g, ref, ref, ident, r, [dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=1)][i % 3], uv)
    g.close()


@pytest.mark.parametrize("nb4", ["2", "1", "0"])
@pytest.mark.parametrize("loop", ["graph", "host"])
def test_reindex_bottomup_second_probes(nb4, loop, monkeypatch):
    """the nb4 second-probe phase on a relabeled graph (parents through ilabel):
    counters, inspections and bottom-up parents equal the emulator's on the relabeled CSR"""
    monkeypatch.setenv("BFS_BU_NB4", nb4)
    scale, seed = 13, 4
    g = pkg.Graph.kronecker(scale, 16, seed, oracle.KRON_ABC, opts=pkg.default_opts(**REIDX))
    uv, ref = oracle.kron_graph(scale, 16, seed, oracle.KRON_ABC)
    new, pos = oracle.degree_reindex(ref, 1)
    rel = oracle.relabel_csr(ref, new, pos)
    for i, r in enumerate(g.sample_roots(scale, seed, 4)):
        pol = [dict(mode=0, alpha=30, beta=1000), dict(mode=1), dict(mode=2, bu_from_level=1)][i % 3]
        _check(g, ref, rel, new, r, dict(loop=loop, **pol), uv)
    g.close()
