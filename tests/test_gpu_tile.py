"""Tiled top-down step (csrc/td_tile.cuh) against the oracle.

The BFS_TILE_* knobs shrink the heavy-row threshold, the tile size and the tile-mode
threshold so that small reindexed graphs run every top-down step tiled with many
tiles, heavy lists longer than one CTA batch (512) and light rows beside them.  Depth
must equal the serial oracle's (Alg. 1 is direction- and order-independent), parents
must validate, and every per-step counter must equal the emulator's (a tile-mode step
discovers exactly the set a plain top-down step discovers).
"""
import numpy as np
import pytest

import oracle
from tests.test_gpu_reindex import REIDX, _check

torch = pytest.importorskip("torch")
pkg = pytest.importorskip("paper_1503_04359_b200")
from paper_1503_04359_b200 import build as pkg_build  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    pkg_build.build()
    torch.cuda.set_device(0)


KNOBS = [
    # heavy degree, max words per tile, mass tiles
    dict(BFS_TILE_H="8", BFS_TILE_WORDS="4", BFS_TILE_COUNT="37"),      # tiny tiles: T in the hundreds
    dict(BFS_TILE_H="2", BFS_TILE_WORDS="48000", BFS_TILE_COUNT="1"),   # one tile, almost every row heavy
    dict(BFS_TILE_H="40", BFS_TILE_WORDS="16", BFS_TILE_COUNT="300"),   # few heavy rows, most arcs light
]


@pytest.mark.parametrize("knobs", KNOBS, ids=["tiny-tiles", "one-tile", "few-heavy"])
@pytest.mark.parametrize("scale,abc,seed", [(14, oracle.KRON_ABC, 1), (12, oracle.ER_ABC, 2)])
def test_tile_mode_parity(monkeypatch, knobs, scale, abc, seed):
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("BFS_TILE_MIN", "1")
    monkeypatch.setenv("BFS_TD_SMALL", "-1")   # no step takes the one-kernel small path
    g = pkg.Graph.kronecker(scale, 16, seed, abc, opts=pkg.default_opts(**REIDX))
    info = pkg.bfs_graph_tiles(g.h)
    assert info["tiles"] > 0 and info["heavy_rows"] > 0, info
    if knobs["BFS_TILE_COUNT"] == "1" and scale == 14:
        assert info["tiles"] == 1
    uv, ref = oracle.kron_graph(scale, 16, seed, abc)
    new, pos = oracle.degree_reindex(ref, 1)
    rel = oracle.relabel_csr(ref, new, pos)
    roots = g.sample_roots(scale, seed, 6)
    pols = [dict(mode=1, loop="graph"), dict(mode=0, loop="graph"), dict(mode=1, loop="host"),
            dict(mode=0, alpha=4, beta=18, loop="host"), dict(mode=3, alpha=500, beta=2, loop="graph"),
            dict(mode=2, bu_from_level=2, loop="graph")]
    for r, pol in zip(roots, pols):
        _check(g, ref, rel, new, r, pol, uv)
    g.close()


def test_tile_index_absent_without_reindex(monkeypatch):
    monkeypatch.setenv("BFS_TILE_H", "2")
    g = pkg.Graph.kronecker(12, 16, 1, oracle.KRON_ABC, opts=pkg.default_opts())
    assert pkg.bfs_graph_tiles(g.h)["tiles"] == 0
    g.close()
    monkeypatch.setenv("BFS_TILE", "0")
    g = pkg.Graph.kronecker(12, 16, 1, oracle.KRON_ABC, opts=pkg.default_opts(**REIDX))
    assert pkg.bfs_graph_tiles(g.h)["tiles"] == 0
    g.close()


def test_tile_mode_hub_root_k16(monkeypatch):
    """default tile sizes, heavy threshold lowered: the first top-down steps from a hub"""
    monkeypatch.setenv("BFS_TILE_H", "256")
    monkeypatch.setenv("BFS_TILE_MIN", "1024")
    monkeypatch.setenv("BFS_TD_SMALL", "-1")
    g = pkg.Graph.kronecker(16, 16, 1, oracle.KRON_ABC, opts=pkg.default_opts(**REIDX))
    assert pkg.bfs_graph_tiles(g.h)["tiles"] > 0
    uv, ref = oracle.kron_graph(16, 16, 1, oracle.KRON_ABC)
    new, pos = oracle.degree_reindex(ref, 1)
    rel = oracle.relabel_csr(ref, new, pos)
    hub = int(np.argmax(ref.degree()))
    for r in [hub] + [int(x) for x in g.sample_roots(16, 1, 3)]:
        _check(g, ref, rel, new, r, dict(mode=0, alpha=15, beta=18, loop="graph"), uv)
        _check(g, ref, rel, new, r, dict(mode=1, loop="graph"), uv)
    g.close()
