"""The partitioned search over REAL NCCL: one process per GPU (torch.multiprocessing
spawn, torch.distributed "nccl" only to ship the 128-byte NCCL id), the same C-ABI
calls bench.py --gpus N makes.  Every rank builds the Kronecker graph, searches the
sampled roots under several policies, and the concatenated owned slices must equal
the serial oracle's depths exactly, validate as a BFS tree, and carry the emulator's
global per-step counters on every rank (Alg. 2/3 push/pull).

Needs >= 2 CUDA devices; skipped otherwise (the round-end GPU pool has one GPU per
box, the 8-GPU driver step runs it).
"""
import os
import socket

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pkg = pytest.importorskip("paper_1503_04359_b200")
from paper_1503_04359_b200 import build as pkg_build  # noqa: E402

pytestmark = pytest.mark.gpu

POLICIES = [dict(mode=0), dict(mode=1), dict(mode=2, bu_from_level=1), dict(mode=0, alpha=2, beta=4),
            dict(mode=3, alpha=500, beta=3)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, scale, seed, reindex, nroots, out):
    import torch
    import torch.distributed as dist

    import paper_1503_04359_b200 as pkg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", rank))
    uid = pkg.bfs_comm_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
    dist.broadcast(t, 0)
    comm = pkg.bfs_comm_create(ws, rank, bytes(t.cpu().tolist()), rank)
    g = pkg.Graph.kronecker(scale, 16, seed, opts=pkg.default_opts(reindex_by_degree=reindex), comm=comm)
    roots = g.sample_roots(scale, seed, nroots)
    res = []
    for i, r in enumerate(roots):
        g.set_policy(**POLICIES[i % len(POLICIES)])
        parent, depth = g.run(int(r))
        run, levels = g.stats()
        res.append((int(r), parent.cpu().numpy(), depth.cpu().numpy(), run, levels))
    out.put((rank, g.local_begin, g.local_end, res))
    g.close()
    pkg.bfs_comm_destroy(comm)
    dist.destroy_process_group()


def _run(ws, scale, seed, reindex, nroots=5):
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, ws, port, scale, seed, reindex, nroots, q)) for r in range(ws)]
    for p in ps:
        p.start()
    got = sorted((q.get(timeout=600) for _ in range(ws)), key=lambda x: x[0])
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


@pytest.mark.timeout(900)
@pytest.mark.parametrize("reindex", [False, True])
def test_nccl_two_ranks_kronecker(reindex):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 CUDA devices (one process per GPU over NCCL)")
    pkg_build.build()
    ws = min(torch.cuda.device_count(), 8) if os.environ.get("BFS_NCCL_ALL_GPUS") else 2
    scale, seed = 14, 5
    got = _run(ws, scale, seed, reindex)
    uv, ref = oracle.kron_graph(scale, 16, seed)
    if reindex:
        lab, pos = oracle.degree_reindex_local(ref, ws)
        rel = oracle.relabel_csr(ref, lab, pos)
    else:
        lab, rel = np.arange(ref.n), ref
    assert got[0][1] == 0 and got[-1][2] == ref.n
    nroots = len(got[0][3])
    assert nroots > 0 and all(len(x[3]) == nroots for x in got)
    for i in range(nroots):
        root = got[0][3][i][0]
        assert all(x[3][i][0] == root for x in got)
        parent = np.concatenate([x[3][i][1] for x in got])
        depth = np.concatenate([x[3][i][2] for x in got])
        want, _ = oracle.bfs(ref, root)
        assert np.array_equal(depth, want), np.nonzero(depth != want)[0][:10]
        assert not oracle.validate(ref, root, depth, parent, ref_depth=want)
        pol = POLICIES[i % len(POLICIES)]
        want_int = np.empty_like(want)
        want_int[lab] = want
        emu = oracle.do_emulate(rel, want_int, alpha=pol.get("alpha", 15), beta=pol.get("beta", 18),
                                policy=pol["mode"], bu_from=pol.get("bu_from_level", 0), coord_hi=got[0][2])
        for x in got:
            levels = x[3][i][4]
            for key, lk in (("dir", "direction"), ("n_f", "frontier"), ("discovered", "discovered"),
                            ("m_f", "m_f"), ("m_u", "m_u"), ("insp", "inspections")):
                assert [lv[lk] for lv in levels] == emu[key].tolist(), key
            run = x[3][i][3]
            assert run["reached"] == int((want >= 0).sum())
            assert run["component_edge_tuples"] == oracle.component_tuples(uv, want)
            assert run["nvlink_bytes"] >= sum(lv["nvlink_bytes"] for lv in levels) and run["nvlink_bytes"] > 0
