"""world_size-2 gloo tests on CPU for the N>1 path's host logic.

Each rank takes its vertex range from the library's own partition arithmetic
(bfs_partition_range, host-only) and runs the partitioned protocol the GPU path
uses -- TD: per-owner claim lists, an allgather of the p x p claim counts, the
claims exchanged point to point and merged by the owner (Alg. 2); BU: allgather
of the next-frontier slices (Alg. 3); an allreduce of the switch counters so that
every rank picks the same direction -- with numpy standing in for the kernels
and gloo for NCCL.  Depth must equal the oracle's and the per-step counters the
emulator's, on both ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1503_04359_b200 as pkg
from tests import graphs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partitioned_bfs(ref, root, lo, hi, nb, p, rank, alpha=15, beta=18, mode=0):
    n = ref.n
    deg = ref.degree()
    visited = np.zeros(hi - lo, bool)
    visited[deg[lo:hi] == 0] = True            # skip mask
    depth = np.full(hi - lo, -1, np.int64)
    seen = np.zeros(n, bool)                  # remote claims already sent
    queue = []
    if lo <= root < hi:
        visited[root - lo] = True
        depth[root - lo] = 0
        queue = [root]

    def allreduce(vals):
        t = torch.tensor(vals, dtype=torch.int64)
        dist.all_reduce(t)
        return t.tolist()

    def coord(vals):   # mode 3: partition 0 is the coordinator; only it fills the slot
        return int(sum(deg[v] for v in vals)) if rank == 0 else 0

    n_f, m_f, m_fc = allreduce([len(queue), int(sum(deg[v] for v in queue)), coord(queue)])
    direction, prev, seen_deg, steps = 0, 0, 0, []
    bu_done, returned = 0, False
    sparse_pulls = [0]
    front = np.zeros(p * nb, bool)
    d = 0
    while n_f > 0:
        seen_deg += m_f
        m_u = ref.arcs - seen_deg
        if mode == 1:
            direction = 0
        elif mode == 3:
            if direction == 0:
                if not returned and m_fc * 10000 >= alpha * ref.arcs:
                    direction = 1
            elif bu_done >= beta:
                direction, returned = 0, True
            bu_done += direction
        elif direction == 0 and m_f * alpha > m_u:
            direction = 1
        elif direction == 1 and n_f * beta < n and n_f < prev:
            direction = 0
        nxt = []
        insp = 0
        if direction == 0:
            out = [[] for _ in range(p)]
            for u in queue:
                for v in ref.row(u):
                    insp += 1
                    if lo <= v < hi:
                        if not visited[v - lo]:
                            visited[v - lo] = True
                            depth[v - lo] = d + 1
                            nxt.append(int(v))
                    elif not seen[v]:
                        seen[v] = True
                        out[v // nb].append(int(v))
            counts = torch.tensor([len(o) for o in out], dtype=torch.int64)
            mat = [torch.zeros(p, dtype=torch.int64) for _ in range(p)]
            dist.all_gather(mat, counts)                       # p x p claim counts
            recv = [torch.zeros(int(mat[q][rank]), dtype=torch.int64) for q in range(p)]
            reqs = []
            for q in range(p):
                if q == rank:
                    continue
                if len(out[q]):
                    reqs.append(dist.isend(torch.tensor(out[q], dtype=torch.int64), q))
                if recv[q].numel():
                    reqs.append(dist.irecv(recv[q], q))
            for r in reqs:
                r.wait()
            for q in range(p):
                for v in recv[q].tolist():                     # owner merge
                    if not visited[v - lo]:
                        visited[v - lo] = True
                        depth[v - lo] = d + 1
                        nxt.append(v)
        elif 4 * n_f < (nb // 8) * (p - 1):
            # sparse pull: owned frontier vertices as lists, bitmap rebuilt locally
            counts = [torch.zeros(1, dtype=torch.int64) for _ in range(p)]
            dist.all_gather(counts, torch.tensor([len(queue)], dtype=torch.int64))
            recv = [torch.zeros(int(counts[q].item()), dtype=torch.int64) for q in range(p)]
            reqs = []
            for q in range(p):
                if q == rank:
                    continue
                if len(queue):
                    reqs.append(dist.isend(torch.tensor(queue, dtype=torch.int64), q))
                if recv[q].numel():
                    reqs.append(dist.irecv(recv[q], q))
            for r in reqs:
                r.wait()
            front = np.zeros(p * nb, bool)
            front[np.asarray(queue, np.int64)] = True
            for q in range(p):
                if q != rank:
                    front[recv[q].numpy()] = True
            sparse_pulls[0] += 1
        if direction == 1:
            if not (4 * n_f < (nb // 8) * (p - 1)):
                mine = np.zeros(nb, bool)
                for v in queue:
                    mine[v - lo] = True
                parts = [torch.zeros(nb, dtype=torch.bool) for _ in range(p)]
                dist.all_gather(parts, torch.from_numpy(mine))      # pull: overwrite every view
                front = torch.cat(parts).numpy()
            for vl in np.nonzero(~visited)[0]:
                for u in ref.row(lo + vl):
                    insp += 1
                    if front[u]:
                        nxt.append(int(lo + vl))
                        depth[vl] = d + 1
                        break
            for v in nxt:
                visited[v - lo] = True
        got = allreduce([len(nxt), int(sum(deg[v] for v in nxt)), insp, coord(nxt)])
        steps.append((direction, n_f, got[0], m_f, m_u, got[2] if direction else m_f))
        prev, n_f, m_f, m_fc = n_f, got[0], got[1], got[3]
        queue = nxt
        d += 1
    return depth, steps, sparse_pulls[0]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cases = [graphs.g1(), graphs.skewed_edges(700, 4000, 3), graphs.disjoint_union(graphs.path(30), graphs.star(50))]
        uv, ref = oracle.kron_graph(10, 16, 3)
        cases.append((ref.n, uv))
        out = []
        for n, e in cases:
            g = oracle.build_csr(n, e, dedup=True, drop_self_loops=True, sort_rows=True)
            lo, hi = pkg.bfs_partition_range(n, world, rank)
            nb = pkg.bfs_partition_range(n, world, 0)[1]
            for root in sorted({0, n - 1, int(np.argmax(g.degree()))}):
                for mode, alpha, beta in ((0, 15, 18), (1, 15, 18), (3, 500, 2), (3, 40, 3)):
                    depth, steps, sp = _partitioned_bfs(g, root, lo, hi, nb, world, rank, alpha, beta, mode)
                    full = [None] * world
                    dist.all_gather_object(full, depth.tolist())
                    want, _ = oracle.bfs(g, root)
                    emu = oracle.do_emulate(g, want, alpha, beta, policy=mode, coord_hi=nb)
                    ok_depth = np.array_equal(np.concatenate(full), want)
                    emu_steps = list(zip(emu["dir"].tolist(), emu["n_f"].tolist(), emu["discovered"].tolist(),
                                         emu["m_f"].tolist(), emu["m_u"].tolist(), emu["insp"].tolist()))
                    out.append((ok_depth, steps == emu_steps, sp))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_protocol_gloo():
    pkg.lib()   # the partition arithmetic comes from the built library
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for pr in ps:
        pr.join(timeout=60)
    for r in (0, 1):
        assert res[r], "no cases ran"
        for ok_depth, ok_steps, _ in res[r]:
            assert ok_depth and ok_steps
        assert sum(x[2] for x in res[r]) > 0, "the sparse (vertex-list) pull was never exercised"
