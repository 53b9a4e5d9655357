"""world_size-2 gloo tests on CPU for the N>1 path's host logic.

Each rank takes its vertex range from the library's own partition arithmetic
(bfs_partition_range, host-only) and runs the partitioned protocol the GPU path
uses -- TD: per-owner (vertex, parent) claim lists, an allgather of the p x p claim
counts, the claims exchanged point to point and merged by the owner (Alg. 2), or on
dense levels (global m_f >= bitmap_min) per-peer outbox bitmaps ORed by the owner with
the parents sent as (vertex, parent, level) logs after the last level; BU:
allgather of the next-frontier slices (Alg. 3); an allreduce of the switch counters
so that every rank picks the same direction -- with numpy standing in for the
kernels and gloo for NCCL.  Depth must equal the oracle's, the parents must
validate, and the per-step counters must equal the emulator's, on both ranks.
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


def _exchange(out, p, rank, width):
    """point-to-point exchange of per-peer int64 arrays (rows of `width` values) after an
    allgather of the p x p counts; returns the received arrays per sender"""
    counts = torch.tensor([len(o) for o in out], dtype=torch.int64)
    mat = [torch.zeros(p, dtype=torch.int64) for _ in range(p)]
    dist.all_gather(mat, counts)
    recv = [torch.zeros((int(mat[q][rank]), width), dtype=torch.int64) for q in range(p)]
    reqs = []
    for q in range(p):
        if q == rank:
            continue
        if len(out[q]):
            reqs.append(dist.isend(torch.tensor(out[q], dtype=torch.int64).reshape(-1, width), q))
        if recv[q].numel():
            reqs.append(dist.irecv(recv[q], q))
    for r in reqs:
        r.wait()
    return recv


def _partitioned_bfs(ref, root, lo, hi, nb, p, rank, alpha=15, beta=18, mode=0, bitmap_min=None):
    n = ref.n
    deg = ref.degree()
    visited = np.zeros(hi - lo, bool)
    visited[deg[lo:hi] == 0] = True            # skip mask
    depth = np.full(hi - lo, -1, np.int64)
    parent = np.full(hi - lo, -1, np.int64)
    seen = np.zeros(n, bool)                  # remote claims already sent
    plog = [[] for _ in range(p)]             # bitmap pushes: (v, parent, level) per owner
    bitmap_levels = 0
    queue = []
    if lo <= root < hi:
        visited[root - lo] = True
        depth[root - lo] = 0
        parent[root - lo] = root
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
            bitmap = bitmap_min is not None and m_f >= bitmap_min   # same global m_f on every rank
            out = [[] for _ in range(p)]
            outbox = np.zeros(p * nb, bool)
            for u in queue:
                for v in ref.row(u):
                    insp += 1
                    if lo <= v < hi:
                        if not visited[v - lo]:
                            visited[v - lo] = True
                            depth[v - lo] = d + 1
                            parent[v - lo] = u
                            nxt.append(int(v))
                    elif not seen[v]:
                        seen[v] = True
                        if bitmap:
                            outbox[v] = True
                            plog[v // nb].append((int(v), int(u), d + 1))
                        else:
                            out[v // nb].append((int(v), int(u)))
            if bitmap:
                bitmap_levels += 1
                # slice q of the outbox to rank q (point to point; gloo has no all_to_all)
                parts = [torch.zeros(nb, dtype=torch.uint8) for _ in range(p)]
                reqs = []
                for q in range(p):
                    if q != rank:
                        reqs.append(dist.isend(torch.from_numpy(outbox[q * nb:(q + 1) * nb].astype(np.uint8)), q))
                        reqs.append(dist.irecv(parts[q], q))
                for r in reqs:
                    r.wait()
                got_bits = np.zeros(nb, bool)
                for q in range(p):
                    if q != rank:
                        got_bits |= parts[q].numpy().astype(bool)
                for vl in np.nonzero(got_bits[:hi - lo] & ~visited)[0]:   # owner OR; parent pending
                    visited[vl] = True
                    depth[vl] = d + 1
                    nxt.append(int(lo + vl))
            else:
                recv = _exchange(out, p, rank, 2)
                for q in range(p):
                    for v, u in recv[q].tolist():              # owner merge
                        if not visited[v - lo]:
                            visited[v - lo] = True
                            depth[v - lo] = d + 1
                            parent[v - lo] = u
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
                        parent[vl] = u
                        break
            for v in nxt:
                visited[v - lo] = True
        got = allreduce([len(nxt), int(sum(deg[v] for v in nxt)), insp, coord(nxt)])
        steps.append((direction, n_f, got[0], m_f, m_u, got[2] if direction else m_f))
        prev, n_f, m_f, m_fc = n_f, got[0], got[1], got[3]
        queue = nxt
        d += 1
    # final aggregation: the parent logs of the bitmap pushes to their owners; a log
    # entry is a parent iff its level is the vertex's depth
    recv = _exchange(plog, p, rank, 3)
    for q in range(p):
        for v, u, lvl in recv[q].tolist():
            if depth[v - lo] == lvl and parent[v - lo] == -1:
                parent[v - lo] = u
    return depth, parent, steps, sparse_pulls[0], bitmap_levels


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
                for mode, alpha, beta, bmin in ((0, 15, 18, None), (1, 15, 18, None), (3, 500, 2, None),
                                                (3, 40, 3, None), (1, 15, 18, 1), (0, 15, 18, 40)):
                    depth, parent, steps, sp, bl = _partitioned_bfs(g, root, lo, hi, nb, world, rank, alpha, beta,
                                                                    mode, bmin)
                    full = [None] * world
                    dist.all_gather_object(full, (depth.tolist(), parent.tolist()))
                    want, _ = oracle.bfs(g, root)
                    emu = oracle.do_emulate(g, want, alpha, beta, policy=mode, coord_hi=nb)
                    d_all = np.concatenate([np.asarray(x[0]) for x in full])
                    p_all = np.concatenate([np.asarray(x[1]) for x in full]).astype(np.int32)
                    ok_depth = np.array_equal(d_all, want) and not oracle.validate(g, root, d_all.astype(np.int32),
                                                                                   p_all, ref_depth=want)
                    emu_steps = list(zip(emu["dir"].tolist(), emu["n_f"].tolist(), emu["discovered"].tolist(),
                                         emu["m_f"].tolist(), emu["m_u"].tolist(), emu["insp"].tolist()))
                    out.append((ok_depth, steps == emu_steps, sp, bl))
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
        for ok_depth, ok_steps, _, _ in res[r]:
            assert ok_depth and ok_steps
        assert sum(x[2] for x in res[r]) > 0, "the sparse (vertex-list) pull was never exercised"
        assert sum(x[3] for x in res[r]) > 0, "the bitmap push was never exercised"
