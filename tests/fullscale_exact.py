"""Exact full-size parity in bench.py's launch configuration (TEST INFRASTRUCTURE).

Two checks, each independent of the CUDA path except for the outputs under test:

  serial_oracle_check   K26-sized graphs: the serial FIFO oracle (oracle.bfs) runs on its
                        own CSR (oracle.build_csr over oracle.kron_edges tuples) for every
                        root; depths must be bit-identical to the GPU's, and the GPU's
                        parents must pass the CSR validator (oracle.validate, V1-V6).
  streaming_check       any size (K29): the streaming validator (oracle.stream_validate_*,
                        SURVEY section 8(c4)) checks V1-V5 of every search against every
                        regenerated input tuple; by the theorem in oracle.c (V1-V5 =>
                        depth = hop distance) this makes the depths exact.

The GPU graph is built exactly as bench.py builds it (Kronecker, dedup, self-loops
dropped, degree reindex, alpha 30 / beta 1000, device-driven loop), outputs in
ORIGINAL labels through the C ABI.  Host threads only run the serial oracle on
disjoint pieces of work (tests/stream_harness.py).
"""
from __future__ import annotations

import concurrent.futures as cf
import time

import numpy as np

import oracle
from tests import stream_harness as H

BENCH_POLICY = dict(mode=0, alpha=30, beta=1000)


def gpu_graph(pkg, scale, ef, seed, abc):
    g = pkg.Graph.kronecker(scale, ef, seed, abc, opts=pkg.default_opts(reindex_by_degree=True))
    g.set_policy(**BENCH_POLICY)
    return g


def serial_oracle_check(pkg, torch, scale, ef, seed, abc, nroots=64, threads=None, log=print) -> dict:
    """Every root: GPU depth == serial oracle depth (bit-exact) and GPU parents valid."""
    threads = threads or H.host_threads()
    n = 1 << scale
    t0 = time.time()
    g = gpu_graph(pkg, scale, ef, seed, abc)
    roots = g.sample_roots(scale, seed, nroots)
    dh = torch.empty(n, dtype=torch.int32).pin_memory()
    ph = torch.empty(n, dtype=torch.int32).pin_memory()
    outs = []
    for r in roots:
        pkg.bfs_run(g.h, int(r), ph, dh)
        outs.append((dh.numpy().copy(), ph.numpy().copy()))
    g.close()
    del dh, ph
    torch.cuda.empty_cache()
    t_gpu = time.time() - t0
    uv = H.generate_edges(scale, ef, seed, abc, threads=threads)
    ref = oracle.build_csr(n, uv)          # every tuple as two arcs: the input edge set itself
    oracle_roots = oracle.sample_roots(ref, scale, seed, nroots)
    del uv
    t_oracle_build = time.time() - t0 - t_gpu
    assert np.array_equal(oracle_roots, roots), "root samples differ"

    def one(k):
        r = int(roots[k])
        want, _ = oracle.bfs(ref, r)
        d, p = outs[k]
        same = bool(np.array_equal(d, want))
        bad = oracle.validate(ref, r, d, p, ref_depth=want)
        return r, same, bad, int((want >= 0).sum()), int(want.max())

    res = []
    with cf.ThreadPoolExecutor(threads) as ex:
        for r, same, bad, reached, levels in ex.map(one, range(len(roots))):
            res.append({"root": r, "depth_equal": same, "fails": {k: list(v) for k, v in bad.items()},
                        "reached": reached, "max_depth": levels})
    out = {"scale": scale, "edgefactor": ef, "seed": seed, "roots": len(roots), "arcs_oracle": int(ref.arcs),
           "gpu_s": round(t_gpu, 1), "oracle_build_s": round(t_oracle_build, 1),
           "check_s": round(time.time() - t0 - t_gpu - t_oracle_build, 1), "threads": threads,
           "depth_equal_all": all(x["depth_equal"] for x in res),
           "validator_failures": sum(sum(v[0] for v in x["fails"].values()) for x in res), "per_root": res}
    log(f"serial oracle check s{scale}: {len(roots)} roots, depth equal {out['depth_equal_all']}, "
        f"validator failures {out['validator_failures']} (gpu {t_gpu:.0f}s, oracle build {t_oracle_build:.0f}s, "
        f"checks {out['check_s']:.0f}s)")
    return out


def streaming_check(pkg, torch, scale, ef, seed, abc, nroots=8, group=8, threads=None, store_edges=None,
                    log=print) -> dict:
    """V1-V5 of nroots searches over all ef * 2^scale regenerated tuples, `group` searches
    per pass.  Outputs are packed vertex-major ([n, group]) on the device."""
    threads = threads or H.host_threads()
    n = 1 << scale
    m = ef << scale
    t0 = time.time()
    g = gpu_graph(pkg, scale, ef, seed, abc)
    roots = g.sample_roots(scale, seed, nroots)
    ngroups = (len(roots) + group - 1) // group
    if store_edges is None:
        store_edges = ngroups > 1
    uv = H.generate_edges(scale, ef, seed, abc, threads=threads) if store_edges else None
    t_gen = time.time() - t0
    dd = torch.empty(n, dtype=torch.int32, device="cuda")
    pd = torch.empty(n, dtype=torch.int32, device="cuda")
    per_root = []
    t_val = 0.0
    for gi in range(ngroups):
        rs = roots[gi * group:(gi + 1) * group]
        R = len(rs)
        d8 = torch.empty((n, R), dtype=torch.int8, device="cuda")
        p32 = torch.empty((n, R), dtype=torch.int32, device="cuda")
        maxd = []
        for j, r in enumerate(rs):
            pkg.bfs_run(g.h, int(r), pd, dd)
            maxd.append(int(dd.max().item()))
            assert maxd[-1] < 127, "depth does not fit the int8 layout"
            d8[:, j] = dd.to(torch.int8)
            p32[:, j] = pd
        d8h = d8.cpu().numpy()
        p32h = p32.cpu().numpy()
        del d8, p32
        torch.cuda.empty_cache()
        t1 = time.time()
        res = H.validate(n, np.asarray(rs, np.int64), d8h, p32h, uv=uv,
                         gen=None if store_edges else (scale, ef, seed, abc), threads=threads)
        t_val += time.time() - t1
        for j, r in enumerate(rs):
            reached = int((d8h[:, j] >= 0).sum())
            per_root.append({"root": int(r), "fails": {k: list(v) for k, v in H.failing_rules(res, j).items()},
                             "reached": reached, "max_depth": maxd[j]})
        del d8h, p32h
        log(f"streaming group {gi + 1}/{ngroups}: {R} roots, failures "
            f"{sum(sum(v[0] for v in x['fails'].values()) for x in per_root[-R:])}")
    g.close()
    del dd, pd
    torch.cuda.empty_cache()
    out = {"scale": scale, "edgefactor": ef, "seed": seed, "roots": len(roots), "tuples_checked": m,
           "tuples_checked_total": m * len(roots), "store_edges": bool(store_edges), "group": group,
           "threads": threads, "gen_s": round(t_gen, 1), "validate_s": round(t_val, 1),
           "failures": sum(sum(v[0] for v in x["fails"].values()) for x in per_root), "per_root": per_root}
    log(f"streaming check s{scale}: {len(roots)} roots x {m} tuples, failures {out['failures']} "
        f"(gen {t_gen:.0f}s, validate {t_val:.0f}s)")
    return out
