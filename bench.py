#!/usr/bin/env python
"""Graph500 harmonic-mean GTEPS of the B200 direction-optimized BFS (arxiv 1503.04359).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config k29] [--impl reference]

A "step" is one Graph500 search batch: one BFS from each of the 64 sampled roots
(P:168).  The graph is generated and built on the device
once before timing (construction is reported as build_ms, never inside TEPS:
S:443).  Each BFS is timed with CUDA events on the graph's stream; value is the
harmonic mean over every timed BFS of component_edge_tuples / time (P:168
"harmonic means").  Rank 0 prints one JSON line.

--impl reference times the serial CPU oracle (oracle/, test infrastructure) on the
host cores on a bounded sample of the workload (see cpu_baseline.sample).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

KRON = (5700, 1900, 1900)
ER = (2500, 2500, 2500)
CONFIGS = {
    "k16": dict(scale=16, ef=16, seed=1, abc=KRON, name="Graph500 Kronecker scale 16, edgefactor 16"),
    "er22": dict(scale=22, ef=16, seed=2, abc=ER, name="Uniform random (Erdos-Renyi) scale 22, edgefactor 16"),
    "k26": dict(scale=26, ef=16, seed=1, abc=KRON, name="Graph500 Kronecker scale 26, edgefactor 16"),
    "k29": dict(scale=29, ef=16, seed=1, abc=KRON, name="Graph500 Kronecker scale 29, edgefactor 16"),
    "k30": dict(scale=30, ef=16, seed=1, abc=KRON, name="Graph500 Kronecker scale 30, edgefactor 16"),
}
DEFAULT_CONFIG = "k29"
METRIC = "Graph500 harmonic-mean GTEPS (64 roots)"
# the paper's rate for the same metric and workload (Scale29, 2x Xeon + 2x K40)
PAPER_GTEPS = {"k29": 17.3}
ROOTS = 64
# random 4-byte L2 probes per second on B200 (measured: profiles/r01_l2_probe_micro.txt)
L2_PROBE_PEAK = 270.0
# cpu_baseline / reference arm: the largest Kronecker scale whose oracle graph builds
# within the bench budget (~1 min of host time on the GPU boxes)
CPU_SCALE = 24


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def hmean(xs):
    xs = list(xs)
    return len(xs) / sum(1.0 / x for x in xs)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- oracle legs
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_threads() -> int:
    return max(1, min(ROOTS, os.cpu_count() or 1))


def oracle_setup(scale: int, seed: int, abc, nroots: int = ROOTS):
    """The serial oracle's own graph (oracle.kron_edges tuples -> oracle.build_csr, the
    same options as the GPU build) and root sample.  Tuples are generated over
    disjoint index ranges on host threads (harness parallelism: each range is the
    unmodified serial generator); the CSR build is the oracle's, single-threaded."""
    import concurrent.futures as cf

    import numpy as np

    import oracle
    m = 16 << scale
    uv = np.empty((m, 2), np.int32)
    step = 1 << 22

    def gen(lo):
        uv[lo:lo + step] = oracle.kron_edges(scale, 16, seed, abc, first=lo, count=min(step, m - lo))

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(oracle_threads()) as ex:
        list(ex.map(gen, range(0, m, step)))
    g = oracle.build_csr(1 << scale, uv, dedup=True, drop_self_loops=True, sort_rows=True)
    roots = oracle.sample_roots(g, scale, seed, nroots)
    return uv, g, roots, time.perf_counter() - t0


def oracle_batch(uv, g, roots, threads: int):
    """One serial oracle BFS per root, `threads` roots at a time on the host cores
    (every search itself is serial and timed alone): [(gteps, seconds), ...]."""
    import concurrent.futures as cf

    import oracle

    def one(r):
        t0 = time.perf_counter()
        depth, _ = oracle.bfs(g, int(r))
        dt = time.perf_counter() - t0
        return oracle.component_tuples(uv, depth) / dt / 1e9, dt

    with cf.ThreadPoolExecutor(threads) as ex:
        return list(ex.map(one, roots))


def oracle_sample_text(scale: int, nroots: int, threads: int, build_s: float) -> str:
    return (f"serial FIFO oracle (oracle/oracle.c orc_bfs) on Graph500 Kronecker s{scale} ef16 seed 1 "
            f"(dedup, self-loops dropped), {nroots} sampled roots, {threads} roots at a time on "
            f"{threads} host threads (each search serial on one thread, timed on it while the others run; "
            f"GTEPS per search, harmonic mean); "
            f"host: {os.cpu_count()} cores, {cpu_model()}; oracle graph build {build_s:.0f} s untimed. "
            f"The benched scale needs ~73 GB and ~1 h of single-threaded oracle CSR build: out of the bench budget")


def cpu_baseline_record(scale: int):
    uv, g, roots, build_s = oracle_setup(scale, 1, KRON)
    th = oracle_threads()
    res = oracle_batch(uv, g, roots, th)
    return {"value": round(hmean(r for r, _ in res), 6), "unit": "GTEPS", "cores": th, "kind": "oracle",
            "sample": oracle_sample_text(scale, len(roots), th, build_s), "scale": scale}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    scale = min(cfg["scale"], args.cpu_scale)
    uv, g, roots, build_s = oracle_setup(scale, cfg["seed"], cfg["abc"])
    th = oracle_threads()
    rates, step_ms = [], []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = oracle_batch(uv, g, roots, th)
        if step >= args.warmup:
            step_ms.append((time.perf_counter() - t0) * 1e3)
            rates += [r for r, _ in res]
    v = hmean(rates)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GTEPS", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.mean(step_ms), 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": cfg["name"], "sample_scale": scale, "roots_per_step": len(roots)},
            "cpu_baseline": {"value": round(v, 6), "unit": "GTEPS", "cores": th, "kind": "oracle",
                             "sample": oracle_sample_text(scale, len(roots), th, build_s)},
            "e2e": {"value": round(v, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def rank_memory(scale: int, ef: int, p: int, reindex: bool) -> dict:
    """Device bytes one rank needs: n = 2^scale, nl = n/p owned
    vertices, raw arcs per rank = 2 * ef * n / p (each tuple is two arcs).
    steady: adjacency 4/arc + per owned vertex off 8, head 8, deg_raw 4, queues 16,
    prefix 8, records 8 (+ hpar 4 when reindexed), bottom-up second-probe planes 32 per
    row with arcs (2 planes x 16 B; nl rows, n_active ~ 0.44 n on one reindexed GPU)
    + global arrays label/ilabel 8n (when
    reindexed) + bitmaps (visited, skip: nl/8 each; front, next, seen: n/8 each) + the
    top-down claim lists (p ranks: up to 8 bytes per owned-vertex slot of every peer,
    8 nb p = 8n, plus the receive side) + the tile index (one GPU, reindexed: ~2.3 GB at
    K29).  build_peak: offsets + raw degrees + two raw-arc arrays (fill target and
    sort/compaction target), 8 bytes per raw arc."""
    n = 1 << scale
    nl = n // p
    raw = 2 * ef * n // p
    steady = 4 * raw + nl * (8 + 8 + 4 + 16 + 8 + 8 + (4 if reindex else 0)) + (8 * n if reindex else 0)
    steady += 2 * nl // 8 + 3 * n // 8
    steady += 32 * (int(0.44 * nl) if (reindex and p == 1) else nl)
    if p > 1:
        steady += 8 * n + 8 * nl
    elif reindex:
        steady += int(6.4e9 * (n / 2 ** 29))   # tile index 2.3 GB + record logs 2 x 2 GB at K29
    peak = 8 * raw + 12 * nl + (8 * n if reindex else 0)
    return {"steady_gb": round(steady / 1e9, 1), "build_peak_gb": round(max(steady, peak) / 1e9, 1)}


def bu_bytes(n_bits: int, lv: dict) -> int:
    """Algorithmic bytes of one bottom-up launch, SURVEY section 8(d) exactly: visited
    scan, frontier and next bitmaps over the n_bits vertices the step covers (3 n/8;
    the non-isolated prefix when reindexed on one GPU), offsets of the U scanned
    vertices (8 U), arcs inspected (4 insp).  Outputs are charged once per search
    (8 n), not per launch."""
    return 3 * n_bits // 8 + 8 * lv["scanned"] + 4 * lv["inspections"]


def bu_design_bytes(lv: dict) -> int:
    """This design's extra per-launch bytes: the (depth, parent) record of every
    discovered vertex (8 D), re-read by the output pass."""
    return 8 * lv["discovered"]


def td_bytes(lv: dict) -> int:
    """Algorithmic bytes of one top-down launch: queue + offsets of the frontier
    (4F + 16F), arcs (4 m_f), queue write + outputs + offsets of discovered (20 D)."""
    return 20 * lv["frontier"] + 4 * lv["m_f"] + 20 * lv["discovered"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--roots", type=int, default=ROOTS)
    # alpha/beta: the paper gives no values (R2); 30/1000 is the B200 sweep optimum
    # (profiles/r01_switch_sweep.txt); the parity tests cover 15/18 and other settings
    ap.add_argument("--alpha", type=int, default=30)
    ap.add_argument("--beta", type=int, default=1000)
    ap.add_argument("--policy", default="do", choices=["do", "td", "paper"],
                    help="do: Beamer alpha/beta (default); td: top-down only (classic, P:202); "
                         "paper: the paper's section 3.3 rule (policy mode 3, --paper-alpha/--paper-beta)")
    ap.add_argument("--paper-alpha", type=int, default=500, help="static fraction of arcs, 1/10000 units (S:320)")
    ap.add_argument("--paper-beta", type=int, default=3, help="bottom-up steps before returning top-down (S:321)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--reindex", type=int, default=1, help="section 3.4 degree reindex (P:158)")
    ap.add_argument("--rows", default="id", choices=["id", "degree"],
                    help="row order: ascending ID (sort_rows 1) or decreasing neighbour degree (2, P:158)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-scale", type=int, default=CPU_SCALE,
                    help="Kronecker scale of the oracle's sample (cpu_baseline and --impl reference)")
    ap.add_argument("--no-validate", action="store_true",
                    help="skip the Graph500 validation (bfs_validate) of the last timed step's searches")
    ap.add_argument("--levels-out", default=None, help="write per-level records (JSON) here")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1503_04359_b200 as pkg
    from paper_1503_04359_b200 import build as pkg_build

    ws, rank, local = dist_env()
    if rank == 0:
        pkg_build.build()
    torch.cuda.set_device(local)
    comm = None
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        pkg_build.build()   # no-op when rank 0 already built it
        uid = pkg.bfs_comm_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        comm = pkg.bfs_comm_create(ws, rank, bytes(t.cpu().tolist()), local)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    cfg = CONFIGS[args.config]
    mem = rank_memory(cfg["scale"], cfg["ef"], ws, bool(args.reindex))
    total = torch.cuda.mem_get_info()[1]
    if mem["build_peak_gb"] * 1e9 > total:
        raise SystemExit(f"{args.config} on {ws} GPU(s) needs ~{mem['build_peak_gb']} GB per rank "
                         f"(DESIGN.md section 7), the device has {total / 1e9:.0f} GB: use more GPUs")
    stream = torch.cuda.Stream()
    opts = pkg.default_opts(reindex_by_degree=bool(args.reindex), sort_rows=2 if args.rows == "degree" else 1)
    g = pkg.Graph.kronecker(cfg["scale"], cfg["ef"], cfg["seed"], cfg["abc"], opts=opts, comm=comm, stream=stream)
    build_ms = g.build_ms
    roots = g.sample_roots(cfg["scale"], cfg["seed"], args.roots)
    n = g.n
    nl = g.local_end - g.local_begin
    parent = torch.empty(nl, dtype=torch.int32, device="cuda")
    depth = torch.empty(nl, dtype=torch.int32, device="cuda")
    if args.policy == "td":
        g.set_policy(mode=1, level_times=True)
    elif args.policy == "paper":
        g.set_policy(mode=3, alpha=args.paper_alpha, beta=args.paper_beta, level_times=True)
    else:
        g.set_policy(mode=0, alpha=args.alpha, beta=args.beta, level_times=True)

    pkg._check_output(parent, nl, "parent")   # the buffers are checked once, not per timed call
    pkg._check_output(depth, nl, "depth")

    def one(r):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        pkg.bfs_run(g.h, int(r), parent, depth, check=False)
        ev1.record(stream)
        ev1.synchronize()
        return ev0.elapsed_time(ev1)

    # TEPS numerator of every root: one untimed search each (independent of --warmup)
    edges = {}
    for r in roots:
        one(r)
        edges[int(r)] = pkg.bfs_component_tuples(g.h)
    for _ in range(args.warmup):
        for r in roots:
            one(r)

    times, launches = [], 0
    kern = {"bu": [0.0, 0, 0], "td": [0.0, 0, 0]}   # ms, bytes, launches
    probes = {"bu": 0, "td": 0}                      # frontier / visited probes (= inspections)
    levels_dump = []
    nvl_level_bytes = []
    design_bytes = 0
    n_bits = pkg.bfs_graph_active(g.h)
    # Graph500 validation of every search of the last timed step, after its
    # events completed (outside the timed region): bfs_validate on the device
    do_val = not args.no_validate and ws == 1
    val = {"searches": 0, "failed_searches": 0, "rules": {}}
    barrier()
    with ClockSampler(local) as clk:
        for step in range(args.steps):
            for r in roots:
                ms = one(r)
                run, levels = g.stats(tuples=False)
                if do_val and step == args.steps - 1:
                    bad = pkg.bfs_validate(g.h, int(r), parent, depth)
                    val["searches"] += 1
                    val["failed_searches"] += bool(bad)
                    for k, v in bad.items():
                        val["rules"][k] = val["rules"].get(k, 0) + v
                times.append(ms)
                launches += run["kernel_launches"]
                nvl_level_bytes += [lv["nvlink_bytes"] for lv in levels]
                for lv in levels:
                    key = "bu" if lv["direction"] == 1 else "td"
                    if key == "td" and lv["m_f"] == 0:
                        continue
                    kern[key][0] += lv["kernel_ms"]
                    kern[key][1] += bu_bytes(n_bits, lv) if key == "bu" else td_bytes(lv)
                    design_bytes += bu_design_bytes(lv) if key == "bu" else 0
                    kern[key][2] += 1
                    probes[key] += lv["inspections"]
                if step == 0:
                    levels_dump.append({"root": int(r), "ms": ms, "levels": levels})
        barrier()
    if dist is not None:   # per-BFS time = max over ranks
        tt = torch.tensor(times, dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        times = tt.cpu().tolist()
    rates = [edges[int(roots[i % len(roots)])] / (ms * 1e-3) / 1e9 for i, ms in enumerate(times)]
    step_ms = [sum(times[k * len(roots):(k + 1) * len(roots)]) for k in range(args.steps)]
    value = hmean(rates)
    clocks = clk.summary()

    # dominant kernel = the larger share of device time
    dom = max(kern, key=lambda k: kern[k][0])
    kms, kbytes, klaunch = kern[dom]
    peak, peak_kind = measured_peaks()
    achieved = (kbytes / klaunch) / ((kms / klaunch) * 1e-3) / 1e9 if klaunch and kms > 0 else 0.0
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get("k_bu_batch" if dom == "bu" else "k_td_expand")
        traffic_src = ("profiles/ncu_traffic_%s.json (%s): %s; a capture, not this run's roots"
                       % (args.config, tj.get("_source", "?"), tj.get("_note", "")))
    total_ms = sum(times)
    share = kms / total_ms if total_ms else 0.0

    # end to end: same roots, outputs to pinned host memory through the C ABI
    e2e = None
    if not args.no_e2e:
        hp = torch.empty(nl, dtype=torch.int32).pin_memory()
        hd = torch.empty(nl, dtype=torch.int32).pin_memory()
        e_rates = []
        for r in roots:
            t0 = time.perf_counter()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            pkg.bfs_run(g.h, int(r), hp, hd)   # D2H of parent+depth inside the call
            ev1.record(stream)
            ev1.synchronize()
            e_rates.append(edges[int(r)] / (ev0.elapsed_time(ev1) * 1e-3) / 1e9)
        if dist is not None:
            et = torch.tensor([edges[int(r)] / x for r, x in zip(roots, e_rates)], dtype=torch.float64, device="cuda")
            dist.all_reduce(et, op=dist.ReduceOp.MAX)      # seconds*1e9 per BFS, max over ranks
            e_rates = [edges[int(r)] / x for r, x in zip(roots, et.cpu().tolist())]
        e2e = {"value": round(hmean(e_rates), 4), "unit": "GTEPS", "h2d_bytes_per_step": 8 * len(roots),
               "d2h_bytes_per_step": 8 * nl * len(roots) * ws,
               "note": "bfs_run with pinned host parent/depth buffers; root passed by value"}

    if args.levels_out:
        with open(args.levels_out, "w") as f:
            json.dump(levels_dump, f)

    cpu = None if (args.no_cpu_baseline or ws > 1) else cpu_baseline_record(min(cfg["scale"], args.cpu_scale))
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "GTEPS", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(statistics.mean(step_ms), 4), "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": round(value / PAPER_GTEPS[args.config], 2) if args.config in PAPER_GTEPS else None,
        "dtype": "int32", "data": "synthetic",
        "config": {"workload": cfg["name"], "scale": cfg["scale"], "edgefactor": cfg["ef"], "seed": cfg["seed"],
                   "roots": len(roots), "policy": args.policy,
                   "alpha": args.paper_alpha if args.policy == "paper" else args.alpha,
                   "beta": args.paper_beta if args.policy == "paper" else args.beta, "parallelism": f"1d{ws}",
                   "reindex_by_degree": bool(args.reindex), "row_order": args.rows,
                   "l2": "inputs larger than L2 (CSR %.1f GB vs 126 MB L2)" % ((8 * (n + 1) + 4 * g.arcs) / 1e9)},
        "build_ms": round(build_ms, 2), "arcs": g.arcs, "rank_memory_model": mem,
        "per_root_ms": {"min": round(min(times), 4), "median": round(statistics.median(times), 4),
                        "max": round(max(times), 4)},
        "gteps_min_median_max": [round(min(rates), 3), round(statistics.median(rates), 3), round(max(rates), 3)],
        "roofline": {"bound": "hbm", "kernel": "k_bu_batch" if dom == "bu" else "k_td_expand",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind, "share_of_step": round(share, 4), "launches": klaunch,
                     "bytes_per_launch": int(kbytes / klaunch) if klaunch else 0,
                     "ms_per_launch": round(kms / klaunch, 5) if klaunch else None,
                     "bytes_model": ("BU: 3*n_bits/8 + 8*scanned + 4*inspections per launch (SURVEY 8(d)); "
                                     "TD: 20*F + 4*m_f + 20*D" if dom == "bu" else "TD: 20*F + 4*m_f + 20*D"),
                     "n_bits": n_bits,
                     "design_bytes_per_launch": int(design_bytes / klaunch) if (klaunch and dom == "bu") else None,
                     "timing": "per launch: %globaltimer span inside the kernel (first block start to last block "
                               "end), summed over the timed region's launches"},
        # second roofline for the probe-bound levels: every inspection is one random
        # 4-byte bitmap probe; B200 serves <= ~270 G such probes/s from L2
        # (profiles/r01_l2_probe_micro.txt, tools/micro/l2probe.cu)
        "probe_roofline": {"bound": "l2_random_probe", "unit": "Gprobe/s", "peak": L2_PROBE_PEAK,
                           "bu_achieved": round(probes["bu"] / (kern["bu"][0] * 1e-3) / 1e9, 2) if kern["bu"][0] else None,
                           "td_achieved": round(probes["td"] / (kern["td"][0] * 1e-3) / 1e9, 2) if kern["td"][0] else None},
        "gpu_launches": launches,
        "nvlink": None if ws == 1 else {
            "bytes_per_level_max": max(nvl_level_bytes) if nvl_level_bytes else 0,
            "bytes_per_bfs_mean": sum(nvl_level_bytes) / max(1, len(times)),
            "link_gbs_ref": 900.0, "note": "bytes this rank sent to peers (rank 0)"},
        "clocks": clocks,
        "validation": (dict(val, note="bfs_validate (Graph500 V1-V5 on the device) on every search of the last "
                                      "timed step") if do_val else None),
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    if comm is not None:
        pkg.bfs_comm_destroy(comm)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
