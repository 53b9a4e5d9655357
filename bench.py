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
# cpu_baseline / reference arm sample: the oracle cannot build s26+ within the bench budget
SAMPLE_SCALE = 20


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
def oracle_sample(budget_s: float, roots_max: int = ROOTS, seed: int = 1):
    """Serial oracle BFS on the bounded sample graph: list of (gteps, seconds) per root."""
    import oracle
    uv, g = oracle.kron_graph(SAMPLE_SCALE, 16, seed)
    roots = oracle.sample_roots(g, SAMPLE_SCALE, seed, roots_max)
    out = []
    t_all = time.perf_counter()
    for r in roots:
        t0 = time.perf_counter()
        depth, _ = oracle.bfs(g, int(r))
        dt = time.perf_counter() - t0
        e = oracle.component_tuples(uv, depth)
        out.append((e / dt / 1e9, dt))
        if time.perf_counter() - t_all > budget_s:
            break
    return out, (uv, g, roots)


def cpu_baseline_record(budget_s: float = 15.0):
    res, _ = oracle_sample(budget_s)
    return {"value": round(hmean(r for r, _ in res), 6), "unit": "GTEPS", "cores": 1, "kind": "oracle",
            "sample": f"serial FIFO oracle (oracle/oracle.c, 1 thread) on Graph500 Kronecker s{SAMPLE_SCALE} ef16 "
                      f"seed 1, {len(res)} roots, harmonic mean; the oracle cannot build the s26+ CSR within the "
                      f"bench budget (s29 needs 68 GiB host RAM and ~1 h of single-core generation)"}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    import oracle
    t0 = time.perf_counter()
    uv, g = oracle.kron_graph(SAMPLE_SCALE, 16, 1)
    build_s = time.perf_counter() - t0
    roots = oracle.sample_roots(g, SAMPLE_SCALE, 1, ROOTS)
    per_step = max(1, min(ROOTS, int(150.0 / max(1, args.steps + args.warmup) / 0.35)))
    rates, step_ms = [], []
    ri = 0
    for step in range(args.warmup + args.steps):
        t_step = 0.0
        for _ in range(per_step):
            r = int(roots[ri % len(roots)])
            ri += 1
            t1 = time.perf_counter()
            depth, _ = oracle.bfs(g, r)
            dt = time.perf_counter() - t1
            t_step += dt
            if step >= args.warmup:
                rates.append(oracle.component_tuples(uv, depth) / dt / 1e9)
        if step >= args.warmup:
            step_ms.append(t_step * 1e3)
    v = hmean(rates)
    sample = (f"serial FIFO oracle (1 thread) on Graph500 Kronecker s{SAMPLE_SCALE} ef16 seed 1 ({per_step} roots "
              f"per step, oracle CSR build {build_s:.1f} s untimed); the {cfg['name']} CSR is out of reach of the "
              f"serial oracle within the bench budget")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GTEPS", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.mean(step_ms), 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": cfg["name"], "sample_scale": SAMPLE_SCALE,
                                            "roots_per_step": per_step},
            "cpu_baseline": {"value": round(v, 6), "unit": "GTEPS", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def bu_bytes(n_global: int, lv: dict) -> int:
    """Algorithmic bytes of one bottom-up launch: visited scan,
    frontier and next bitmaps (3 n/8), offsets of scanned vertices (8 U), arcs
    inspected (4 insp), outputs of discovered vertices (8 D)."""
    return 3 * n_global // 8 + 8 * lv["scanned"] + 4 * lv["inspections"] + 8 * lv["discovered"]


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

    def one(r):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        pkg.bfs_run(g.h, int(r), parent, depth)
        ev1.record(stream)
        ev1.synchronize()
        return ev0.elapsed_time(ev1)

    # warm-up: also caches the TEPS numerator per root (outside the timed region)
    edges = {}
    for _ in range(args.warmup):
        for r in roots:
            one(r)
            if int(r) not in edges:
                edges[int(r)] = pkg.bfs_component_tuples(g.h)

    times, launches = [], 0
    kern = {"bu": [0.0, 0, 0], "td": [0.0, 0, 0]}   # ms, bytes, launches
    probes = {"bu": 0, "td": 0}                      # frontier / visited probes (= inspections)
    levels_dump = []
    nvl_level_bytes = []
    barrier()
    with ClockSampler(local) as clk:
        for step in range(args.steps):
            for r in roots:
                ms = one(r)
                run, levels = g.stats(tuples=False)
                times.append(ms)
                launches += run["kernel_launches"]
                nvl_level_bytes += [lv["nvlink_bytes"] for lv in levels]
                for lv in levels:
                    key = "bu" if lv["direction"] == 1 else "td"
                    if key == "td" and lv["m_f"] == 0:
                        continue
                    kern[key][0] += lv["kernel_ms"]
                    kern[key][1] += bu_bytes(n, lv) if key == "bu" else td_bytes(lv)
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
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("k_bu_batch" if dom == "bu" else "k_td_expand")
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

    cpu = None if (args.no_cpu_baseline or ws > 1) else cpu_baseline_record()
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
        "build_ms": round(build_ms, 2), "arcs": g.arcs,
        "per_root_ms": {"min": round(min(times), 4), "median": round(statistics.median(times), 4),
                        "max": round(max(times), 4)},
        "gteps_min_median_max": [round(min(rates), 3), round(statistics.median(rates), 3), round(max(rates), 3)],
        "roofline": {"bound": "hbm", "kernel": "k_bu_batch" if dom == "bu" else "k_td_expand",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                     "share_of_step": round(share, 4), "launches": klaunch,
                     "bytes_per_launch": int(kbytes / klaunch) if klaunch else 0},
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
