"""Turn a round-2 refresh run (tools/_r2_final3.sh, prefix g_) into the profiles/ files
the judge reads: bench line, other configs, launch-list summary, BU DRAM traffic,
GPU tests, smoke, per-level dump."""
import collections
import csv
import io
import json
import shutil
import sys

P = sys.argv[1] if len(sys.argv) > 1 else "g"
G = f"gpurun_out/{P}_"


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


shutil.copy(G + "gpu_tests.txt", "profiles/r02_gpu_tests.txt")
shutil.copy(G + "smoke.log", "profiles/r02_smoke.log")
shutil.copy(G + "levels.json", "profiles/r02_levels_k29_final.json")
open("profiles/r02_bench_k29.json", "w").write(open(G + "bench.json").read().strip().splitlines()[-1] + "\n")
with open("profiles/r02_other_configs.txt", "w") as f:
    f.write("# bench.py --config C --no-cpu-baseline --no-e2e on one B200, final round-2 code "
            "(same box as profiles/r02_bench_k29.json)\n")
    for c in ("k26", "er22", "k16"):
        x = last_json(G + f"bench_{c}.json")
        f.write(f"{c} {x['value']} GTEPS hmean; min/median/max {x['gteps_min_median_max']} ; per-root ms "
                f"{x['per_root_ms']} ; roofline frac {x['roofline']['frac']} ; build_ms {x['build_ms']}\n")
# launch list
rows = list(csv.reader(open(G + "launches.csv")))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
search = {"k_bu_batch", "k_emit_perm", "k_td_tile", "k_tile_rec", "k_td_finish", "k_b2q", "k_scan_dev",
          "k_mark_unreached", "k_td_chunk_starts", "k_init", "k_q2b", "k_tile_list", "k_td_small", "k_l2_demote"}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[start + 1:]:
    if len(r) <= max(ki, vi, ui):
        continue
    name = r[ki].split("(")[0].split("::")[-1]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
sel = {k: v for k, v in tot.items() if k in search or k.startswith("k_td_expand")}
all_ms = sum(sel.values())
with open("profiles/r02_launches_k29_summary.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none over `BFS_HOST_LOOP=1 python bench.py --steps 1 "
            "--warmup 0 --no-e2e --no-cpu-baseline --no-validate` (K29, reindex, alpha 30 / beta 1000; host loop: ncu "
            "cannot see kernels inside conditional graphs, the kernels are the same), final round-2 code.  Per-launch "
            "times are cold-cache and serialised: compare SHARES.  Raw list: profiles/r02_launches_k29.csv\n")
    f.write(f"# search kernels only (the capture also holds the graph build and the TEPS-numerator pass): "
            f"{sum(cnt[k] for k in sel)} launches, {all_ms:.1f} ms\n")
    f.write(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg ms':>9s}\n")
    for k, v in sorted(sel.items(), key=lambda x: -x[1]):
        f.write(f"{k[:34]:34s} {cnt[k]:8d} {v:10.3f} {100 * v / all_ms:6.2f}% {v / cnt[k]:9.4f}\n")
shutil.copy(G + "launches.csv", "profiles/r02_launches_k29.csv")
# BU traffic
lines = [ln for ln in open(G + "traffic.csv") if ln.startswith('"')]
rr = list(csv.reader(io.StringIO("".join(lines))))
h = rr[0]
mi, vv, ii = h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rr[1:]:
    d.setdefault(r[ii], {})[r[mi]] = float(r[vv].replace(",", ""))
b = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in d.values()]
json.dump({"k_bu_batch": int(sum(b) / len(b)),
           "_source": "r02_bu_traffic_final.csv (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k k_bu_batch)",
           "_note": f"mean DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per k_bu_batch launch over the 8 "
                    f"first sampled K29 roots ({len(b)} launches; host loop, cold-cache ncu replay; final round-2 code)"},
          open("profiles/ncu_traffic_k29.json", "w"), indent=1)
shutil.copy(G + "traffic.csv", "profiles/r02_bu_traffic_final.csv")
x = last_json(G + "bench.json")
print(x["value"], x["gteps_min_median_max"], x["e2e"]["value"], x["roofline"]["frac"], x["clocks"])
print(open("profiles/r02_other_configs.txt").read())
print(open("profiles/r02_launches_k29_summary.txt").read()[-900:])
