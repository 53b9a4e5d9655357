"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel
launch count, total time and share (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[start + 1:]:
    if len(r) <= max(ki, vi, ui):
        continue
    name = r[ki].split("(")[0].split("::")[-1]
    if "<" in r[ki].split("(")[0]:
        name = r[ki].split("(")[0].split("::")[-1]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"# {sys.argv[1]}: {sum(cnt.values())} launches, {all_ms:.1f} ms total")
print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg ms':>9s}")
for k, v in tot.most_common():
    print(f"{k[:40]:40s} {cnt[k]:8d} {v:10.3f} {100*v/all_ms:6.2f}% {v/cnt[k]:9.4f}")
