"""Summarise a bench --levels-out dump: per-BFS time split and the slowest roots.

    python tools/levels_summary.py gpurun_out/levels_ab.json [top]
"""
import json
import sys

L = json.load(open(sys.argv[1]))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n = len(L)
tot = sum(r["ms"] for r in L)
lv = sum(lv["ms"] for r in L for lv in r["levels"])
bu = sum(lv["kernel_ms"] for r in L for lv in r["levels"] if lv["direction"] == 1)
td = sum(lv["kernel_ms"] for r in L for lv in r["levels"] if lv["direction"] == 0)
print(f"per BFS ms: total {tot / n:.3f}  levels {lv / n:.3f}  bu {bu / n:.3f}  td {td / n:.3f}  "
      f"level overhead {(lv - bu - td) / n:.3f}  init+emit {(tot - lv) / n:.3f}")
L.sort(key=lambda r: -r["ms"])
for r in L[:top] + L[-2:]:
    print(r["root"], round(r["ms"], 2), " ".join(("B" if x["direction"] else "T") + "%d:%.2f" % (x["frontier"], x["kernel_ms"])
                                              for x in r["levels"]))
