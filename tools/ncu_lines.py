"""Per-CUDA-source-line warp-stall samples of one kernel launch from an .ncu-rep.

    python tools/ncu_lines.py rep.ncu-rep k_bu_batch [launch_index] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}", "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows:
    if r and r[0].isdigit() and len(r) > si and r[si].isdigit():
        lines.append((int(r[si]), int(r[0]), r[1].strip()))
tot = sum(x[0] for x in lines) or 1
for s, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  L{ln:<5d} {src[:110]}")
