"""Per-CUDA-source-line L2 sector counts (theoretical vs ideal) of one kernel launch.

    python tools/ncu_l2lines.py rep.ncu-rep k_bu_batch [launch_index] [top]
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
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
L2 = hdr.index("L2 Theoretical Sectors Global")
IDEAL = hdr.index("L2 Theoretical Sectors Global Ideal")
ST = hdr.index("Warp Stall Sampling (All Samples)")
res = []
for r in rows[hi + 1:]:
    if len(r) > L2 and r[0].isdigit():
        try:
            v = float(r[L2] or 0)
            st = float(r[ST] or 0)
        except ValueError:
            continue
        if v > 0 or st > 0:
            res.append((v, int(r[0]), r[1].strip()[:90], float(r[IDEAL] or 0), st))
tst = sum(x[4] for x in res) or 1
for v, ln, src, idl, st in sorted(res, reverse=True)[:top]:
    print(f"{v / 1e6:8.1f}M ideal {idl / 1e6:7.1f}M stall {100 * st / tst:5.1f}%  L{ln} {src}")
