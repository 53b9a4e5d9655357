"""Per-launch time and DRAM bytes from an `ncu --csv --log-file` metrics list
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum).

    python tools/ncu_csv_kernels.py gpurun_out/x.csv [min_ms]
"""
import csv
import io
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
min_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
rows = list(csv.reader(io.StringIO("".join(lines))))
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = {}
for r in rows[1:]:
    e = d.setdefault(r[ii], {"kernel": r[ki].split("(")[0].replace("(anonymous namespace)::", "")})
    e[r[mi]] = float(r[vi].replace(",", ""))
for k, m in d.items():
    t = m.get("gpu__time_duration.sum", 0) / 1e6
    rd = m.get("dram__bytes_read.sum", 0) / 1e9
    wr = m.get("dram__bytes_write.sum", 0) / 1e9
    if t >= min_ms:
        print(f"{k:>5} {m['kernel'][-40:]:>40} {t:8.3f} ms  R {rd:6.2f} GB  W {wr:5.2f} GB  {(rd + wr) / t * 1e3:6.0f} GB/s")
