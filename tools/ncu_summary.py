"""Summarise an .ncu-rep (raw page) into the metrics we track; optional JSON out."""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1,
         "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if w.startswith("gpu__time"):
                    v = v * SCALE.get(u, 1)
                    w = "duration_ms"
                elif "bytes" in w:
                    v = v * SCALE.get(u, 1)
                d[w] = v
        res.append(d)
    return res


if __name__ == "__main__":
    rs = rows(sys.argv[1])
    for d in rs:
        rd = d.get("dram__bytes_read.sum", 0)
        wr = d.get("dram__bytes_write.sum", 0)
        ms = d.get("duration_ms", 0)
        print(f"{d['kernel'][:40]:40s} {ms:8.3f} ms  dram R {rd/1e9:6.3f} GB W {wr/1e9:6.3f} GB "
              f"= {(rd+wr)/ms/1e6 if ms else 0:7.1f} GB/s  L2hit {d.get('lts__t_sector_hit_rate.pct',0):5.1f}%  "
              f"warps {d.get('sm__warps_active.avg.pct_of_peak_sustained_active',0):5.1f}%  regs {d.get('launch__registers_per_thread',0):.0f}")
    if len(sys.argv) > 2:
        json.dump(rs, open(sys.argv[2], "w"), indent=1)
