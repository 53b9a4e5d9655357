"""Average DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) per
kernel from one `ncu --set full` capture -> JSON read by bench.py as roofline.traffic.

    python tools/traffic_from_ncu.py gpurun_out/r01_full_k29.ncu-rep profiles/ncu_traffic_k29.json
"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import rows  # noqa: E402

acc = collections.defaultdict(list)
for d in rows(sys.argv[1]):
    name = d["kernel"].split("(")[0].split("::")[-1].split("<")[0]
    acc[name].append(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0))
out = {k: int(sum(v) / len(v)) for k, v in acc.items()}
out["_source"] = os.path.basename(sys.argv[1])
out["_note"] = "mean DRAM bytes per captured launch (one root, cold-cache ncu replay)"
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(out)
