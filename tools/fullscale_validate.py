"""Exact full-size validation of the bench configuration, recorded as JSON.

    python tools/fullscale_validate.py --k26-roots 64 --k29-roots 64 --out profiles/r02_fullscale_validation.json

K26: serial oracle depths vs the GPU's (bit-exact) + CSR validator on the GPU parents.
K29: streaming validator (V1-V5 over every regenerated tuple) on the GPU outputs.
Test infrastructure only (tests/fullscale_exact.py); the product path never runs this.
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1503_04359_b200 as pkg  # noqa: E402
from paper_1503_04359_b200 import build as pkg_build  # noqa: E402
from tests import fullscale_exact as FX  # noqa: E402
from tests import stream_harness as H  # noqa: E402


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


ap = argparse.ArgumentParser()
ap.add_argument("--k26-roots", type=int, default=64)
ap.add_argument("--k29-roots", type=int, default=64)
ap.add_argument("--group", type=int, default=8)
ap.add_argument("--out", default="gpurun_out/fullscale_validation.json")
a = ap.parse_args()
pkg_build.build()
oracle.build_library()
torch.cuda.set_device(0)
rec = {"when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "host_threads": H.host_threads(),
       "cpu": cpu_model(), "gpu": torch.cuda.get_device_name(0),
       "config": "Kronecker ef16 seed 1, dedup, self-loops dropped, degree reindex, alpha 30 / beta 1000 "
                 "(bench.py launch configuration), outputs in original labels through the C ABI"}


def save():
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(rec, f, indent=1)


if a.k26_roots:
    rec["k26_serial_oracle"] = FX.serial_oracle_check(pkg, torch, 26, 16, 1, oracle.KRON_ABC, nroots=a.k26_roots)
    save()
if a.k29_roots:
    rec["k29_streaming"] = FX.streaming_check(pkg, torch, 29, 16, 1, oracle.KRON_ABC, nroots=a.k29_roots,
                                              group=a.group)
    save()
print(json.dumps({k: ({kk: vv for kk, vv in v.items() if kk != "per_root"} if isinstance(v, dict) else v)
                  for k, v in rec.items()}))
