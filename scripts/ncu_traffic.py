#!/usr/bin/env python3
"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of each
kernel class from an `ncu --set full` report, written to profiles/traffic.json with
the hash of the library sources it was captured on (bench.py reports it only for
matching sources).

    python scripts/ncu_traffic.py gpurun_out/prof_X.ncu-rep [--capture "how it was taken"]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import source_hash  # noqa: E402

CLASSES = {"k1": ("k1_gather",), "k2": ("k2_ct", "k2_cl", "k2_prime", "k2a_split", "k2b_split"),
           "k3": ("k3_identify", "k3_clw")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--capture", default="")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "traffic.json"))
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    rd = hdr.index("dram__bytes_read.sum")
    wr = hdr.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = {}
    for r in rows[2:]:
        name = r[ki]
        cls = next((c for c, pre in CLASSES.items() if any(p in name for p in pre)), None)
        if cls is None:
            continue
        b = (float(r[rd].replace(",", "")) * scale.get(units[rd], 1.0) +
             float(r[wr].replace(",", "")) * scale.get(units[wr], 1.0))
        acc.setdefault(cls, []).append((name.split("(")[0], b))
    out = {"source_hash": source_hash(), "capture": a.capture or a.report, "kernels": {}}
    for cls, v in acc.items():
        out["kernels"][cls] = {"dram_bytes_per_launch": sum(b for _, b in v) / len(v), "launches": len(v),
                               "per_launch": [{"kernel": n, "bytes": b} for n, b in v]}
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: v["dram_bytes_per_launch"] for k, v in out["kernels"].items()}))


if __name__ == "__main__":
    main()
