#!/usr/bin/env python
"""Write profiles/r02_traffic.json from ncu --set full captures (run here on gpurun's files):
dram__bytes_read.sum + dram__bytes_write.sum per launch of the captured kernel, which bench.py
reports as roofline.traffic for the matching config.

    python tools/traffic_json.py k8=gpurun_out/f02/k8.ncu-rep:c4 persistent=gpurun_out/f02/kp.ncu-rep:c2
"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, val = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        tot += float(val[i].replace(",", "")) * UNIT[units[i]]
    return tot, val[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""


def main():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", "r02_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[1:]:
        key, rest = arg.split("=", 1)
        rep, cfg = rest.rsplit(":", 1)
        b, name = dram_bytes(rep)
        data[key] = {"bytes_per_launch": b, "config": cfg, "kernel": name,
                     "source": f"ncu --set full, {os.path.basename(rep)} ({cfg}), dram read + write"}
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
