"""DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), duration and grid of every
--set full capture in a directory -> JSON (the roofline.traffic figures of bench.py).
usage: python tools/ncu_traffic.py DIR SOURCE_NOTE > profiles/rNN/ncu_traffic.json"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "usecond": 1e3,
        "nsecond": 1.0, "msecond": 1e6}


def main(d, note=""):
    out = {"source": note, "unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)", "kernels": {}}
    for rep in sorted(glob.glob(os.path.join(d, "full_*.ncu-rep"))):
        k = os.path.basename(rep)[5:-8]
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) < 3:
            continue
        h, u, v = rows[0], rows[1], rows[2]

        def get(name):
            i = h.index(name)
            return float(v[i].replace(",", "")) * UNIT.get(u[i], 1.0)
        r, w = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        out["kernels"][k] = {"read": r, "write": w, "traffic": r + w, "duration_ns": get("gpu__time_duration.sum"),
                             "grid": int(get("launch__grid_size"))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
