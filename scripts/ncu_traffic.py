"""Read an `ncu --set full` report of the SpMM kernel and record its DRAM
traffic per launch into profiles/traffic.json under the given key.

    python scripts/ncu_traffic.py gpurun_out/prof.ncu-rep reddit_f602_p1_c1 [grid]

An optional third argument keeps only the launches whose grid size string
contains it (a report holding several SpMM widths).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, key = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = []
    gi = head.index("Grid Size")
    grid = sys.argv[3] if len(sys.argv) > 3 else None
    for v in vals:
        if grid and grid not in v[gi]:
            continue
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = head.index(k)
            b += float(v[i].replace(",", "")) * scale[units[i]]
        tot.append(b)
    path = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[key] = int(sum(tot) / len(tot))
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(key, data[key])


if __name__ == "__main__":
    main()
