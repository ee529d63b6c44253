#!/usr/bin/env python3
"""Print an ncu --csv launch list as one line per launch: kernel, µs, DRAM GB read/write, GB/s."""
import csv
import sys
from collections import OrderedDict


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    launches = OrderedDict()
    for r in rows:
        key = r["ID"]
        d = launches.setdefault(key, {"name": r["Kernel Name"][:70]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r["Metric Name"]] = v * scale
    return list(launches.values())


if __name__ == "__main__":
    print(sys.argv[1])
    for d in load(sys.argv[1]):
        t = d.get("gpu__time_duration.sum", 0)
        rd = d.get("dram__bytes_read.sum", 0)
        wr = d.get("dram__bytes_write.sum", 0)
        bw = (rd + wr) / (t * 1e-6) / 1e9 if t else 0
        print(f"  {t:10.1f} us  rd {rd/1e9:7.3f} GB  wr {wr/1e9:7.3f} GB  {bw:7.0f} GB/s  {d['name']}")
