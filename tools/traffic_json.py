"""Build profiles/traffic.json (bench.py's roofline.traffic) from the committed ncu launch lists.

usage: python tools/traffic_json.py BENCH_JSON LAUNCH_PREFIX > profiles/traffic.json

LAUNCH_PREFIX_<config>.csv are `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` lists of `bench.py --configs none --config <config>` (tools/gpu/r02_final_evidence.sh). The last step's
passes are the last P launches (P = len(pass_ms) in the bench record); the dominant pass is the one whose
CUDA-event time in the bench record is largest. Bytes are dram__bytes_read.sum + dram__bytes_write.sum.
"""
import csv
import io
import json
import sys


def launches(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = {}
    for r in csv.DictReader(io.StringIO(txt)):
        d = rows.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"].split("(")[0]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return [rows[k] for k in sorted(rows)]


def main():
    bench = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    prefix = sys.argv[2]
    recs = {"batched1024": bench, **bench.get("configs", {})}
    out = {"_source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none (" + prefix + "_*.csv, tools/gpu/r02_final_evidence.sh, "
                      "tools/traffic_json.py); per launch: dominant = the pass bench.py's pass_ms names slowest, "
                      "step = the sum over one step's passes (bytes)"}
    for name, rec in recs.items():
        pm = (rec.get("roofline") or {}).get("pass_ms")
        if not pm:
            continue
        try:
            ls = launches(f"{prefix}_{name}.csv")
        except (OSError, ValueError):
            continue
        step = ls[-len(pm):]
        b = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in step]
        dom = max(range(len(pm)), key=lambda i: pm[i])
        out[name] = {"dominant": int(b[dom]), "dominant_kernel": step[dom]["kernel"], "step": int(sum(b))}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
