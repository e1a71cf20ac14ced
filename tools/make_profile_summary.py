#!/usr/bin/env python
"""Condense ncu outputs into profiles/ (committed evidence).

    python tools/make_profile_summary.py --launches gpurun_out/launches.csv \
        --full sjlt_apply_S=gpurun_out/prof_bench_sjlt.ncu-rep \
        --full gauss_S=gpurun_out/prof_bench_gauss.ncu-rep --tag r01
"""
import argparse
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and r[0].isdigit()]
    by = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0]
        ns = float(r[-1].replace(",", ""))
        ent = by.setdefault(name, {"launches": 0, "total_ms": 0.0})
        ent["launches"] += 1
        ent["total_ms"] += ns / 1e6
    total = sum(v["total_ms"] for v in by.values())
    for v in by.values():
        v["share"] = v["total_ms"] / total if total else 0.0
        v["avg_ms"] = v["total_ms"] / v["launches"]
    return by, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--command", default="python bench.py --steps 2 --warmup 3")
    ap.add_argument("--full", action="append", default=[])
    ap.add_argument("--tag", default="r01")
    args = ap.parse_args()
    out = {"tag": args.tag, "kernels": {}}
    if args.launches:
        by, total = launches(args.launches)
        out["launch_list"] = {"source": os.path.basename(args.launches),
                              "command": args.command,
                              "note": "ncu --metrics gpu__time_duration.sum --clock-control none "
                                      "(cold-cache, serialised: compare shares)",
                              "total_ms": total, "kernels": by}
    for spec in args.full:
        key, path = spec.split("=", 1)
        k = ncu_summary.summarise(path)[0]

        def num(s):
            return float(str(s).split()[0].replace(",", ""))
        rd = num(k["dram__bytes_read.sum"])
        wr = num(k["dram__bytes_write.sum"])
        unit_r = str(k["dram__bytes_read.sum"]).split()[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(unit_r, 1)
        wr *= scale.get(str(k["dram__bytes_write.sum"]).split()[1], 1)
        k["dram_bytes_per_launch"] = rd + wr
        k["report"] = os.path.basename(path)
        out["kernels"][key] = k
    dst = os.path.join(ROOT, "profiles", "ncu_summary.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"ncu_summary_{args.tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
