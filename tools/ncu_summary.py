#!/usr/bin/env python
"""Summarise an ncu report (raw page) into the numbers we track."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second"]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", "")[:90]}
        for k in KEYS:
            if k in d:
                ent[k] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = {k.split("stalled_")[1]: d[k] for k in hdr
                  if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:6]
        ent["top_stalls"] = top
        res.append(ent)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps({"report": p, "kernels": summarise(p)}, indent=1))
