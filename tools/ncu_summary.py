#!/usr/bin/env python
"""Summarise ncu reports into the JSON lines kept under profiles/ (one line per kernel launch).

    python tools/ncu_summary.py REPORT.ncu-rep [...] > summary.jsonl
Reads `ncu -i REPORT --page raw --csv` and keeps the metrics the roofline discussion uses."""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units, data = r[0], r[1], r[2:]
    for row in data:
        d = {}
        for k in KEEP:
            if k in head:
                i = head.index(k)
                d[k] = f"{row[i]} {units[i]}".strip()
        d["kernel"] = row[head.index("Kernel Name")]
        yield d


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in rows(p):
            d["report"] = p
            print(json.dumps(d))
