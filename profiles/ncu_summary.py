#!/usr/bin/env python
"""Summarise ncu output into the markdown committed under profiles/.

    python profiles/ncu_summary.py launches <launches.csv>          # per-kernel time shares
    python profiles/ncu_summary.py report <prof.ncu-rep> [...]      # key metrics per launch
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

KEY_METRICS = [
    "gpu__time_duration.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.sum",
    "smsp__inst_executed.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warp_latency_issue_stalled_math_pipe_throttle",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def _csv_rows(text: str):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path: str) -> str:
    rows = _csv_rows(open(path).read())
    hdr, body = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = {}
    for r in body:
        name = r[ki].split("(")[0]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        per.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale)
    total = sum(sum(v) for v in per.values())
    out = ["| kernel | launches | total ms | mean ms | share |", "|---|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v):.3f} | {sum(v)/len(v):.3f} | {100*sum(v)/total:.2f} % |")
    out.append(f"| all | {sum(len(v) for v in per.values())} | {total:.3f} | | 100 % |")
    return "\n".join(out)


def report(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = _csv_rows(raw)
    hdr, units, body = rows[0], rows[1], rows[2:]
    out = []
    for r in body:
        rec = dict(zip(hdr, r))
        out.append(f"### `{rec.get('Kernel Name', '?')[:110]}`")
        out.append(f"grid {rec.get('Grid Size')} block {rec.get('Block Size')}")
        out.append("")
        out.append("| metric | value | unit |")
        out.append("|---|---|---|")
        for m in KEY_METRICS:
            if m in rec:
                out.append(f"| `{m}` | {rec[m]} | {units[hdr.index(m)]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    mode, *paths = sys.argv[1:]
    for p in paths:
        print(f"## {p}\n")
        print(launches(p) if mode == "launches" else report(p))
        print()
