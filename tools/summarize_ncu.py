"""Summaries of ncu output for profiles/ (tracked).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/r01_launches.md
    python tools/summarize_ncu.py full gpurun_out/prof_c2.ncu-rep > profiles/r01_ncu_full.md

`launches`: per-kernel count / mean / share of the launch list
(gpu__time_duration.sum, cold-cache and serialised under ncu: compare shares).
`full`: selected metrics per profiled kernel from `ncu -i ... --page raw --csv`.
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "GPU DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__inst_executed.avg.per_cycle_active", "IPC / SMSP"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "L1 global load bytes"),
    ("smsp__cycles_active.avg", "SMSP active cycles"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long-scoreboard"),
    ("smsp__pcsamp_warps_issue_stalled_barrier", "pcsamp stalled barrier"),
    ("smsp__pcsamp_warps_issue_stalled_long_scoreboard", "pcsamp stalled long_scoreboard"),
    ("smsp__pcsamp_warps_issue_stalled_short_scoreboard", "pcsamp stalled short_scoreboard"),
    ("smsp__pcsamp_warps_issue_stalled_wait", "pcsamp stalled wait"),
    ("smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "pcsamp stalled math throttle"),
    ("smsp__pcsamp_warps_issue_stalled_selected", "pcsamp selected"),
    ("smsp__pcsamp_warps_issue_stalled_mio_throttle", "pcsamp stalled mio throttle"),
    ("smsp__pcsamp_warps_issue_stalled_lg_throttle", "pcsamp stalled lg throttle"),
    ("smsp__pcsamp_warps_issue_stalled_sleeping", "pcsamp stalled sleeping"),
    ("smsp__pcsamp_warps_issue_stalled_no_instructions", "pcsamp stalled no instruction"),
]


def _short(name: str) -> str:
    name = name.split("(")[0]
    for pre in ("void ", "akv::"):
        name = name.replace(pre, "")
    return name[:60]


def launches(path: str) -> str:
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((_short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")), r["Metric Unit"]))
    agg = collections.OrderedDict()
    for n, v, u in rows:
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1e-3)
        agg.setdefault(n, []).append(v * scale)
    out = ["| kernel | launches | mean us | min us | max us |", "|---|---|---|---|---|"]
    for n, v in agg.items():
        out.append(f"| `{n}` | {len(v)} | {sum(v) / len(v):.2f} | {min(v):.2f} | {max(v):.2f} |")
    return "\n".join(out) + "\n"


def full(path: str) -> str:
    if path.endswith(".csv"):  # an exported `--page raw --csv`
        with open(path) as f:
            text = f.read()
    else:
        res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
        if res.returncode != 0:
            return "ncu -i failed:\n" + res.stderr
        text = res.stdout
    rd = list(csv.reader(io.StringIO(text)))
    hdr, units = rd[0], rd[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for row in rd[2:]:
        kn = row[idx["Kernel Name"]] if "Kernel Name" in idx else "?"
        out.append(f"### `{_short(kn)}`\n\n| metric | value | unit |\n|---|---|---|")
        for m, label in FULL_METRICS:
            if m in idx:
                out.append(f"| {label} (`{m}`) | {row[idx[m]]} | {units[idx[m]]} |")
        out.append("")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    sys.stdout.write(launches(path) if mode == "launches" else full(path))
