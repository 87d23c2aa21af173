"""Summarise an ncu report (--set full) or a launch-list CSV into markdown for profiles/.

    python tools/ncu_summary.py report.ncu-rep [...]      # per-kernel key metrics
    python tools/ncu_summary.py --launches launches.csv   # per-kernel time shares
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(rep):
    hdr, units, data = raw(rep)
    lines = [f"### {rep}", ""]
    for row in data:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"**{name[:110]}**")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"| {label} (`{key}`) | {row[i]} {units[i]} |")
        stalls = [(hdr[i], row[i]) for i in range(len(hdr))
                  if hdr[i].startswith("smsp__average_warps_issue_stalled") and hdr[i].endswith(".ratio")]
        stalls = sorted(((float(v.replace(",", "")), k) for k, v in stalls if v not in ("", "n/a")), reverse=True)[:6]
        if stalls:
            lines.append("")
            lines.append("top stall reasons (warps per issue-active cycle): " +
                         ", ".join(f"{k.split('stalled_')[1].split('_per_issue')[0]} {v:.2f}" for v, k in stalls))
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        name = r[ki].split("(")[0][:70]
        agg.setdefault(name, []).append(v)
    # the capture's -k filter restricts the list to this library's kernels (names show up with or
    # without their sa:: / unnamed namespace depending on the ncu version)
    ours = dict(agg)
    lines = ["| kernel | launches | avg us | total us |", "|---|---|---|---|"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} |")
    return "\n".join(lines)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))
