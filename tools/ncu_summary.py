"""Summarise an ncu report (--set full) and a launch-list CSV into profiles/.

    python tools/ncu_summary.py gpurun_out/r01_sweep.ncu-rep gpurun_out/r01_launches.csv \
        profiles/r01_sweep_f64_8192.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__shared_mem_per_block_dynamic"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(r, hdr, units) for r in rows[2:]]


def main(rep, launches, dest):
    lines = [f"# ncu summary: `{rep}`", ""]
    for r, hdr, units in raw(rep):
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"## {name[:120]}")
        lines.append("")
        lines.append("| metric | unit | value |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in hdr:
                lines.append(f"| {k} | {units[hdr.index(k)]} | {r[hdr.index(k)]} |")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        lines.append("")
        lines.append("stall samples (share): " + ", ".join(
            f"{h} {100 * v / tot:.1f}%" for v, h in sorted(st, reverse=True)[:8]))
        lines.append("")
    if launches:
        per = defaultdict(list)
        with open(launches) as f:
            rdr = csv.reader(l for l in f if not l.startswith("=="))
            hdr = next(rdr)
            ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
            ui = hdr.index("Metric Unit")
            for row in rdr:
                if row[mi] == "gpu__time_duration.sum":
                    v = float(row[vi].replace(",", ""))
                    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(row[ui], 1.0)
                    per[row[ki].split("(")[0][:90]].append(v * scale)
        tot = sum(sum(v) for v in per.values())
        lines.append(f"## launch list `{launches}` (cold-cache, serialised; compare shares)")
        lines.append("")
        lines.append("| kernel | launches | total us | share | avg us |")
        lines.append("|---|---|---|---|---|")
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% | "
                         f"{sum(v) / len(v):.1f} |")
    with open(dest, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if len(sys.argv) not in (3, 4) or not sys.argv[-1].endswith(".md"):
        sys.exit("usage: ncu_summary.py REPORT.ncu-rep [LAUNCHES.csv] DEST.md")
    main(sys.argv[1], sys.argv[2] if len(sys.argv) == 4 else None, sys.argv[-1])
