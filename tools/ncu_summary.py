"""Summarise ncu --set full reports (one kernel each) into a markdown table + traffic json.
Usage: python tools/ncu_summary.py out.md traffic.json name=report.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA-pipe inst % (active)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) inst % (active)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU inst % (active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x[0] or 0)) for k, x in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                    key=lambda t: -t[1])
    return d, stalls


def to_bytes(val, unit):
    f = float(val)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    md, tj = sys.argv[1], sys.argv[2]
    reps = [a.split("=", 1) for a in sys.argv[3:]]
    lines = ["| metric | " + " | ".join(n for n, _ in reps) + " |", "|---|" + "---|" * len(reps)]
    data = [raw(p) for _, p in reps]
    for k, label in KEYS:
        cells = []
        for d, _ in data:
            v = d.get(k)
            cells.append(f"{v[0]} {v[1]}".strip() if v else "-")
        lines.append(f"| {label} (`{k}`) | " + " | ".join(cells) + " |")
    lines.append("| top stall reasons (pc samples) | " + " | ".join(
        ", ".join(f"{n} {100 * c / max(1, sum(x for _, x in st)):.0f}%" for n, c in st[:4]) for _, st in data) + " |")
    traffic = {}
    for (name, _), (d, _) in zip(reps, data):
        r, w = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if r and w:
            traffic[name] = to_bytes(*r) + to_bytes(*w)
    open(md, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tj, "w"), indent=1)


if __name__ == "__main__":
    main()
