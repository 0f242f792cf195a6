"""Summarise ncu reports (raw page) into small text files kept under profiles/<round>/.

    python profiles/summarize.py <report.ncu-rep> <out.txt>
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def summarize(rep, out):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(r.splitlines()))
    h, units = rows[0], rows[1]
    lines = []
    for row in rows[2:]:
        lines.append("kernel: " + row[h.index("Kernel Name")])
        for k in KEYS:
            if k in h:
                lines.append(f"  {k} = {row[h.index(k)]} {units[h.index(k)]}")
        st = [(n[33:], float(row[i] or 0)) for i, n in enumerate(h)
              if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
        st = sorted(st, key=lambda x: -x[1])[:6]
        lines.append("  top stall samples: " + ", ".join(f"{a}={int(b)}" for a, b in st))
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    summarize(sys.argv[1], sys.argv[2])
