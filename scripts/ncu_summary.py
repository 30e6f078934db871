"""Summarise an ncu report (--page raw --csv) into a markdown table.

usage: python scripts/ncu_summary.py report.ncu-rep [out.md]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6, "ns"),
    ("dram_rd_MB", "dram__bytes_read.sum", None, None),
    ("dram_wr_MB", "dram__bytes_write.sum", None, None),
    ("dram_%peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None, None),
    ("sm_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", None, None),
    ("warps_active_%", "sm__warps_active.avg.pct_of_peak_sustained_active", None, None),
    ("regs", "launch__registers_per_thread", None, None),
    ("block", "launch__block_size", None, None),
    ("grid", "launch__grid_size", None, None),
    ("smem_bank_confl", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", None, None),
    ("inst_M", "smsp__inst_executed.sum", None, None),
    ("issue_active_%", "sm__inst_issued.avg.pct_of_peak_sustained_active", None, None),
]


def to_mb(v, unit):
    v = float(v)
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    return v * scale


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = ["| kernel | " + " | ".join(m[0] for m in METRICS) + " |", "|" + "---|" * (len(METRICS) + 1)]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        cells = []
        for label, key, _, _ in METRICS:
            if key not in hdr:
                cells.append("-")
                continue
            i = hdr.index(key)
            v, u = r[i], units[i]
            if label == "time_ms":
                f = float(v) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3,
                                "ms": 1.0}.get(u, 1.0)
                cells.append(f"{f:.4f}")
            elif label.endswith("_MB"):
                cells.append(f"{to_mb(v, u):.1f}")
            elif label == "inst_M":
                cells.append(f"{float(v) / 1e6:.1f}")
            else:
                cells.append(v)
        out.append(f"| {name} | " + " | ".join(cells) + " |")
    text = "\n".join(out)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
