"""Per-launch summary of an `ncu --set full` report (dev tool):
python tools/ncu_summary.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

COLS = [("grid", "launch__grid_size"), ("us", "gpu__time_duration.sum"),
        ("dram_rd_MB", "dram__bytes_read.sum"), ("dram_wr_MB", "dram__bytes_write.sum"),
        ("regs", "launch__registers_per_thread"),
        ("warps_active%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("issue%", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("fmaheavy%", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("alu%", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        ("fp64%", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
        ("dram%", "dram__bytes_read.sum.pct_of_peak_sustained_elapsed"),
        ("mem_thru%", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed")]


def main(path, title=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ix = {k: i for i, k in enumerate(h)}
    if title:
        print(title)
    print("kernel | " + " | ".join(c for c, _ in COLS))
    for r in rows[2:]:
        vals = []
        for c, m in COLS:
            if m not in ix:
                vals.append("-")
                continue
            v = r[ix[m]].replace(",", "")
            u = units[ix[m]]
            try:
                f = float(v)
                if u in ("byte",):
                    f /= 1e6
                elif u in ("Kbyte",):
                    f /= 1e3
                elif u in ("Gbyte",):
                    f *= 1e3
                elif u in ("nsecond", "ns"):
                    f /= 1e3
                elif u in ("msecond", "ms"):
                    f *= 1e3
                v = f"{f:.1f}"
            except ValueError:
                pass
            vals.append(v)
        print(r[ix["Kernel Name"]].split("(")[0].replace("void ", "")[:40] + " | " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
