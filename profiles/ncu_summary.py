"""Summarise an ncu report: per kernel the metrics the roofline uses.
usage: python profiles/ncu_summary.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
    ("smsp__inst_executed.sum", "inst"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k, _ in WANT if k in hdr}
    name_i = hdr.index("Kernel Name")
    for r in rows[2:]:
        name = r[name_i].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        parts = [f"{lab}={r[idx[k]]}{units[idx[k]] if lab in ('time','dram_rd','dram_wr') else ''}"
                 for k, lab in WANT if k in idx]
        print(name.strip(), "|", " ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1])
