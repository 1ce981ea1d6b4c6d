"""Summarise ncu output for profiles/.

  python profiles/ncu_summary.py <report.ncu-rep> [...]     per-kernel metrics + top stalls
  python profiles/ncu_summary.py --json out.json <rep> ...  also write {kernel: metrics} JSON
  python profiles/ncu_summary.py --launches <list.csv>      aggregate a
      `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel

The JSON's dram_bytes (= dram__bytes_read.sum + dram__bytes_write.sum of one
launch) is what bench.py reports as roofline.traffic."""
import collections
import csv
import io
import json
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
    ("launch__grid_size", "grid"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("smsp__inst_executed.sum", "inst"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def kernel_name(raw):
    """'void gmd::<unnamed>::k_conv2<3, 0>(gmd::ConvArgs, ...)' -> 'k_conv2'."""
    name = raw.split("(")[0]
    for junk in ("(anonymous namespace)::", "<unnamed>::", "unnamed>::", "gmd::", "void "):
        name = name.replace(junk, "")
    return name.split("<")[0].strip()


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    res = {}
    for r in rows[2:]:
        name = kernel_name(r[name_i])
        m = {}
        for k, lab in WANT:
            if k in hdr:
                i = hdr.index(k)
                v = num(r[i])
                if lab == "time":
                    v = v * SCALE.get(units[i], 1) if v is not None else None  # -> ms
                elif lab.startswith("dram"):
                    v = v * SCALE.get(units[i], 1) if v is not None else None  # -> bytes
                m[lab] = v
        stalls = {}
        for i, k in enumerate(hdr):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k:
                v = num(r[i])
                if v:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
        tot = sum(stalls.values()) or 1.0
        m["stalls"] = {k: round(v / tot, 3) for k, v in
                       sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        m["dram_bytes"] = (m.get("dram_rd") or 0) + (m.get("dram_wr") or 0)
        res[name] = m
    return res


def launches(path):
    per = collections.OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = kernel_name(r["Kernel Name"])
        t = num(r["Metric Value"]) * SCALE.get(r["Metric Unit"], 1)
        c = per.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += t
    total = sum(v[1] for v in per.values()) or 1.0
    print(f"{'kernel':28s} {'launches':>8s} {'total_ms':>10s} {'mean_ms':>9s} {'share':>6s}")
    for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} {n:8d} {t:10.4f} {t / n:9.4f} {t / total:6.3f}")


def main(argv):
    if argv and argv[0] == "--launches":
        for p in argv[1:]:
            launches(p)
        return
    jpath = None
    if argv and argv[0] == "--json":
        jpath, argv = argv[1], argv[2:]
    allm = {}
    for p in argv:
        for name, m in report(p).items():
            allm[name] = m
            parts = " ".join(f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}"
                             for k, v in m.items() if k != "stalls")
            print(f"{name} | {parts}\n    stalls: {m['stalls']}")
    if jpath:
        with open(jpath, "w") as f:
            json.dump(allm, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
