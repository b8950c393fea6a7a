"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py full <report.ncu-rep>      # per-kernel table from a --set full capture
  python tools/ncu_summary.py launches <launches.csv>    # per-kernel share of a gpu__time_duration launch list
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "MB rd", 1e-6),
    ("dram__bytes_write.sum", "MB wr", 1e-6),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram %", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %", 1),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
    ("launch__registers_per_thread", "regs", 1),
]

UNIT_SCALE = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
              "byte": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def short(name):
    name = name.split("(")[0]
    for p in ("void ", "infllm::", "<unnamed>::"):
        name = name.replace(p, "")
    return name


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    ki = head.index("Kernel Name")
    cols = [(head.index(m), lab, sc, m) for m, lab, sc in FULL_METRICS if m in head]
    print("| kernel | " + " | ".join(c[1] for c in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for r in data:
        vals = []
        for i, lab, sc, m in cols:
            v = r[i].replace(",", "")
            try:
                x = float(v) * UNIT_SCALE.get(units[i], 1.0) if m.endswith(".sum") else float(v)
                x = x * sc if m.endswith(".sum") else x
                vals.append(f"{x:.1f}" if x < 1e6 else f"{x:.0f}")
            except ValueError:
                vals.append(v)
        print(f"| {short(r[ki])} | " + " | ".join(vals) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if r[mi] != "gpu__time_duration.sum":
            continue
        ns = float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1.0)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | avg us | share of serialised device time |")
    print("|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t / n / 1e3:.2f} | {100 * t / tot:.1f}% |")
    print(f"\ntotal {sum(a[0] for a in agg.values())} launches, {tot / 1e3:.1f} us serialised")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
