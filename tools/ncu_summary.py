#!/usr/bin/env python
"""Summarises ncu outputs into a markdown block for profiles/.

  python tools/ncu_summary.py launches <launches.csv>        # per-kernel share of device time
  python tools/ncu_summary.py report <file.ncu-rep> [...]     # key metrics of a --set full capture
  python tools/ncu_summary.py hotspots <file.ncu-rep> [N]     # warp-stall samples by source line
"""
import collections
import csv
import subprocess
import sys

KEY_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads per warp instruction (warp efficiency)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def short(name):
    n = name.split("(")[0].replace("bdsm_b200::<unnamed>::", "").replace("void ", "")
    if "cub::" in name or "DeviceRadixSort" in name or "DeviceScan" in name or "DeviceSelect" in name:
        for tag in ("Onesweep", "Histogram", "ExclusiveSum", "Select", "Scan", "Upsweep", "Downsweep"):
            if tag.lower() in name.lower():
                return f"CUB {tag}"
        return "CUB (other)"
    return n[:60]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[start + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        k = short(r[ki])
        if "native::" in r[ki] or "at::" in r[ki]:
            k = "torch (workload generation, not in the timed step)"
        tot[k] += v * scale
        cnt[k] += 1
    T = sum(tot.values())
    print("| kernel | launches | total ms (ncu, serialised) | share |")
    print("|---|---:|---:|---:|")
    for k, v in tot.most_common():
        print(f"| {k} | {cnt[k]} | {v:.2f} | {100 * v / T:.2f}% |")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = short(r[h.index("Kernel Name")]) if "Kernel Name" in h else "?"
        print(f"**{name}** ({path.split('/')[-1]})\n")
        print("| metric | value |")
        print("|---|---|")
        for m, label in KEY_METRICS:
            if m in h:
                i = h.index(m)
                print(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
        print()


def hotspots(path, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    per, src = collections.Counter(), {}
    cur = None
    for r in rows[3:]:
        if len(r) < 7:
            continue
        if r[0] and r[0].isdigit():
            cur = int(r[0])
            src[cur] = r[1].strip()
        try:
            per[cur] += int(r[4])
        except ValueError:
            pass
    tot = sum(per.values()) or 1
    print("| share of warp-stall samples | line | source |")
    print("|---:|---:|---|")
    for line, s in per.most_common(n):
        print(f"| {100 * s / tot:.1f}% | {line} | `{src.get(line, '')[:90]}` |")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "report":
        for p in sys.argv[2:]:
            report(p)
    elif cmd == "hotspots":
        hotspots(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
