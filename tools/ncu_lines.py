#!/usr/bin/env python
"""Per-source-line instruction and warp-stall shares of one kernel in an ncu report.

  python tools/ncu_lines.py <file.ncu-rep> [N] [launch-index]
"""
import collections
import csv
import subprocess
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if len(sys.argv) > 3:
        cmd += ["--launch-skip", sys.argv[3], "--launch-count", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    per, stall, src, f = collections.Counter(), collections.Counter(), {}, None
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) < 8 or not r[0].isdigit():
            continue
        key = (f, int(r[0]))
        src[key] = r[1].strip()
        try:
            per[key] += int(r[7])
            stall[key] += int(r[4])
        except ValueError:
            pass
    T, S = sum(per.values()) or 1, sum(stall.values()) or 1
    print(f"warp instructions {T}, stall samples {S}")
    print("| inst % | stall % | line | source |")
    print("|---:|---:|---|---|")
    for k, v in stall.most_common(n):
        print(f"| {100 * per[k] / T:.1f} | {100 * v / S:.1f} | {k[0]}:{k[1]} | `{src[k][:80]}` |")


if __name__ == "__main__":
    main()
