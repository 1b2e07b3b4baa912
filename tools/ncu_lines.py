"""Aggregate an ncu report's per-SASS stall samples / instructions by CUDA source line.

usage: python tools/ncu_lines.py REPORT.ncu-rep [top_n] [kernel_regex]
"""
import csv
import io
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    kre = sys.argv[3] if len(sys.argv) > 3 else None
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kre:
        cmd += ["-k", "regex:" + kre]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    stalls, instr, text = {}, {}, {}
    fname, line = "?", None
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = {h: i for i, h in enumerate(row) if h not in hdr} if False else None
            hdr = {}
            for i, h in enumerate(row):
                hdr.setdefault(h, i)
            continue
        if hdr is None or len(row) < 6:
            continue
        if row[0]:
            line = (fname, int(row[0]))
            text[line] = row[1].strip()
            continue
        if line is None:
            continue
        try:
            s = float(row[hdr["Warp Stall Sampling (All Samples)"] + 2] or 0)
            n = float(row[hdr["Instructions Executed"] + 2] or 0)
        except (ValueError, KeyError):
            continue
        stalls[line] = stalls.get(line, 0) + s
        instr[line] = instr.get(line, 0) + n
    ts, ti = sum(stalls.values()) or 1, sum(instr.values()) or 1
    print(f"total stall samples {ts:.0f}  warp instructions {ti:.3e}")
    for ln in sorted(stalls, key=lambda x: -stalls[x])[:top]:
        print(f"{stalls[ln] / ts * 100:5.1f}% st {instr[ln] / ti * 100:5.1f}% in  {ln[0]}:{ln[1]:<4d} {text.get(ln, '')[:90]}")


if __name__ == "__main__":
    main()
