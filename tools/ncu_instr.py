"""Per-source-line warp-instruction and stall shares for one kernel of an ncu report.
usage: python tools/ncu_instr.py REPORT kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kre], capture_output=True, text=True).stdout
stalls, instr, text = {}, {}, {}
fname, line, hdr = "?", None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
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
        s_ = float(row[hdr["Warp Stall Sampling (All Samples)"] + 2] or 0)
        n_ = float(row[hdr["Instructions Executed"] + 2] or 0)
    except (ValueError, KeyError):
        continue
    stalls[line] = stalls.get(line, 0) + s_
    instr[line] = instr.get(line, 0) + n_
ti, ts = sum(instr.values()) or 1, sum(stalls.values()) or 1
print(f"warp instructions {ti:.4g}, stall samples {ts:.0f}")
for ln in sorted(instr, key=lambda x: -(instr[x] / ti + stalls[x] / ts))[:top]:
    print(f"{instr[ln] / ti * 100:5.1f}% in {stalls[ln] / ts * 100:5.1f}% st  {ln[0]}:{ln[1]:<4d} {text.get(ln, '')[:90]}")
