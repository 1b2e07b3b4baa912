"""Summarise an `ncu --set full` report into profiles/: a text summary per
kernel (averaged over its captured launches) and the per-launch DRAM traffic
JSON that bench.py folds into its roofline line.

usage: python tools/ncu_summary.py REPORT.ncu-rep TAG "note" [name=regex ...]
  e.g. python tools/ncu_summary.py gpurun_out/prof_r01d.ncu-rep r01d "..." \
         'leaf_map=leaf_map_kernel<32>' 'leaf_map_heavy=leaf_map_kernel<256>' 'tri_hist_fused=tri_hist_kernel'
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),  # ns -> ms (converted below by unit)
    "dram_read": ("dram__bytes_read.sum", 1),
    "dram_write": ("dram__bytes_write.sum", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "mem_pct": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "inst": ("smsp__inst_executed.sum", 1),
    "regs": ("launch__registers_per_thread", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1),
    "smem_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
}
SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3,
         "nsecond": 1e-6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    rep, tag, note = sys.argv[1], sys.argv[2], sys.argv[3]
    names = [a.split("=", 1) for a in sys.argv[4:]]
    # REPORT may also be the `ncu -i ... --page raw --csv` dump of a report that
    # stayed on the GPU box (full reports with sources exceed gpurun's copy-back limit)
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in data:
        kname = r[col["Kernel Name"]]
        label = next((nm for nm, rx in names if re.search(re.escape(rx) if "<" in rx else rx, kname)), None)
        if label is None:
            continue
        vals = {}
        for key, (metric, _) in METRICS.items():
            if metric not in col:
                continue
            raw = r[col[metric]].replace(",", "")
            try:
                v = float(raw)
            except ValueError:
                continue
            u = units[col[metric]]
            if key == "duration_ms":
                v *= SCALE.get(u, 1e-6)
            elif key.startswith("dram"):
                v *= SCALE.get(u, 1)
            vals[key] = v
        a = acc.setdefault(label, {"n": 0})
        a["n"] += 1
        for kk, v in vals.items():
            a[kk] = a.get(kk, 0.0) + v
    lines = [f"ncu --set full --clock-control none; {note}"]
    traffic = {}
    for label, a in acc.items():
        n = a.pop("n")
        m = {kk: v / n for kk, v in a.items()}
        dram = m.get("dram_read", 0) + m.get("dram_write", 0)
        lines.append(
            f"{label}: launches {n}, duration {m.get('duration_ms', 0):.4f} ms, dram {dram / 1e9:.3f} GB "
            f"({dram / 1e9 / max(m.get('duration_ms', 1e-9), 1e-9) * 1e3:.0f} GB/s), SM {m.get('sm_pct', 0):.1f} %, "
            f"mem {m.get('mem_pct', 0):.1f} %, warps active {m.get('warps_active_pct', 0):.1f} %, "
            f"issue active {m.get('issue_active_pct', 0):.1f} %, inst {m.get('inst', 0):.4g}, regs {m.get('regs', 0):.0f}, "
            f"L2 hit {m.get('l2_hit_pct', 0):.1f} %, L1 hit {m.get('l1_hit_pct', 0):.1f} %, "
            f"smem bank conflicts {m.get('smem_conflicts', 0):.3g}")
        traffic[label] = {"dram_bytes_per_launch": dram, "source": f"profiles/{tag}_ncu_full_summary.txt"}
    text = "\n".join(lines) + "\n"
    open(f"profiles/{tag}_ncu_full_summary.txt", "w").write(text)
    try:  # merge: other kernels' entries (other configs' captures) stay
        merged = json.load(open("profiles/ncu_traffic.json"))
    except (OSError, ValueError):
        merged = {}
    merged.update(traffic)
    json.dump(merged, open("profiles/ncu_traffic.json", "w"), indent=1)
    print(text)


if __name__ == "__main__":
    main()
