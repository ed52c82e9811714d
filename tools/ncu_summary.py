"""One-line-per-kernel summary of an ncu --set full report (read here, not on the box).

    python tools/ncu_summary.py gpurun_out/r34/prof_c3.ncu-rep [label]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

WANT = {
    "Duration": "dur",
    "DRAM Throughput": "dram_pct",
    "Memory Throughput": "mem",
    "Compute (SM) Throughput": "sm_pct",
    "Registers Per Thread": "regs",
    "Achieved Occupancy": "occ",
    "Theoretical Occupancy": "theo_occ",
    "L1/TEX Hit Rate": "l1_hit",
    "L2 Hit Rate": "l2_hit",
    "Issue Slots Busy": "issue",
    "Block Size": "bs",
    "Grid Size": "grid",
    "Warp Cycles Per Issued Instruction": "cpi",
}


def main(path, label=""):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    out = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if r[mi] in WANT:
            key = WANT[r[mi]]
            if key == "mem" and r[ui] == "%":
                continue
            out[r[ii]][key] = f"{r[vi]} {r[ui]}".strip()
            names[r[ii]] = r[ki].split("(")[0]
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh = rr[0]
        for r in rr[2:]:
            i = r[hh.index("ID")]
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if m in hh:
                    out[i][m] = f"{r[hh.index(m)]} {rr[1][hh.index(m)]}"
    print(f"ncu --set full --clock-control none ({path}) {label}")
    print("Times under ncu are serialised / cold-cache: compare shares, not absolutes.")
    for i in sorted(out, key=int):
        d = out[i]
        print(f"[{i}] {names.get(i)}: " + ", ".join(f"{k}={v}" for k, v in d.items()))


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
