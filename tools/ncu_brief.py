"""One-line-per-kernel summary of an ncu --set full report (for profiles/).   python tools/ncu_brief.py REP..."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem"]

for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    for v in rows[2:]:
        d = dict(zip(h, v))
        print(f"== {rep}: {d.get('Kernel Name')}")
        print("  " + "; ".join(f"{k}={d.get(k)}" for k in KEYS if d.get(k) not in (None, "")))
        st = [(k, float(x.replace(",", ""))) for k, x in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and x]
        tot = sum(x for _, x in st) or 1.0
        print("  stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * x / tot:.1f}%"
                                       for k, x in sorted(st, key=lambda t: -t[1])[:8]))
