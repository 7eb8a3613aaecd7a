"""Summarise every launch of an ncu --set full report, one block per distinct
kernel (launches of the same kernel with the same grid are averaged):
duration, DRAM bytes, pipe activity, occupancy, registers and stall reasons.

  python tools/ncu_multi_summary.py report.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
col = {k: i for i, k in enumerate(h)}
WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe % active"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (shared) pipe % active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "DFMA inst % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem"),
]
TO_BASE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(r, k):
    try:
        return float(r[col[k]].replace(",", ""))
    except (KeyError, ValueError):
        return None


groups = OrderedDict()
for r in rows[2:]:
    name = r[col["Kernel Name"]].replace("void ", "").replace("unnamed>::", "").replace("<unnamed>::", "")
    key = (name.split("(")[0], r[col["launch__grid_size"]])
    groups.setdefault(key, []).append(r)

for (name, grid), rs in groups.items():
    print(f"== {name}  grid {grid}  x{len(rs)} launches")
    for k, label in WANT:
        if k not in col:
            continue
        vs = [val(r, k) for r in rs]
        vs = [v for v in vs if v is not None]
        if not vs:
            continue
        u = units[col[k]]
        mean = sum(vs) / len(vs)
        if u in TO_BASE and ("byte" in u or u in ("ns", "us", "ms", "s")):
            base = mean * TO_BASE[u]
            if "byte" in u:
                print(f"   {label:30s} {base / 1e6:12.3f} MB")
            else:
                print(f"   {label:30s} {base * 1e6:12.2f} us")
        else:
            print(f"   {label:30s} {mean:12.2f} {u}")
    st = {}
    for k in h:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            st[k.split("stalled_")[1]] = sum((val(r, k) or 0.0) for r in rs)
    tot = sum(st.values()) or 1.0
    print("   stalls: " + ", ".join(f"{k}={100 * x / tot:.1f}%" for k, x in sorted(st.items(), key=lambda t: -t[1])
                                   if x > 0.02 * tot))
