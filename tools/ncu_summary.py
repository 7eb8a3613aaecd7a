"""Summarise an ncu report: SOL, pipes, stall reasons, top stall sites."""
import csv, subprocess, sys, io
rep = sys.argv[1]
def page(p):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
raw = page("raw")
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k, uu, vv in zip(h, u, v):
    if k in want:
        print(f"{k:80s} {vv} {uu}")
tot = 0; st = {}
for k, vv in zip(h, v):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        st[k.split("stalled_")[1]] = int(float(vv or 0))
tot = sum(st.values())
print("stalls:", ", ".join(f"{k}={100*x/tot:.1f}%" for k, x in sorted(st.items(), key=lambda t: -t[1]) if x > 0.005 * tot))
src = page("source")
hh = src[1]; rows = [dict(zip(hh, r)) for r in src[2:]]
rows.sort(key=lambda x: -int(x.get("Warp Stall Sampling (All Samples)") or 0))
t = sum(int(x.get("Warp Stall Sampling (All Samples)") or 0) for x in rows)
for x in rows[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    n = int(x["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{100*n/t:5.1f}% {x['Address'][-5:]} {x['Source'][:90]}")
