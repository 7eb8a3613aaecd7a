"""Per-source-line warp-stall samples of one kernel in an ncu report (the
cuda,sass source view; ncu aggregates each CUDA line's SASS).

  python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows:
    if r and r[0].isdigit() and len(r) > ix:
        try:
            lines.append((float(r[ix]), int(r[0]), r[1][:100]))
        except ValueError:
            pass
tot = sum(v for v, _, _ in lines) or 1.0
for v, ln, s in sorted(lines, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  L{ln}: {s}")
