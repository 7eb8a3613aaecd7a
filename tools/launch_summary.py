"""Per-update kernel breakdown from an ncu --metrics gpu__time_duration.sum CSV."""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
i_name, i_val, i_id = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[i_id]), r[i_name], float(r[i_val].replace(",", ""))))
    except Exception:
        pass
fi = [k for k, (i, n, v) in enumerate(data) if "fused3_kernel" in n]
def short(n):
    return n.replace("htr::<unnamed>::", "").replace("(anonymous namespace)::", "")[:80]
seg = data[fi[-1] - 1:]
tot = sum(v for _, _, v in seg)
for i, n, v in seg:
    print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}%  {short(n)}")
print(f"---- last update: {len(seg)} launches, {tot/1e3:.1f} us")
