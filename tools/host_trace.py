"""Host/device timeline of consecutive HT-RISE skip updates on config 5:
CUDA runtime API calls (CUPTI, host side) and kernels (device side) of one
update, relative to the end of the previous update's last synchronize."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
y1 = w.make_batch(1, "cuda")
torch.cuda.synchronize()
rep.reserve(64 * w.batch)
dt = ht.DeviceTensor(y1, w.shape)
for _ in range(3):
    rep, upd = ht.ht_rise_update(rep, dt)
ctx.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(6):
        with torch.profiler.record_function("update"):
            rep, upd = ht.ht_rise_update(rep, dt)
    ctx.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ev = [e for e in ev if e.get("ph") == "X"]
ups = sorted([e for e in ev if e["name"] == "update"], key=lambda e: e["ts"])
for u in ups[2:4]:
    t0 = u["ts"]
    print(f"--- update: host {u['dur']:.1f} us")
    inside = sorted([e for e in ev if e is not u and (t0 <= e["ts"] <= t0 + u["dur"] + 2000)
                     and e.get("cat") in ("cuda_runtime", "kernel", "gpu_memcpy", "gpu_memset", "cuda_driver")],
                    key=lambda e: e["ts"])
    for e in inside:
        if e["ts"] > t0 + u["dur"] and e.get("cat") in ("cuda_runtime", "cuda_driver"):
            continue
        print(f"  {e['ts'] - t0:9.1f} +{e['dur']:8.1f}  {e.get('cat', ''):12s} {e['name'][:70]}")
    nxt = [x for x in ups if x["ts"] > t0]
    if len(nxt) > 1:
        print(f"  next update starts at {nxt[1]['ts'] - t0:.1f}")
