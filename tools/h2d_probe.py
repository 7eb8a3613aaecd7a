"""Host->device copy bandwidth from pinned memory (the e2e leg's floor), and
the e2e update through the public API on the same buffer."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS
w = CONFIGS["c5"]
dev = torch.empty(w.shape[::-1], dtype=torch.float64, device="cuda")
t0 = time.perf_counter(); host = torch.empty(w.shape[::-1], dtype=torch.float64).pin_memory(); t1 = time.perf_counter()
print(f"pin 4.3 GB: {t1 - t0:.2f} s, numa/cpus {os.cpu_count()}")
host.fill_(1.0)
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"torch H2D {host.numel() * 8 / dt / 1e9:.1f} GB/s")
ctx = ht.Context(0); ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
y1 = w.make_batch(1, "cuda")
host.copy_(y1.reshape(w.shape[::-1]))
hn = host.numpy().transpose()
rep.reserve(16 * w.batch)
for i in range(4):
    t0 = time.perf_counter(); rep, u = ht.ht_rise_update(rep, hn); dt = time.perf_counter() - t0
    print(f"e2e update {dt * 1e3:.1f} ms = {host.numel() * 8 / dt / 1e9:.1f} GB/s skipped={u.skipped}")
