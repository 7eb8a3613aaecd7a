"""Device-time breakdown of decode for config 5 (latent of one 256-sample
batch -> 128^3 x 256 reconstruction, 4.3 GB written), through the C-ABI
with device-resident input and output."""
import ctypes as C
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

w = CONFIGS["c5"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
r11, r12, _ = rep.core_shape((0, 0))
lat = torch.randn(w.batch, r12, r11, dtype=torch.float64, device="cuda")
out = torch.empty_like(y0)
shape = (C.c_int64 * 3)(r11, r12, w.batch)
dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))  # noqa: E731


def call():
    ctx.check(ht.lib().htr_decode(ctx.handle, rep._h, dp(lat), 1, shape, dp(out), 1))


call()
ctx.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        call()
    ctx.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total
        cnt[e.name] += 1
busy = sum(tot.values()) / 3
print(f"decode c5: {busy:.1f} us device time per call; 4.295 GB written -> {4.295e9 / (busy * 1e-6) / 1e9:.0f} GB/s")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v / 3:9.1f} us  x{cnt[k] / 3:.0f}  {k[:90]}")

# relative_test_error summand of the same batch (encode + residual decode,
# the reconstruction compared in HBM and never written)
ys = (C.c_int64 * 4)(*w.shape)
err = C.c_double()


def rte():
    ctx.check(ht.lib().htr_relative_error(ctx.handle, rep._h, dp(y0), 1, ys, 4, C.byref(err)))


rte()
ctx.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        rte()
    ctx.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total
        cnt[e.name] += 1
busy = sum(tot.values()) / 3
print(f"relative error c5 (rte {err.value:.3e}): {busy:.1f} us device time per call; "
      f"4.295 GB read twice -> {2 * 4.295e9 / (busy * 1e-6) / 1e9:.0f} GB/s")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v / 3:9.1f} us  x{cnt[k] / 3:.0f}  {k[:90]}")
