"""Timing of the DMMA GEMM engine on mode-0 products (through htr_mode_multiply
with device operands) against numpy; prints TF/s and the kernel chosen."""
import os, sys, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2412_16544_b200 import htrise as ht
ctx = ht.Context(0)
def dp(t): return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))
for (J, O, Q) in [(400, 5120, 400), (128, 32768, 20), (400, 20480, 400)]:
    X = torch.randn(O, J, dtype=torch.float64, device="cuda")          # canonical (J, O)
    Mt = torch.randn(J, Q, dtype=torch.float64, device="cuda")         # column-major Q x J
    out = torch.empty(O, Q, dtype=torch.float64, device="cuda")
    shape = (C.c_int64 * 2)(J, O)
    call = lambda: ctx.check(ht.lib().htr_mode_multiply(ctx.handle, dp(X), 1, shape, 2, 0, dp(Mt), Q, dp(out), 1))
    call(); ctx.synchronize()
    # check: out(q, o) = sum_j M(q, j) X(j, o); M(q,j) = Mt_storage[q + Q j]
    Mq = Mt.reshape(-1)[: Q * J].reshape(J, Q).T          # (Q, J)
    want = (Mq @ X.T).T                                     # (O, Q) storage == canonical (Q, O)
    err = (out - want).abs().max().item() / want.abs().max().item()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5): call()
        ctx.synchronize()
    for e in prof.key_averages():
        if e.device_type == torch.autograd.DeviceType.CUDA and "gemm" in e.key:
            us = e.device_time_total / e.count
            tf = 2.0 * J * O * Q / (us * 1e-6) / 1e12
            print(f"J={J} O={O} Q={Q}: {us:8.1f} us  {tf:5.1f} TF/s  relerr {err:.1e}  {e.key[:60]}")
