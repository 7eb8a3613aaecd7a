"""H2D bandwidth from pinned memory with 1, 2 and 4 concurrent streams (chunks
of one 4.3 GB buffer): can the e2e leg go faster than one copy engine?"""
import time

import torch

n = 128 ** 3 * 256
host = torch.empty(n, dtype=torch.float64).pin_memory()
host.fill_(1.0)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for k in (1, 2, 4):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chunk = n // k
        for j in range(k):
            with torch.cuda.stream(streams[j]):
                dev[j * chunk:(j + 1) * chunk].copy_(host[j * chunk:(j + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{k} streams: {n * 8 / dt / 1e9:.1f} GB/s")
