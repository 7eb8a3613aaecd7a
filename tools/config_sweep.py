"""Per-config timings on one GPU: BHT-l2r on batch 0, then the HT-RISE
stream (skip / non-skip update latency from the library's own wall clock,
like UpdateReport.seconds in ht_rise.hpp:117-121) and GB/s of streamed data."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
ap.add_argument("--max-batches", type=int, default=40)
a = ap.parse_args()
ctx = ht.Context(0); ht.set_default_context(ctx)
rows = []
for name in a.configs.split(","):
    w = CONFIGS[name]
    y0 = w.make_batch(0, "cuda"); torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
    t_bht_first = time.perf_counter() - t0  # includes lazy module loading of the kernels it meets first
    t0 = time.perf_counter()
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
    t_bht = time.perf_counter() - t0
    del y0
    skip_t, full_t, fused = [], [], 0
    nb = min(w.n_batches, a.max_batches)
    for b in range(1, nb):
        yb = w.make_batch(b, "cuda"); torch.cuda.synchronize()
        rep, upd = ht.ht_rise_update(rep, ht.DeviceTensor(yb, w.shape))
        (skip_t if upd.skipped else full_t).append(upd.seconds)
        fused += upd.used_fused_path
        del yb
    # the same kind of batches as one stream (ht_rise_update_many, batches
    # resident on the device): per-batch time with the host round trips
    # pipelined behind the device work (CUDA events on the library stream)
    P = min(nb - 1, 8 if w.bytes_per_batch < 1e9 else 3)
    K = 24
    stream_ms = None
    if P >= 1:
        pool = [ht.DeviceTensor(w.make_batch(b, "cuda"), w.shape) for b in range(1, P + 1)]
        rep.reserve(rep.accumulated + (2 * K + 4) * w.batch)
        vals, _ = ht.ht_rise_update_many(rep, [pool[i % P] for i in range(4)])
        rep = vals[-1]
        ctx.synchronize()
        st = torch.cuda.ExternalStream(ctx.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        vals, reps = ht.ht_rise_update_many(rep, [pool[i % P] for i in range(K)])
        e1.record(st)
        e1.synchronize()
        wall = time.perf_counter() - t0
        stream_ms = e0.elapsed_time(e1) / K
        stream_wall_ms = 1e3 * wall / K
        stream_skips = sum(int(r.skipped) for r in reps)
        rep = vals[-1]
        del pool, vals
    gb = w.bytes_per_batch / 1e9
    med = sorted(skip_t)[len(skip_t) // 2] if skip_t else None
    row = {"config": name, "batch_GB": round(gb, 4), "bht_l2r_ms": round(1e3 * t_bht, 2),
           "bht_l2r_first_ms": round(1e3 * t_bht_first, 2),
           "updates": nb - 1, "skips": len(skip_t), "fused_path": fused,
           "skip_ms_median": round(1e3 * med, 3) if skip_t else None,
           "skip_ms_mean": round(1e3 * sum(skip_t) / len(skip_t), 3) if skip_t else None,
           "skip_ms_first": round(1e3 * skip_t[0], 3) if skip_t else None,
           "nonskip_ms_mean": round(1e3 * sum(full_t) / len(full_t), 3) if full_t else None,
           "skip_GBps_median": round(gb / med, 1) if skip_t else None,
           "stream_ms_per_batch": round(stream_ms, 4) if stream_ms else None,
           "stream_wall_ms_per_batch": round(stream_wall_ms, 4) if stream_ms else None,
           "stream_skips": f"{stream_skips}/{K}" if stream_ms else None,
           "stream_GBps": round(gb / stream_ms * 1e3, 1) if stream_ms else None,
           "ranks": {str(k): v for k, v in rep.ranks().items()}}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del rep
    torch.cuda.empty_cache()
