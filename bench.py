#!/usr/bin/env python
"""HT-RISE update throughput on B200 (BASELINE.json metric: GB/s of streamed
tensor data, with the fused kernel's HBM roofline fraction).

One step = one HT-RISE update of a config-5 batch (128^3 x 256 f64 = 4.295 GB,
tree (1,(2,3)), eps 1e-3) through libhtrise_cuda.so. The stream is first
seeded with BHT-l2r on batch 0 (untimed, like the reference's CLI); steps then
cycle through distinct pre-generated batches that are resident in HBM (each
4.3 GB >> the 126 MB L2, so no flush is needed). The headline times the K
steps as one stream (ht_rise_update_many: the reference CLI's loop over
batches, with batch i+1's encode queued before batch i's decision is read
back); "per_call" times the same K steps as K ht_rise_update calls.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: launched by torchrun, one rank per GPU; every batch is sharded
along the batch axis (N/G samples per rank, "weak" in samples per GPU is NOT
the case: total work per step is fixed -> scaling "strong"), the skip test's
two norms are all-reduced over NCCL inside the library.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HT-RISE update GB/s of streamed tensor data"
UNIT = "GB/s"


HBM_NOMINAL_GBS = 8000.0
FP64_DMMA_TFLOPS = 37.18  # profiles/r1_microbench_fp64.txt (best DMMA.8x8x4 line)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.source = "nvidia-smi"

    def _run(self):
        if self._run_nvml():
            return
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run_nvml(self) -> bool:
        """Poll NVML directly every millisecond (the timed region of a default
        run is ~10 ms: one nvidia-smi process start would cover it with a
        single sample). False when NVML is unavailable (nvidia-smi fallback)."""
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            try:
                uuid = str(torch.cuda.get_device_properties(self.device).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid if not uuid.startswith("GPU-") else uuid).encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons(h)
        except Exception:
            return False
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap
        while True:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = int(reasons(h))
                try:
                    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                except Exception:
                    pw = 0.0
                self.samples.append([str(sm), str(mx), f"{pw:.1f}", hex(r)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
            except Exception:
                pass
            if self._stop.wait(0.001):
                break
        self.source = "nvml"
        return True

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, n in enumerate(names):
                if len(s) > 4 + i and s[4 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(self.samples), "source": self.source}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _host_info():
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["lscpu_model"] = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return info


def _c5_host_batch(w, b, n):
    """Batch b of config 5 (n samples) in host memory, canonical order: the
    device generator's bytes when a GPU is present (the same bytes the GPU
    arm streams), else the same generator on the CPU."""
    import numpy as np
    import torch

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    y = w.make_batch(b, dev, batch=n).cpu().numpy()
    return np.asfortranarray(y.reshape((n,) + tuple(reversed(w.dims))).transpose(3, 2, 1, 0))


def cpu_reference(steps: int, warmup: int, budget_s: float, all_cores: bool = True):
    """The reference's algorithm on the host: the oracle port (numpy
    restatement of ht_rise.hpp:99-186, op for op; the reference itself needs
    Eigen, absent here) timing FULL config-5 updates (256 samples, 4.295 GB,
    the same workload as the GPU step) with ONE thread, as the reference runs
    (no OpenMP/threads, CMakeLists.txt:1-20; OPENBLAS limited to 1 through
    threadpoolctl), the way the reference times them (UpdateReport.seconds,
    ht_rise.hpp:102-121). The stream is seeded untimed by the oracle's
    BHT-l2r on a 32-sample batch (ranks 20/20/20/400, as at 256). At most
    `steps` timed updates, fewer when the `budget_s` wall-clock budget runs
    out (at least one). Optionally one more update with every host thread,
    reported separately."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import htrise_oracle as ho
    from paper_2412_16544_b200.workloads import CONFIGS

    w = CONFIGS["c5"]
    t_seed = time.perf_counter()
    rep, _ = ho.bht_l2r(_c5_host_batch(w, 0, 32), ho.custom_tree_1_23(), w.eps)
    t_seed = time.perf_counter() - t_seed
    y = _c5_host_batch(w, 1, w.batch)
    nbytes = 8.0 * y.size
    t_start = time.perf_counter()
    times = []
    skipped = 0
    with threadpool_limits(1):
        for _ in range(min(warmup, 1)):
            ho.ht_rise_update(rep, y)
        while len(times) < max(1, steps):
            _, upd = ho.ht_rise_update(rep, y)
            times.append(upd.seconds)
            skipped += int(upd.skipped)
            if time.perf_counter() - t_start + times[-1] > budget_s:
                break
    mean = sum(times) / len(times)
    out = {"value": nbytes / mean / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
           "seconds_per_update": mean, "updates_timed": len(times), "skipped": skipped,
           "sample": f"{len(times)} full config-5 ht_rise_update calls (256 x 128^3 f64, 4.295 GB each, skip path) "
                     f"of the oracle port, 1 thread, UpdateReport.seconds; stream seeded untimed by BHT-l2r on "
                     f"32 samples ({t_seed:.0f} s)",
           "host": _host_info()}
    if all_cores:
        with threadpool_limits(os.cpu_count()):
            _, upd = ho.ht_rise_update(rep, y)
        out["all_cores"] = {"value": nbytes / upd.seconds / 1e9, "unit": UNIT, "cores": os.cpu_count(),
                            "seconds_per_update": upd.seconds,
                            "sample": "1 full config-5 update, OpenBLAS on every host thread (numpy's "
                                      "elementwise passes stay single-threaded)"}
    return out


def run_reference(args):
    world, rank, local = _dist_env()
    if rank != 0:
        return 0
    from paper_2412_16544_b200.workloads import CONFIGS
    cb = cpu_reference(args.steps, args.warmup, budget_s=args.ref_budget)
    steps_ms = cb["seconds_per_update"] * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": cb["updates_timed"], "warmup": min(args.warmup, 1), "ms_per_step": steps_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c5: {CONFIGS['c5'].description}", "batch_bytes": 8 * 128 ** 3 * 256,
                       "samples_per_gpu": 256, "parallelism": "1 host thread (the reference is single-threaded)",
                       "sample": "full 256-sample updates, count bounded by the time budget (cpu_baseline.sample)"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _first_kernel_label(config):
    """The streaming kernel the roofline entry times (the first launch of the
    skip-path encode, bracketed by CUDA events inside the library)."""
    if config == "c4":
        return "quad_stream_kernel (first 4-leaf subtree pass over y + ||Y||^2, DFMA f64)"
    if config == "c3":
        return "fused3_kernel (leaves 1, 2 of the balanced tree + ||Y||^2, DMMA f64)"
    return "fused3_kernel (leaf projections + ||Y||^2, DMMA f64)"


def run_ours(args):
    import numpy as np
    import torch

    from paper_2412_16544_b200 import htrise as ht
    from paper_2412_16544_b200.workloads import CONFIGS

    world, rank, local = _dist_env()
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPUs")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = ht.Context(local)
    ht.set_default_context(ctx)
    if world > 1:
        uid = [ht.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(uid[0], world, rank)

    w = CONFIGS[args.config]
    if w.batch % world:
        raise SystemExit(f"batch {w.batch} not divisible by {world} GPUs")
    n_local = w.batch // world
    off = rank * n_local
    shape = tuple(w.dims) + (n_local,)
    local_bytes = 8 * math.prod(shape)
    global_bytes = local_bytes * world

    # seed the stream with BHT-l2r on batch 0 (untimed), then a pool of
    # distinct resident batches for the updates
    y0 = w.make_batch(0, "cuda", batch=n_local, sample_offset=off)
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, shape), w.tree(), w.eps)
    del y0
    pool_n = max(2, min(args.pool, args.steps + args.warmup))
    pool = [w.make_batch(1 + i, "cuda", batch=n_local, sample_offset=off) for i in range(pool_n)]
    torch.cuda.synchronize()
    rep.reserve((2 + args.steps * 4 + args.warmup * 2 + 4) * n_local)

    def barrier():
        if dist is not None:
            dist.barrier()

    for i in range(args.warmup):
        rep, upd = ht.ht_rise_update(rep, ht.DeviceTensor(pool[i % pool_n], shape))
    ctx.synchronize()

    stream = torch.cuda.ExternalStream(ctx.stream())
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count()
    skipped = 0
    fused_used = 0
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for i in range(args.steps):
            rep, upd = ht.ht_rise_update(rep, ht.DeviceTensor(pool[(args.warmup + i) % pool_n], shape))
            skipped += int(upd.skipped)
            fused_used += int(upd.used_fused_path)
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    call_launches = ctx.launch_count() - launches0
    call_ms = e0.elapsed_time(e1) / args.steps

    # the same K batches as one stream (ht_rise_update_many: batch i+1's
    # encode is queued before batch i's skip decision is read back, so the
    # device does not idle across the host round trip of each decision)
    def batches(k0, k):
        return [ht.DeviceTensor(pool[(k0 + i) % pool_n], shape) for i in range(k)]

    vals, _ = ht.ht_rise_update_many(rep, batches(0, args.warmup))
    rep = vals[-1]
    ctx.synchronize()
    launches0 = ctx.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks2:
        e0.record(stream)
        vals, reports = ht.ht_rise_update_many(rep, batches(args.warmup, args.steps))
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    rep = vals[-1]
    stream_skipped = sum(int(u.skipped) for u in reports)
    stream_fused = sum(int(u.used_fused_path) for u in reports)
    launches = ctx.launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps

    # the same K steps once more with the library's CUDA events around the
    # streaming kernel of every step (the roofline entry's kernel time). The
    # event recorded between the two launches of a step keeps the tail from
    # starting as a programmatic dependent of the streaming kernel (~15 us per
    # step), so the headline region above runs without them.
    ctx.set_option(ht.OPT_PROFILE_EVENTS, 1)
    ctx.reset_timing()
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    vals, _ = ht.ht_rise_update_many(rep, batches(args.warmup, args.steps))
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    rep = vals[-1]
    ms_instr = e0.elapsed_time(e1) / args.steps
    fused_ms, fused_calls, _, _ = ctx.kernel_timing()
    ctx.set_option(ht.OPT_PROFILE_EVENTS, 0)
    if dist is not None:
        t = torch.tensor([ms, call_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, call_ms = float(t[0].item()), float(t[1].item())
    value = global_bytes / (ms * 1e-3) / 1e9
    call_value = global_bytes / (call_ms * 1e-3) / 1e9

    # end to end through the public API: pinned host batch -> H2D -> update
    e2e = None
    if args.e2e_steps > 0:
        host = pool[0].cpu().pin_memory()
        host_np = host.numpy().reshape(tuple(reversed(shape))).transpose()  # canonical, zero copy
        # untimed warm-up: the first host-input call grows the device pool by
        # one batch-sized upload buffer
        rep, _ = ht.ht_rise_update(rep, host_np)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            rep, upd = ht.ht_rise_update(rep, host_np)
            _ = upd.proj_error  # the scalar result is read back on the host
        t1 = time.perf_counter()
        e2e_ms = (t1 - t0) * 1e3 / args.e2e_steps
        if dist is not None:
            t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": global_bytes / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": local_bytes,
               "d2h_bytes_per_step": 16, "ms_per_step": e2e_ms, "steps": args.e2e_steps,
               "host_buffer": "pinned", "d2h": "||y||^2 and ||latent||^2, written by the tail kernel to mapped host memory"}

    # the step after the path: decode one batch's latents
    # into device memory, and relative_test_error's summand of one batch
    # (encode + residual decode, the reconstruction compared in HBM)
    recon = None
    if args.decode_steps > 0:
        yd = ht.DeviceTensor(pool[0], shape)
        lat, _ = ht.encode(rep, yd)
        lat_d = ht.DeviceTensor(torch.from_numpy(np.ascontiguousarray(lat.transpose(2, 1, 0))).cuda(), lat.shape)
        out_d = ht.DeviceTensor(pool[-1], shape)  # the last use of this pool slot
        rel = ht.relative_error(rep, yd)  # warm-up (also the residual path's workspace)
        ht.decode(rep, lat_d, out=out_d)
        ctx.synchronize()

        def timed(fn):
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(args.decode_steps):
                fn()
            e1.record(stream)
            e1.synchronize()
            t = e0.elapsed_time(e1) / args.decode_steps
            if dist is not None:
                tt = torch.tensor([t], device="cuda", dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt.item())
            return t

        dec_ms = timed(lambda: ht.decode(rep, lat_d, out=out_d))
        rte_ms = timed(lambda: ht.relative_error(rep, yd))
        recon = {"decode": {"ms_per_batch": dec_ms, "value": global_bytes / (dec_ms * 1e-3) / 1e9,
                            "unit": "GB/s of reconstruction written", "kernel": "expand_kernel + decode2_kernel"},
                 "relative_error": {"ms_per_batch": rte_ms, "value": global_bytes / (rte_ms * 1e-3) / 1e9,
                                    "unit": "GB/s of test tensor", "rte": rel,
                                    "kernels": "fused3 + tail3 (encode), expand + decode2<resid> (nothing written)"},
                 "calls": args.decode_steps, "timing": "CUDA events around back-to-back C-ABI calls, device in/out"}

    peak, peak_kind = _peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            # (measured on config 5's fused kernel; other configs: not captured)
            traffic = json.load(f)["traffic_bytes"] * (local_bytes / (8 * 128 ** 3 * 256)) if args.config == "c5" else None
    except Exception:
        pass
    roof = None
    if fused_calls:
        avg = fused_ms / fused_calls
        achieved = local_bytes / (avg * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": _first_kernel_label(args.config),
                "kernel_ms": avg, "share_of_step": avg / ms_instr, "peak_kind": peak_kind,
                "timed_in": {"region": "an instrumented repeat of the timed region (same K batches, same stream, "
                                       "CUDA events around the kernel of every step)",
                             "ms_per_step": ms_instr, "launches": int(fused_calls)},
                "algorithmic_bytes_per_launch": local_bytes,
                "frac_of_nominal_8000": achieved / HBM_NOMINAL_GBS}
        # the same kernel against the FP64 tensor pipe (c5 sits
        # at the FP64/HBM ridge): per slab (s, i2) it contracts n0 x n1 with
        # U1 (n1 x r1) and then U0^T (r0 x n0); DMMA tiles pad r to 8
        rk = rep.ranks()
        if len(w.dims) == 3 and (1, 0) in rk and (2, 0) in rk:
            n0, n1, n2 = w.dims
            r0, r1 = rk[(1, 0)], rk[(2, 0)]
            pad = lambda r: -(-r // 8) * 8  # noqa: E731
            slabs = n_local * n2
            flops = 2.0 * slabs * (n0 * n1 * r1 + r0 * n0 * r1)
            flops_issued = 2.0 * slabs * (n0 * n1 * pad(r1) + pad(r0) * n0 * pad(r1))
            tf = flops / (avg * 1e-3) / 1e12
            # the whole update: both floors (one read of Y at the measured HBM
            # peak; the algorithmic FP64 work of fused3 + tail3 at the measured
            # DMMA peak) against the measured step time
            rt = rk.get((1, 1), 0)
            r2 = rk.get((2, 1), 0)
            # a full-rank transfer node (rt = r1 r2) holds the identity basis
            # (BHT-l2r's Cholesky-certified shortcut): its projection is no work
            ident = rt == r1 * r2 and np.array_equal(rep.basis_matrix((1, 1)), np.eye(rt))
            tail_flops = 2.0 * n_local * (r0 * r1 * n2 * r2 + (0 if ident else r0 * (r1 * r2) * rt))
            t_hbm = local_bytes / (peak * 1e9) * 1e3
            t_fp64 = (flops + tail_flops) / (FP64_DMMA_TFLOPS * 1e12) * 1e3
            floor = max(t_hbm, t_fp64)
            roof["update"] = {"hbm_floor_ms": t_hbm, "fp64_floor_ms": t_fp64, "binding": "fp64" if t_fp64 > t_hbm else "hbm",
                              "algorithmic_flops": flops + tail_flops, "identity_transfer": bool(ident),
                              "ms_per_step": ms, "frac": floor / ms,
                              "hbm_frac": t_hbm / ms}
            roof["fp64_pipe"] = {"achieved": tf, "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s",
                                 "frac": tf / FP64_DMMA_TFLOPS,
                                 "issued_frac": flops_issued / (avg * 1e-3) / 1e12 / FP64_DMMA_TFLOPS,
                                 "algorithmic_flops_per_launch": flops, "issued_flops_per_launch": flops_issued,
                                 "peak_kind": "measured: DMMA.8x8x4 microbenchmark, profiles/r1_microbench_fp64.txt"}

    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_reference(1, 0, budget_s=args.cpu_seconds)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{args.config}: {w.description}", "batch_bytes": global_bytes,
                           "samples_per_gpu": n_local, "parallelism": f"batch-shard x{world}",
                           "l2": f"{pool_n} distinct resident batches of {local_bytes / 1e6:.0f} MB cycled "
                                 f"({pool_n * local_bytes / 1e6:.0f} MB > 126 MB L2, no flush needed)",
                           "distinct_batches": pool_n, "api": "ht_rise_update_many (K batches, one stream)",
                           "skipped_updates": stream_skipped, "fused_path_updates": stream_fused},
                "per_call": {"api": "ht_rise_update, one call per batch (host round trip per decision)",
                             "value": call_value, "ms_per_step": call_ms, "skipped_updates": skipped,
                             "fused_path_updates": fused_used, "gpu_launches": int(call_launches)},
                "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks2.summary(), "clocks_per_call": clocks.summary(), "reconstruction": recon}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--pool", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--decode-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=30.0)
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "ours" and args.gpus > 1 and env_world is None:
        # one process per GPU: launch ourselves under torchrun
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
