"""Seeded synthetic stand-ins for the five BASELINE.json configs.

The paper measures on PDEBench / gels / BigEarthNet / MineRL data
(PAPER.md:1509-1801), none of which is available here; these generators
reproduce the *shapes, sizes and value models* BASELINE.json names instead
(SURVEY.md §8(d), Appendix B). Generation is plumbing: it runs in torch on
the target device, untimed, and each batch is a flat float64 tensor in the
reference's canonical order (first index fastest).

Pinned readings of the ambiguities listed in SURVEY.md Appendix B:
  c1  noise N(0, 1e-12) read as variance -> sigma = 1e-6; factor vectors
      shared by the batch, weights per sample; seed 0.
  c2  periodic grid x_i = 2 pi i / 64; t = global sample index in the stream;
      noise sigma = 1e-6 absolute; seed 2.
  c3  6 components (per-mode orthonormal Gaussian factors, N(0,1) weights per
      sample); from batch 25 (1-based) 6 more switch on and all 12 stay on;
      the 8-long field mode holds 12 factors (first 8 orthonormal, 4 more
      Gaussian unit vectors); noise 1e-5 relative to the batch norm (an
      absolute 1e-5 would put ||noise||/||Y|| ~ 2e-3 above eps = 1e-3 and make
      every leaf full-rank, contradicting the config's 6 -> 12 rank story);
      seed 3.
  c4  leaf bases and transfer tensors fixed per stream, root coefficients
      per sample; noise 1e-4 relative per sample; seed 4.
  c5  factors fixed per stream, core 20^3 N(0,1) per sample; noise 1e-4
      relative per sample (drawn per group of 16 samples so that shards of a
      multiple of 16 samples reproduce the unsharded bytes); seed 5.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Tuple

import torch

from . import htrise as ht


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _orth(rows: int, cols: int, g, device) -> torch.Tensor:
    a = torch.randn(rows, cols, generator=g, device=device, dtype=torch.float64)
    q, _ = torch.linalg.qr(a)
    return q


@dataclass
class Workload:
    name: str
    dims: Tuple[int, ...]
    batch: int
    n_batches: int
    eps: float
    tree_kind: str  # "balanced" or "1_23"
    seed: int
    description: str

    def tree(self) -> "ht.DimensionTree":
        if self.tree_kind == "1_23":
            return ht.tree_1_23()
        return ht.DimensionTree.balanced(len(self.dims))

    @property
    def shape(self) -> Tuple[int, ...]:
        return tuple(self.dims) + (self.batch,)

    @property
    def bytes_per_batch(self) -> int:
        return 8 * int(math.prod(self.shape))

    def make_batch(self, b: int, device="cuda", batch: int | None = None, sample_offset: int = 0) -> torch.Tensor:
        """Flat float64 tensor of batch b (0-based) in canonical order. With
        `batch`/`sample_offset` it yields a shard of the batch (multi-GPU)."""
        n = self.batch if batch is None else batch
        return _MAKERS[self.name](self, b, torch.device(device), n, sample_offset)


# ---- c1 -------------------------------------------------------------------

def _c1(w: Workload, b: int, dev, n: int, off: int) -> torch.Tensor:
    g = _gen(dev, w.seed)
    R = 5
    facs = [torch.randn(w.dims[k], R, generator=g, device=dev, dtype=torch.float64) for k in range(4)]
    weights = torch.randn(w.batch, R, generator=g, device=dev, dtype=torch.float64)[off:off + n]
    # torch C-order (s, i3, i2, i1, i0) == canonical (i0, i1, i2, i3, s)
    y = torch.einsum("sr,ar,br,cr,dr->sdcba", weights, facs[0], facs[1], facs[2], facs[3])
    gn = _gen(dev, 1000 + w.seed * 7919 + b)
    noise = torch.randn(w.batch, *y.shape[1:], generator=gn, device=dev, dtype=torch.float64)[off:off + n]
    return (y + 1e-6 * noise).contiguous().reshape(-1)


# ---- c2 -------------------------------------------------------------------

def _c2(w: Workload, b: int, dev, n: int, off: int) -> torch.Tensor:
    g = _gen(dev, w.seed)
    J = 8
    k = torch.randint(1, 7, (J, 3), generator=g, device=dev).to(torch.float64)
    ph = 2 * math.pi * torch.rand(J, 3, generator=g, device=dev, dtype=torch.float64)
    om = 0.01 + 0.09 * torch.rand(J, generator=g, device=dev, dtype=torch.float64)
    x = 2 * math.pi * torch.arange(w.dims[0], device=dev, dtype=torch.float64) / w.dims[0]
    f = [torch.sin(k[:, a:a + 1] * x[None, :] + ph[:, a:a + 1]) for a in range(3)]  # J x 64 each
    t = torch.arange(b * w.batch + off, b * w.batch + off + n, device=dev, dtype=torch.float64)
    amp = torch.cos(om[None, :] * t[:, None])  # n x J
    y = torch.einsum("sj,ja,jb,jc->scba", amp, f[0], f[1], f[2])
    gn = _gen(dev, 2000 + b)
    noise = torch.randn(w.batch, *y.shape[1:], generator=gn, device=dev, dtype=torch.float64)[off:off + n]
    return (y + 1e-6 * noise).contiguous().reshape(-1)


# ---- c3 -------------------------------------------------------------------

def _c3(w: Workload, b: int, dev, n: int, off: int) -> torch.Tensor:
    g = _gen(dev, w.seed)
    facs = []
    for k in range(4):
        nk = w.dims[k]
        if nk >= 12:
            facs.append(_orth(nk, 12, g, dev))
        else:
            q = _orth(nk, nk, g, dev)
            extra = torch.randn(nk, 12 - nk, generator=g, device=dev, dtype=torch.float64)
            extra = extra / extra.norm(dim=0, keepdim=True)
            facs.append(torch.cat([q, extra], dim=1))
    active = 12 if b >= 24 else 6
    gw = _gen(dev, 3000 + b)
    weights = torch.randn(w.batch, 12, generator=gw, device=dev, dtype=torch.float64)[off:off + n, :active]
    f = [fk[:, :active] for fk in facs]
    y = torch.einsum("sr,ar,br,cr,dr->sdcba", weights, f[0], f[1], f[2], f[3])
    gn = _gen(dev, 3500 + b)
    noise = torch.randn(w.batch, *y.shape[1:], generator=gn, device=dev, dtype=torch.float64)[off:off + n]
    # relative to the full batch's signal norm (weights of all samples)
    wfull = torch.randn(w.batch, 12, generator=_gen(dev, 3000 + b), device=dev, dtype=torch.float64)[:, :active]
    scale = 1e-5 * float(wfull.norm()) / math.sqrt(w.batch * math.prod(w.dims))
    return (y + scale * noise).contiguous().reshape(-1)


# ---- c4 -------------------------------------------------------------------

def _c4(w: Workload, b: int, dev, n: int, off: int) -> torch.Tensor:
    g = _gen(dev, w.seed)
    r = 4
    leaves = [_orth(8, r, g, dev) for _ in range(8)]
    transfers = {lvl: [torch.randn(r, r, r, generator=g, device=dev, dtype=torch.float64) for _ in range(cnt)]
                 for lvl, cnt in ((2, 4), (1, 2))}

    def combine(fl, fr, core):  # frame rows: a + n_left * b (first fastest)
        f = torch.einsum("ijk,ai,bj->bak", core, fl, fr)  # C-order (b, a, k): a fastest after reshape
        return f.reshape(fl.shape[0] * fr.shape[0], core.shape[2])

    l2 = [combine(leaves[2 * i], leaves[2 * i + 1], transfers[2][i]) for i in range(4)]
    l1 = [combine(l2[2 * i], l2[2 * i + 1], transfers[1][i]) for i in range(2)]
    gr = _gen(dev, 4000 + b)
    roots = torch.randn(w.batch, r, r, generator=gr, device=dev, dtype=torch.float64)[off:off + n]
    out = torch.empty(n, l1[1].shape[0], l1[0].shape[0], device=dev, dtype=torch.float64)
    gn = _gen(dev, 4500 + b)
    for s in range(n):
        # canonical (a, b) with a (left span) fastest == torch C-order (b, a)
        m = l1[1] @ roots[s].T @ l1[0].T
        out[s] = m
    noise = torch.randn(w.batch, *out.shape[1:], generator=gn, device=dev, dtype=torch.float64)[off:off + n]
    norms = out.reshape(n, -1).norm(dim=1) / math.sqrt(out[0].numel())
    out += 1e-4 * norms[:, None, None] * noise
    return out.reshape(-1)


# ---- c5 -------------------------------------------------------------------

def _c5(w: Workload, b: int, dev, n: int, off: int) -> torch.Tensor:
    g = _gen(dev, w.seed)
    r = 20
    A = [_orth(w.dims[k], r, g, dev) for k in range(3)]
    gc = _gen(dev, 5000 + b)
    out = torch.empty(n, w.dims[2], w.dims[1], w.dims[0], device=dev, dtype=torch.float64)
    numel = w.dims[0] * w.dims[1] * w.dims[2]
    # cores for the whole batch from one stream, then the shard's slice
    cores = torch.randn(w.batch, r, r, r, generator=gc, device=dev, dtype=torch.float64)[off:off + n]
    # noise per group of 16 samples from its own seed: identical bytes for
    # any sharding whose shard size is a multiple of 16
    group = 16
    s0 = 0
    while s0 < n:
        gidx = (off + s0) // group
        s1 = min(n, (gidx + 1) * group - off)
        c = cores[s0:s1]  # (s, a2, a1, a0) C-order
        y = torch.einsum("szyx,ix->szyi", c, A[0])
        y = torch.einsum("szyi,jy->szji", y, A[1])
        y = torch.einsum("szji,kz->skji", y, A[2])
        gn = _gen(dev, 5500 * 4096 + b * 4096 + gidx)
        lo = (off + s0) - gidx * group  # first sample of this piece within its group
        nz = torch.randn(group, numel, generator=gn, device=dev, dtype=torch.float64)[lo:lo + (s1 - s0)]
        sc = 1e-4 * y.reshape(s1 - s0, -1).norm(dim=1) / math.sqrt(numel)
        out[s0:s1] = y + (sc[:, None] * nz).reshape(y.shape)
        s0 = s1
    return out.reshape(-1)


_MAKERS = {"c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4, "c5": _c5}

CONFIGS = {
    "c1": Workload("c1", (16, 16, 16, 16), 64, 1, 1e-4, "balanced", 0,
                   "BHT-l2r one-shot, 16^4 x 64, 5 rank-1 terms, balanced tree, eps 1e-4"),
    "c2": Workload("c2", (64, 64, 64), 32, 20, 1e-3, "1_23", 2,
                   "HT-RISE stream, 64^3, 20 batches of 32, separable sinusoids, tree (1,(2,3)), eps 1e-3"),
    "c3": Workload("c3", (32, 32, 32, 8), 16, 50, 1e-3, "balanced", 3,
                   "HT-RISE with rank growth at batch 25, 32^3 x 8, 50 batches of 16, eps 1e-3"),
    "c4": Workload("c4", (8,) * 8, 4, 10, 1e-2, "balanced", 4,
                   "BHT-l2r then HT-RISE, 8^8, 10 batches of 4, random rank-4 HT, eps 1e-2"),
    "c5": Workload("c5", (128, 128, 128), 256, 40, 1e-3, "1_23", 5,
                   "throughput, 128^3, 40 batches of 256 (4.3 GB), Tucker rank 20, tree (1,(2,3)), eps 1e-3"),
}
