// Skip-path tail for balanced 4-way trees ((1,2),(3,4)) (config 3): after
// fused3_kernel has projected modes 0 and 1 slab by slab (W = [r0 r1, n2, n3, S]),
// one CTA per sample s finishes the encode (bht.hpp:381-399):
//
//   T[col, a]      = sum_q  W_s[q, col] B12[q, a]            col = i2 + n2 i3, q = a0 + r0 a1
//   V[i3, c2, a]   = sum_i2 T[(i2, i3), a] U2[i2, c2]
//   X[a, c2, c3]   = sum_i3 V[i3, c2, a] U3[i3, c3]
//   latent_s[a, b] = sum_j  X[a, j] B34[j, b]                j = c2 + r2 c3
//   ||latent_s||^2
//
// The transfer over leaves (1,2) is applied FIRST: it shrinks the r0 r1 rows
// of W_s to r12 before the remaining leaves are touched, so every later step
// is tiny. The mode products commute, so the result equals the reference's
// leaves-then-transfers order up to rounding. With few samples (config 3: 16)
// each sample is split over a thread-block cluster of up to 8 CTAs, one or
// more i3 slices each, whose partial X land in the rank-0 CTA through
// distributed shared memory and are summed there in CTA order. Step 1 is the only sizeable
// contraction (ncols x r12 x r0 r1) and runs on the FP64 tensor cores with W
// read straight from L2 (fused3 has just written it); the rest are plain
// DFMA loops over shared memory. The last CTA to finish (ticket counter) also
// reduces ||y||^2 (fused3's per-CTA partials) and ||latent||^2 in a fixed
// order. Replaces two leaf projections, two transfer projections, the latent
// norm pass and two scalar reductions (7 launches) of the generic path.
#include <cooperative_groups.h>

#include <algorithm>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace htr {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

// pitch (doubles) of the staged B12 columns: = 4 (mod 16), so the B-fragment
// reads (k = t4, column g4) of a half-warp fall into distinct bank pairs
__host__ __device__ __forceinline__ int b12_pitch(int R01) {
    int p = R01 + ((4 - R01 % 16) + 16) % 16;
    return p;
}

// This CTA's columns of W_s: the i3 slices crank, crank + C, ... (C = CTAs per
// sample), n2 columns each; local column lc -> column i2 + n2 i3 of W_s.
struct ColMap {
    int n2, crank, C, ncols;  // ncols = n2 * (owned slices)
    __device__ __forceinline__ int global(int lc) const {
        const int seg = lc / n2;
        return (lc - seg * n2) + n2 * (crank + C * seg);
    }
};

// T tiles for G m-tiles (8 local columns each) x NT n-tiles (8 outputs a)
template <int G, int NT>
__device__ __forceinline__ void step1_group(const double* __restrict__ W, const double* Bs, double* Ts, int R01,
                                            int pitchB, const ColMap& cm, int tpitch, int r12, int mt0, int nt0, int g4,
                                            int t4) {
    double acc[G][NT][2];
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* wp[G];
    bool ok[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int lc = 8 * (mt0 + kWarps * i) + g4;
        ok[i] = lc < cm.ncols;
        wp[i] = W + static_cast<int64_t>(R01) * (ok[i] ? cm.global(lc) : 0);
    }
    auto load = [&](int k, double (&av)[G]) {
#pragma unroll
        for (int i = 0; i < G; ++i) av[i] = (ok[i] && k < R01) ? __ldcg(wp[i] + k) : 0.0;
    };
    double cur[G], nxt[G];
    load(t4, cur);
    load(t4 + 4, nxt);
    for (int k0 = 0; k0 < R01; k0 += 4) {
        double fut[G];
        load(k0 + 8 + t4, fut);
        const int k = k0 + t4;
        double b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = Bs[k + pitchB * (8 * (nt0 + j) + g4)];  // zero-padded rows/columns
#pragma unroll
        for (int i = 0; i < G; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma(acc[i][j], cur[i], b[j]);
#pragma unroll
        for (int i = 0; i < G; ++i) {
            cur[i] = nxt[i];
            nxt[i] = fut[i];
        }
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int lc = 8 * (mt0 + kWarps * i) + g4;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a = 8 * (nt0 + j) + 2 * t4 + h;
                if (lc < cm.ncols && a < r12) Ts[lc + tpitch * a] = acc[i][j][h];
            }
    }
}

// the m-tiles of one warp for NT n-tiles starting at nt0
template <int NT>
__device__ __forceinline__ void step1_tiles(const double* __restrict__ W, const double* Bs, double* Ts, int R01,
                                            int pitchB, const ColMap& cm, int tpitch, int r12, int warp, int nt0,
                                            int g4, int t4) {
    const int mtA = (cm.ncols + 7) / 8;
    const int cnt = warp < mtA ? (mtA - warp + kWarps - 1) / kWarps : 0;
    int t = 0;
    for (; cnt - t >= 4; t += 4) step1_group<4, NT>(W, Bs, Ts, R01, pitchB, cm, tpitch, r12, warp + kWarps * t, nt0, g4, t4);
    if (cnt - t >= 2) {
        step1_group<2, NT>(W, Bs, Ts, R01, pitchB, cm, tpitch, r12, warp + kWarps * t, nt0, g4, t4);
        t += 2;
    }
    if (cnt - t >= 1) step1_group<1, NT>(W, Bs, Ts, R01, pitchB, cm, tpitch, r12, warp + kWarps * t, nt0, g4, t4);
}

// own: the most i3 slices a CTA owns = ceil(n3 / C)
__host__ __device__ __forceinline__ int64_t tail4_smem_doubles(int R01, int r12, int r2, int r3, int64_t n2, int own,
                                                               int C) {
    const int nt = (r12 + 7) / 8;
    const int64_t xs = static_cast<int64_t>(r12) * (r2 * r3 + 1);
    return static_cast<int64_t>(8 * nt) * b12_pitch(R01) + 8 + static_cast<int64_t>(r12) * (n2 * own + 1) +
           static_cast<int64_t>(own) * r2 * r12 + xs * (C > 1 ? C : 1);
}

template <bool CL>
__global__ void __launch_bounds__(kThreads) tail4_kernel(const Tail4Args a) {
    extern __shared__ __align__(16) double sm[];
    const int r2 = a.r2, r3 = a.r3, r12 = a.r12, r34 = a.r34, R01 = a.R01;
    const int n2 = static_cast<int>(a.n2), n3 = static_cast<int>(a.n3);
    // the sample's i3 slices are dealt round-robin to the C CTAs of its cluster
    const int C = CL ? a.csize : 1;
    const int crank = CL ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
    const int own = crank < n3 ? (n3 - crank + C - 1) / C : 0;
    const int own_max = (n3 + C - 1) / C;
    const ColMap cm{n2, crank, C, n2 * own};
    const int pitchB = b12_pitch(R01);
    const int tpitch = n2 * own_max + 1;
    const int ntiles = (r12 + 7) / 8;
    const int R23 = r2 * r3, xpitch = R23 + 1;
    double* Bs = sm;                            // [8 ntiles][pitchB] (+ 8 doubles of slack for the k overrun)
    double* Ts = Bs + 8 * ntiles * pitchB + 8;  // [r12][tpitch]
    double* Vs = Ts + r12 * tpitch;             // [own][r2][r12]
    double* Xs = Vs + own_max * r2 * r12;       // [C][r12][xpitch]: every CTA's partial X (rank 0's copy is summed)
    __shared__ double red[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int64_t s = blockIdx.x / C;

    // the transfer basis over leaves (1,2), zero-padded to whole tiles
    for (int e = tid; e < 8 * ntiles * pitchB + 8; e += kThreads) {
        const int c = e / pitchB, q = e - c * pitchB;
        Bs[e] = (c < r12 && q < R01) ? a.B12[q + static_cast<int64_t>(R01) * c] : 0.0;
    }
    __syncthreads();
    // launched as a programmatic dependent of the fused leaf kernel: its W
    // and ||y||^2 partials are complete and visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- step 1: T = W_s^T B12 on DMMA (M = this CTA's columns of W_s, N = r12,
    // K = R01), the n-tiles in groups of up to three (W_s, L2-resident, is
    // re-read per group)
    {
        const double* W = a.W + s * static_cast<int64_t>(R01) * n2 * n3;
        for (int nt0 = 0; nt0 < ntiles; nt0 += 3) {
            const int nt = min(3, ntiles - nt0);
            if (nt == 3) step1_tiles<3>(W, Bs, Ts, R01, pitchB, cm, tpitch, r12, warp, nt0, g4, t4);
            else if (nt == 2) step1_tiles<2>(W, Bs, Ts, R01, pitchB, cm, tpitch, r12, warp, nt0, g4, t4);
            else step1_tiles<1>(W, Bs, Ts, R01, pitchB, cm, tpitch, r12, warp, nt0, g4, t4);
        }
    }
    __syncthreads();

    // ---- step 2: V[l3, c2, a] = sum_i2 T[(i2, l3), a] U2[i2, c2] (l3: owned slice) ----
    for (int e = tid; e < own * r2 * r12; e += kThreads) {
        // a fastest: the odd pitch of T keeps a warp's reads conflict-free
        const int aa = e % r12, c2 = (e / r12) % r2, l3 = e / (r12 * r2);
        const double* t = Ts + tpitch * aa + n2 * l3;
        const double* u = a.U2 + static_cast<int64_t>(n2) * c2;
        double v0 = 0.0, v1 = 0.0;
        int i2 = 0;
        for (; i2 + 1 < n2; i2 += 2) {
            v0 = fma(t[i2], __ldg(u + i2), v0);
            v1 = fma(t[i2 + 1], __ldg(u + i2 + 1), v1);
        }
        if (i2 < n2) v0 = fma(t[i2], __ldg(u + i2), v0);
        Vs[l3 + own_max * (c2 + r2 * aa)] = v0 + v1;
    }
    __syncthreads();

    // ---- step 3: this CTA's part of X[a, c2 + r2 c3] = sum_i3 V[i3, c2, a] U3[i3, c3],
    // written into slot crank of the cluster's rank-0 CTA (distributed shared memory)
    {
        double* xdst = Xs + static_cast<int64_t>(crank) * r12 * xpitch;
        if constexpr (CL) xdst = cg::this_cluster().map_shared_rank(xdst, 0);
        for (int e = tid; e < r12 * R23; e += kThreads) {
            const int c2 = e % r2, c3 = (e / r2) % r3, aa = e / R23;
            const double* v = Vs + own_max * (c2 + r2 * aa);
            const double* u = a.U3 + static_cast<int64_t>(n3) * c3;
            double x = 0.0;
            for (int l3 = 0; l3 < own; ++l3) x = fma(v[l3], __ldg(u + crank + C * l3), x);
            xdst[aa * xpitch + c2 + r2 * c3] = x;
        }
    }
    if constexpr (CL) {
        cg::this_cluster().sync();  // every part has landed in rank 0 (no DSMEM access after this)
        if (crank != 0) return;
        // the parts summed in CTA order (deterministic)
        for (int e = tid; e < r12 * xpitch; e += kThreads) {
            double x = Xs[e];
            for (int q = 1; q < C; ++q) x += Xs[static_cast<int64_t>(q) * r12 * xpitch + e];
            Xs[e] = x;
        }
    }
    __syncthreads();

    // ---- step 4: latent_s[a, b] = sum_j X[a, j] B34[j, b] ----
    double* out = a.latent + s * static_cast<int64_t>(r12) * r34;
    double lsq = 0.0;
    for (int e = tid; e < r12 * r34; e += kThreads) {
        const int aa = e % r12, b = e / r12;
        const double* x = Xs + aa * xpitch;
        const double* bb = a.B34 + static_cast<int64_t>(R23) * b;
        double v0 = 0.0, v1 = 0.0;
        int j = 0;
        for (; j + 1 < R23; j += 2) {
            v0 = fma(x[j], __ldg(bb + j), v0);
            v1 = fma(x[j + 1], __ldg(bb + j + 1), v1);
        }
        if (j < R23) v0 = fma(x[j], __ldg(bb + j), v0);
        const double v = v0 + v1;
        out[e] = v;
        lsq = fma(v, v, lsq);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsq += __shfl_xor_sync(0xffffffffu, lsq, o);
    if (lane == 0) red[warp] = lsq;
    __syncthreads();
    __shared__ bool last;
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        a.latsq[s] = t;
        __threadfence();
        last = atomicAdd(a.ticket, 1u) == static_cast<unsigned>(a.S) - 1;  // one ticket per sample
    }
    __syncthreads();
    if (!last) return;
    // last CTA: both scalar reductions in a fixed order (deterministic no
    // matter which CTA finishes last)
    __threadfence();
    double ys = 0.0, ls = 0.0;
    for (int64_t i = tid; i < a.n_ysq; i += kThreads) ys += __ldcg(a.ysq_partials + i);
    for (int64_t i = tid; i < a.S; i += kThreads) ls += __ldcg(a.latsq + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ys += __shfl_xor_sync(0xffffffffu, ys, o);
        ls += __shfl_xor_sync(0xffffffffu, ls, o);
    }
    __shared__ double red2[2][kWarps];
    if (lane == 0) {
        red2[0][warp] = ys;
        red2[1][warp] = ls;
    }
    __syncthreads();
    if (tid == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < kWarps; ++w) {
            t0 += red2[0][w];
            t1 += red2[1][w];
        }
        a.out[0] = t0;
        a.out[2] = t1;
        if (a.host_out) {
            a.host_out[0] = t0;
            a.host_out[2] = t1;
        }
        *a.ticket = 0u;
    }
}

// CTAs per sample: split while the grid stays within two CTAs per SM, every
// CTA keeps at least one i3 slice and the shared memory fits
int tail4_csize(const Tail4Args& a, int num_sms) {
    int c = 1;
    while (c < 8 && 2 * c <= a.n3 && a.S * 2 * c <= 2 * static_cast<int64_t>(num_sms) &&
           8 * tail4_smem_doubles(a.R01, a.r12, a.r2, a.r3, a.n2, static_cast<int>((a.n3 + 2 * c - 1) / (2 * c)), 2 * c) <=
               200 * 1024)
        c *= 2;
    return c;
}

void launch_t(const Tail4Args& a, size_t smem, cudaStream_t s) {
    const bool cl = a.csize > 1;
    if (smem > 46 * 1024)
        ensure_smem_limit(cl ? reinterpret_cast<const void*>(tail4_kernel<true>)
                             : reinterpret_cast<const void*>(tail4_kernel<false>),
                          smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(a.S * a.csize));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(a.csize);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cl ? 2 : 1;
    if (cl)
        cudaLaunchKernelEx(&cfg, tail4_kernel<true>, a);
    else
        cudaLaunchKernelEx(&cfg, tail4_kernel<false>, a);
}

}  // namespace

bool tail4_supported(int R01, int r12, int r34, int r2, int r3, int64_t n2, int64_t n3) {
    if (R01 < 1 || r12 < 1 || r34 < 1 || r2 < 1 || r3 < 1 || r12 > 96 || R01 > 576 || r2 > 24 || r3 > 24) return false;
    if (n2 < 1 || n3 < 1 || n2 * n3 > 4096) return false;
    return 8 * tail4_smem_doubles(R01, r12, r2, r3, n2, static_cast<int>(n3), 1) <= 200 * 1024;
}

void launch_tail4(const Tail4Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    Tail4Args b = a;
    b.csize = tail4_csize(a, num_sms);
    const int own = static_cast<int>((a.n3 + b.csize - 1) / b.csize);
    const size_t smem = 8 * static_cast<size_t>(tail4_smem_doubles(a.R01, a.r12, a.r2, a.r3, a.n2, own, b.csize));
    launch_t(b, smem, s);
    ++*launches;
}

}  // namespace htr
