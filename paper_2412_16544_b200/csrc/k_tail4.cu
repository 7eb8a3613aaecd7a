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
// leaves-then-transfers order up to rounding. Step 1 is the only sizeable
// contraction (ncols x r12 x r0 r1) and runs on the FP64 tensor cores with W
// read straight from L2 (fused3 has just written it); the rest are plain
// DFMA loops over shared memory. The last CTA to finish (ticket counter) also
// reduces ||y||^2 (fused3's per-CTA partials) and ||latent||^2 in a fixed
// order. Replaces two leaf projections, two transfer projections, the latent
// norm pass and two scalar reductions (7 launches) of the generic path.
#include <algorithm>

#include "kernels.cuh"

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

// T tiles for G m-tiles (8 columns of W_s each) x NT n-tiles (8 outputs a)
template <int G, int NT>
__device__ __forceinline__ void step1_group(const double* __restrict__ W, const double* Bs, double* Ts, int R01,
                                            int pitchB, int ncols, int tpitch, int r12, int mt0, int g4, int t4) {
    double acc[G][NT][2];
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* wp[G];
    bool ok[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int col = 8 * (mt0 + kWarps * i) + g4;
        ok[i] = col < ncols;
        wp[i] = W + static_cast<int64_t>(R01) * (ok[i] ? col : 0);
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
        for (int j = 0; j < NT; ++j) b[j] = Bs[k + pitchB * (8 * j + g4)];  // zero-padded rows/columns
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
        const int col = 8 * (mt0 + kWarps * i) + g4;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a = 8 * j + 2 * t4 + h;
                if (col < ncols && a < r12) Ts[col + tpitch * a] = acc[i][j][h];
            }
    }
}

template <int NT>
__global__ void __launch_bounds__(kThreads) tail4_kernel(const Tail4Args a) {
    extern __shared__ __align__(16) double sm[];
    const int r2 = a.r2, r3 = a.r3, r12 = a.r12, r34 = a.r34, R01 = a.R01;
    const int n2 = static_cast<int>(a.n2), n3 = static_cast<int>(a.n3);
    const int ncols = n2 * n3;
    const int pitchB = b12_pitch(R01);
    const int tpitch = ncols + 1;
    double* Bs = sm;                        // [8 NT][pitchB] (+ 8 doubles of slack for the k overrun)
    double* Ts = Bs + 8 * NT * pitchB + 8;  // [r12][tpitch]
    double* Vs = Ts + r12 * tpitch;         // [n3][r2][r12]
    double* Xs = Vs + n3 * r2 * r12;        // [r12][r2 r3]
    __shared__ double red[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int64_t s = blockIdx.x;

    // the transfer basis over leaves (1,2), zero-padded to whole tiles
    for (int e = tid; e < 8 * NT * pitchB + 8; e += kThreads) {
        const int c = e / pitchB, q = e - c * pitchB;
        Bs[e] = (c < r12 && q < R01) ? a.B12[q + static_cast<int64_t>(R01) * c] : 0.0;
    }
    __syncthreads();
    // launched as a programmatic dependent of the fused leaf kernel: its W
    // and ||y||^2 partials are complete and visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- step 1: T = W_s^T B12 on DMMA (M = columns of W_s, N = r12, K = R01) ----
    {
        const double* W = a.W + s * static_cast<int64_t>(R01) * ncols;
        const int mtA = (ncols + 7) / 8;
        const int cnt = warp < mtA ? (mtA - warp + kWarps - 1) / kWarps : 0;
        int t = 0;
        for (; cnt - t >= 4; t += 4) step1_group<4, NT>(W, Bs, Ts, R01, pitchB, ncols, tpitch, r12, warp + kWarps * t, g4, t4);
        if (cnt - t >= 2) {
            step1_group<2, NT>(W, Bs, Ts, R01, pitchB, ncols, tpitch, r12, warp + kWarps * t, g4, t4);
            t += 2;
        }
        if (cnt - t >= 1) step1_group<1, NT>(W, Bs, Ts, R01, pitchB, ncols, tpitch, r12, warp + kWarps * t, g4, t4);
    }
    __syncthreads();

    // ---- step 2: V[i3, c2, a] = sum_i2 T[(i2, i3), a] U2[i2, c2] ----
    for (int e = tid; e < n3 * r2 * r12; e += kThreads) {
        // a fastest: the odd pitch of T keeps a warp's reads conflict-free
        const int aa = e % r12, c2 = (e / r12) % r2, i3 = e / (r12 * r2);
        const double* t = Ts + tpitch * aa + n2 * i3;
        const double* u = a.U2 + static_cast<int64_t>(n2) * c2;
        double v0 = 0.0, v1 = 0.0;
        int i2 = 0;
        for (; i2 + 1 < n2; i2 += 2) {
            v0 = fma(t[i2], __ldg(u + i2), v0);
            v1 = fma(t[i2 + 1], __ldg(u + i2 + 1), v1);
        }
        if (i2 < n2) v0 = fma(t[i2], __ldg(u + i2), v0);
        Vs[i3 + n3 * (c2 + r2 * aa)] = v0 + v1;
    }
    __syncthreads();

    // ---- step 3: X[a, c2 + r2 c3] = sum_i3 V[i3, c2, a] U3[i3, c3] ----
    const int R23 = r2 * r3;
    for (int e = tid; e < r12 * R23; e += kThreads) {
        const int c2 = e % r2, c3 = (e / r2) % r3, aa = e / R23;
        const double* v = Vs + n3 * (c2 + r2 * aa);
        const double* u = a.U3 + static_cast<int64_t>(n3) * c3;
        double x = 0.0;
        for (int i3 = 0; i3 < n3; ++i3) x = fma(v[i3], __ldg(u + i3), x);
        Xs[aa * (R23 + 1) + c2 + r2 * c3] = x;
    }
    __syncthreads();

    // ---- step 4: latent_s[a, b] = sum_j X[a, j] B34[j, b] ----
    double* out = a.latent + s * static_cast<int64_t>(r12) * r34;
    double lsq = 0.0;
    for (int e = tid; e < r12 * r34; e += kThreads) {
        const int aa = e % r12, b = e / r12;
        const double* x = Xs + aa * (R23 + 1);
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
        last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
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

size_t tail4_smem(int R01, int r12, int r2, int r3, int64_t n2, int64_t n3) {
    const int nt = (r12 + 7) / 8;
    const size_t ncols = static_cast<size_t>(n2 * n3);
    return sizeof(double) * (static_cast<size_t>(8 * nt) * b12_pitch(R01) + 8 + static_cast<size_t>(r12) * (ncols + 1) +
                             static_cast<size_t>(n3) * r2 * r12 + static_cast<size_t>(r12) * (r2 * r3 + 1));
}

template <int NT>
void launch_t(const Tail4Args& a, size_t smem, cudaStream_t s) {
    if (smem > 46 * 1024) ensure_smem_limit(reinterpret_cast<const void*>(tail4_kernel<NT>), smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(a.S));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, tail4_kernel<NT>, a);
}

}  // namespace

bool tail4_supported(int R01, int r12, int r34, int r2, int r3, int64_t n2, int64_t n3) {
    if (R01 < 1 || r12 < 1 || r34 < 1 || r2 < 1 || r3 < 1 || r12 > 24 || R01 > 576 || r2 > 24 || r3 > 24) return false;
    if (n2 < 1 || n3 < 1 || n2 * n3 > 4096) return false;
    return tail4_smem(R01, r12, r2, r3, n2, n3) <= 200 * 1024;
}

void launch_tail4(const Tail4Args& a, cudaStream_t s, int64_t* launches) {
    const size_t smem = tail4_smem(a.R01, a.r12, a.r2, a.r3, a.n2, a.n3);
    switch ((a.r12 + 7) / 8) {
        case 1: launch_t<1>(a, smem, s); break;
        case 2: launch_t<2>(a, smem, s); break;
        default: launch_t<3>(a, smem, s); break;
    }
    ++*launches;
}

}  // namespace htr
