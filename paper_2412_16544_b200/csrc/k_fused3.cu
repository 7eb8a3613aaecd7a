// K1: fused all-leaf projection of a 3-way batch on the FP64 tensor cores.
//
// Replaces the skip-path hot loop of encode (reference bht.hpp:373-399 ->
// project_mode 357-365 -> unfold/GEMM/fold, tensor.hpp:150-205) and the
// frobenius_norm pass over y (ht_rise.hpp:111): for a batch Y[N0, N1, n2, S]
// (canonical, first index fastest) it computes in ONE read of Y
//
//     Z[a0, a1, a2, s] = sum_{i0,i1,i2} Y[i0,i1,i2,s] U0[i0,a0] U1[i1,a1] U2[i2,a2]
//     ||Y||^2
//
// which is the leaf-projected working tensor of encode for every 3-way tree
// ((1,(2,3)) and ((1,2),3)); the interior transfer projection then runs on
// the 1/(N0 N1 n2 / r0 r1 r2)-size Z.
//
// Data path per warp and slab X = Y[:, :, i2, s] (N0 x N1, contiguous):
//   step 1  P = U0^T X     (8x4x8 DMMA tiles; X fragments come straight from
//                           HBM into registers with 16-byte ld.global.nc, each
//                           element loaded exactly once, prefetched 8 chunks
//                           ahead; U0^T fragments from shared memory)
//   step 2  W = P U1       (P's accumulator fragments are re-used in
//                           registers as the A operand: the k index of the
//                           MMA is permuted to match the C layout)
//   step 3  Z_s += W (x) U2[i2, :]   (CTA-wide, shared-memory accumulators,
//                           flushed per sample to a partial buffer that a
//                           second kernel reduces in a fixed order).
// Everything is deterministic: no atomics, fixed reduction trees.
#include <algorithm>
#include <cstdio>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kPrefetch = 8;  // chunks of 8 rows in flight per warp
constexpr int kMaxZ = 8192;   // r0*r1*r2 accumulators kept in shared memory

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 ldg_stream(const double* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

struct RangeInfo {
    int64_t T;      // total slabs = n2 * S
    int64_t maxs;   // sample slots per CTA
};

__host__ __device__ __forceinline__ int64_t cta_begin(int64_t T, int64_t b, int64_t B) { return (T * b) / B; }

template <int N0, int N1, int MT0, int MT1>
__global__ void __launch_bounds__(kThreads, 1) fused3_kernel(const Fused3Args a, const RangeInfo ri) {
    constexpr int NC = N0 / 8;   // k-chunks (8 rows of i0) per column block
    constexpr int NP = N1 / 16;  // n-tile pairs per slab
    constexpr int STEPS = NP * NC;
    extern __shared__ __align__(16) double smem[];
    double2* U0f = reinterpret_cast<double2*>(smem);                 // [NC][MT0][32]
    double2* U1f = U0f + NC * MT0 * 32;                              // [N1/8][MT1][32]
    const int R01 = a.r0 * a.r1;
    const int R = R01 * a.r2;
    double* Wbuf = reinterpret_cast<double*>(U1f + (N1 / 8) * MT1 * 32);  // [2][kWarps][R01]
    double* Zs = Wbuf + 2 * kWarps * R01;                                   // [R]
    double* U2s = Zs + R;                                                   // [n2 * r2]
    __shared__ double red[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;

    // ---- stage basis fragments (zero-padded to 8-multiples) ----
    for (int idx = tid; idx < NC * MT0 * 32; idx += kThreads) {
        const int l = idx & 31, mt = (idx >> 5) % MT0, c = idx / (32 * MT0);
        const int i0 = 8 * c + 2 * (l & 3), col = 8 * mt + (l >> 2);
        double2 v;
        v.x = col < a.r0 ? a.U0[i0 + static_cast<int64_t>(N0) * col] : 0.0;
        v.y = col < a.r0 ? a.U0[i0 + 1 + static_cast<int64_t>(N0) * col] : 0.0;
        U0f[idx] = v;
    }
    for (int idx = tid; idx < (N1 / 8) * MT1 * 32; idx += kThreads) {
        const int l = idx & 31, mt = (idx >> 5) % MT1, nt = idx / (32 * MT1);
        const int i1 = 8 * nt + 2 * (l & 3), col = 8 * mt + (l >> 2);
        double2 v;
        v.x = col < a.r1 ? a.U1[i1 + static_cast<int64_t>(N1) * col] : 0.0;
        v.y = col < a.r1 ? a.U1[i1 + 1 + static_cast<int64_t>(N1) * col] : 0.0;
        U1f[idx] = v;
    }
    for (int e = tid; e < R; e += kThreads) Zs[e] = 0.0;
    for (int64_t e = tid; e < a.n2 * a.r2; e += kThreads) U2s[e] = a.U2[e];
    __syncthreads();

    const int64_t B = gridDim.x, b = blockIdx.x;
    const int64_t tb = cta_begin(ri.T, b, B), te = cta_begin(ri.T, b + 1, B);
    const int64_t ngroups = (te - tb + kWarps - 1) / kWarps;
    const int64_t s_first = tb / a.n2;
    const int64_t slab_elems = static_cast<int64_t>(N0) * N1;

    // prefetch stream: (group, pair, chunk) counters of the chunk kPrefetch
    // steps ahead of the one being consumed
    const int lane_off = 2 * t4 + N0 * g4;  // row offset in a chunk + column in an n-tile
    int64_t pf_g = 0;
    int pf_pair = 0, pf_c = 0;
    auto pf_issue = [&](double2 (&dst)[2]) {
        const int64_t t = tb + kWarps * pf_g + warp;
        if (t < te) {
            const double* p = a.Y + t * slab_elems + static_cast<int64_t>(16 * N0) * pf_pair + 8 * pf_c + lane_off;
            dst[0] = ldg_stream(p);
            dst[1] = ldg_stream(p + 8 * N0);
        } else {
            dst[0] = make_double2(0.0, 0.0);
            dst[1] = make_double2(0.0, 0.0);
        }
        if (++pf_c == NC) {
            pf_c = 0;
            if (++pf_pair == NP) {
                pf_pair = 0;
                ++pf_g;
            }
        }
    };

    double2 ring[kPrefetch][2];
#pragma unroll
    for (int k = 0; k < kPrefetch; ++k) pf_issue(ring[k]);

    double ysq0 = 0.0, ysq1 = 0.0, ysq2 = 0.0, ysq3 = 0.0;
    int64_t cur_s = -1;
    const int64_t maxs = ri.maxs;

    for (int64_t g = 0; g < ngroups; ++g) {
        const int64_t t = tb + kWarps * g + warp;
        const bool active = t < te;
        double wacc[MT0][MT1][2];
#pragma unroll
        for (int i = 0; i < MT0; ++i)
#pragma unroll
            for (int j = 0; j < MT1; ++j) wacc[i][j][0] = wacc[i][j][1] = 0.0;

        for (int pair = 0; pair < NP; ++pair) {
            double pacc[MT0][2][2];
#pragma unroll
            for (int i = 0; i < MT0; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) pacc[i][j][0] = pacc[i][j][1] = 0.0;
#pragma unroll 1
            for (int c0 = 0; c0 < NC; c0 += kPrefetch) {
#pragma unroll
                for (int cc = 0; cc < kPrefetch; ++cc) {
                    const int c = c0 + cc;
                    const double2 x0 = ring[cc][0], x1 = ring[cc][1];
                    pf_issue(ring[cc]);  // refill with the chunk kPrefetch steps ahead
                    ysq0 = fma(x0.x, x0.x, ysq0);
                    ysq1 = fma(x0.y, x0.y, ysq1);
                    ysq2 = fma(x1.x, x1.x, ysq2);
                    ysq3 = fma(x1.y, x1.y, ysq3);
                    double2 u[MT0];
#pragma unroll
                    for (int ma = 0; ma < MT0; ++ma) u[ma] = U0f[(c * MT0 + ma) * 32 + lane];
                    // dependent MMAs on one accumulator are 2*MT0 issues apart
#pragma unroll
                    for (int ma = 0; ma < MT0; ++ma) {
                        dmma(pacc[ma][0], u[ma].x, x0.x);
                        dmma(pacc[ma][1], u[ma].x, x1.x);
                    }
#pragma unroll
                    for (int ma = 0; ma < MT0; ++ma) {
                        dmma(pacc[ma][0], u[ma].y, x0.y);
                        dmma(pacc[ma][1], u[ma].y, x1.y);
                    }
                }
            }
            // step 2: W += P U1 over the pair's 16 columns
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int ntile = 2 * pair + nt;
                double2 u[MT1];
#pragma unroll
                for (int mb = 0; mb < MT1; ++mb) u[mb] = U1f[(ntile * MT1 + mb) * 32 + lane];
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int mb = 0; mb < MT1; ++mb)
#pragma unroll
                        for (int ma = 0; ma < MT0; ++ma)
                            dmma(wacc[ma][mb], pacc[ma][nt][j], j ? u[mb].y : u[mb].x);
            }
        }

        // publish this warp's W (compact a0 + r0*a1 layout)
        double* wdst = Wbuf + ((g & 1) * kWarps + warp) * R01;
        if (active) {
#pragma unroll
            for (int ma = 0; ma < MT0; ++ma)
#pragma unroll
                for (int mb = 0; mb < MT1; ++mb)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int a0 = 8 * ma + g4, a1 = 8 * mb + 2 * t4 + j;
                        if (a0 < a.r0 && a1 < a.r1) wdst[a0 + a.r0 * a1] = wacc[ma][mb][j];
                    }
        }
        __syncthreads();

        // step 3: Z_s += W (x) U2[i2, :] over the group's slabs; runs of
        // slabs of one sample accumulate in registers, one Z pass per run
        const double* wsrc = Wbuf + (g & 1) * kWarps * R01;
        const int64_t rem_slabs = te - (tb + kWarps * g);
        const int nact = static_cast<int>(rem_slabs < kWarps ? rem_slabs : kWarps);
        int w0 = 0;
        while (w0 < nact) {
            const int64_t t0 = tb + kWarps * g + w0;
            const int64_t s = t0 / a.n2;
            const int64_t i20 = t0 - s * a.n2;
            int w1 = w0 + 1;
            while (w1 < nact && (t0 + (w1 - w0)) / a.n2 == s) ++w1;
            if (s != cur_s) {
                if (cur_s >= 0) {
                    double* zp = a.zpart + ((b * maxs) + (cur_s - s_first)) * R;
                    for (int e = tid; e < R; e += kThreads) {
                        zp[e] = Zs[e];
                        Zs[e] = 0.0;
                    }
                }
                cur_s = s;
            }
            int p = tid % R01, a2 = tid / R01;
            for (int e = tid; e < R; e += kThreads) {
                double acc = Zs[e];
                const double* u2 = U2s + i20 + a.n2 * a2;
                for (int w = w0; w < w1; ++w) acc = fma(wsrc[w * R01 + p], u2[w - w0], acc);
                Zs[e] = acc;
                p += kThreads;
                while (p >= R01) {
                    p -= R01;
                    ++a2;
                }
            }
            w0 = w1;
        }
    }
    if (cur_s >= 0) {
        double* zp = a.zpart + ((b * maxs) + (cur_s - s_first)) * R;
        for (int e = tid; e < R; e += kThreads) zp[e] = Zs[e];
    }

    // ||Y||^2 partial of this CTA (fixed shuffle tree, fixed warp order)
    double ys = (ysq0 + ysq1) + (ysq2 + ysq3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ys += __shfl_xor_sync(0xffffffffu, ys, o);
    if (lane == 0) red[warp] = ys;
    __syncthreads();
    if (tid == 0) {
        double sum = 0.0;
        for (int w = 0; w < kWarps; ++w) sum += red[w];
        a.ysq_partials[b] = sum;
    }
}

// Z[e + R s] = sum over the CTAs whose slab range meets sample s, in CTA
// order. One CTA per sample; the contributing CTA range is found once.
__global__ void fused3_reduce_kernel(const Fused3Args a, RangeInfo ri, int64_t B) {
    __shared__ int64_t range[2];
    const int64_t R = static_cast<int64_t>(a.r0) * a.r1 * a.r2;
    for (int64_t s = blockIdx.x; s < a.S; s += gridDim.x) {
        if (threadIdx.x == 0) {
            const int64_t lo = s * a.n2, hi = lo + a.n2;
            int64_t bl = (lo * B) / ri.T;
            while (bl > 0 && cta_begin(ri.T, bl, B) > lo) --bl;
            while (cta_begin(ri.T, bl + 1, B) <= lo) ++bl;
            int64_t bh = bl;
            while (bh + 1 < B && cta_begin(ri.T, bh + 1, B) < hi) ++bh;
            range[0] = bl;
            range[1] = bh;
        }
        __syncthreads();
        const int64_t bl = range[0], bh = range[1];
        for (int64_t e = threadIdx.x; e < R; e += blockDim.x) {
            double acc = 0.0;
            for (int64_t bb = bl; bb <= bh; ++bb) {
                const int64_t tb = cta_begin(ri.T, bb, B);
                acc += a.zpart[((bb * ri.maxs) + (s - tb / a.n2)) * R + e];
            }
            a.Z[e + R * s] = acc;
        }
        __syncthreads();
    }
}

template <int N0, int N1, int MT0, int MT1>
int launch_impl(const Fused3Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    const int64_t T = a.n2 * a.S;
    const int64_t B = std::min<int64_t>(num_sms, T);
    const int64_t per = (T + B - 1) / B;
    RangeInfo ri{T, (per + a.n2 - 1) / a.n2 + 1};
    const int64_t R01 = static_cast<int64_t>(a.r0) * a.r1;
    const size_t smem = sizeof(double) * (static_cast<size_t>(N0 / 8) * MT0 * 64 + static_cast<size_t>(N1 / 8) * MT1 * 64 +
                                          2 * kWarps * R01 + R01 * a.r2 + a.n2 * a.r2);
    auto kfn = fused3_kernel<N0, N1, MT0, MT1>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kfn<<<static_cast<unsigned>(B), kThreads, smem, s>>>(a, ri);
    const int rb = static_cast<int>(std::min<int64_t>(a.S, 65535));
    fused3_reduce_kernel<<<rb, 256, 0, s>>>(a, ri, B);
    *launches += 2;
    return static_cast<int>(B);
}

template <int N>
int dispatch_mt(int mt, const Fused3Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    switch (mt) {
        case 1: return launch_impl<N, N, 1, 1>(a, num_sms, s, launches);
        case 2: return launch_impl<N, N, 2, 2>(a, num_sms, s, launches);
        case 3: return launch_impl<N, N, 3, 3>(a, num_sms, s, launches);
        default: return -1;
    }
}

}  // namespace

bool fused3_supported(int64_t n0, int64_t n1, int64_t n2, int r0, int r1, int r2) {
    if (n0 != n1 || (n0 != 64 && n0 != 128)) return false;
    if (r0 < 1 || r1 < 1 || r2 < 1 || r0 > 24 || r1 > 24) return false;
    if (static_cast<int64_t>(r0) * r1 * r2 > kMaxZ) return false;
    const int64_t R01 = static_cast<int64_t>(r0) * r1;
    const int mt = (std::max(r0, r1) + 7) / 8;
    const size_t smem =
        sizeof(double) * (static_cast<size_t>(n0 / 8) * mt * 64 * 2 + 2 * kWarps * R01 + R01 * r2 + n2 * r2);
    return smem <= 227 * 1024;
}

int64_t fused3_workspace_doubles(int64_t n0, int64_t n1, int64_t n2, int64_t S, int r0, int r1, int r2,
                                 int num_sms) {
    (void)n0;
    (void)n1;
    const int64_t T = n2 * S;
    const int64_t B = std::min<int64_t>(num_sms, T);
    const int64_t per = (T + B - 1) / B;
    const int64_t maxs = (per + n2 - 1) / n2 + 1;
    return B * maxs * static_cast<int64_t>(r0) * r1 * r2 + B;  // zpart + ysq partials
}

int launch_fused3(int64_t n0, int64_t n1, const Fused3Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    (void)n1;
    const int mt = (std::max(a.r0, a.r1) + 7) / 8;
    if (n0 == 128) return dispatch_mt<128>(mt, a, num_sms, s, launches);
    if (n0 == 64) return dispatch_mt<64>(mt, a, num_sms, s, launches);
    return -1;
}

}  // namespace htr
