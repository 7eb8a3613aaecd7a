// Skip-path tail for 3-way trees (1,(2,3)): one CTA per sample s computes
//
//   Z_s[a0, a1, a2]  = sum_i2 W[(s,i2), a0 + r0 a1] U2[i2, a2]      (slab-axis contraction)
//   latent_s[a0, b]  = sum_{a1,a2} Z_s[a0, a1, a2] B[a1 + r1 a2, b]  (transfer projection,
//                                                                     bht.hpp:385-399)
//   ||latent_s||^2
//
// on the FP64 tensor cores, with Z_s kept in shared memory between the two
// contractions. W is the per-slab output of fused3_kernel (L2-resident),
// B the transfer node's basis matrix (r1 r2 x rt), streamed from L2.
// Replaces two generic GEMM launches and the latent norm pass; deterministic.
#include <algorithm>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kGroup = 4;    // tiles per warp per pass
constexpr int kU2Pitch = 28; // doubles: conflict-free B-fragment reads (<= 24 columns)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kThreads, 2) tail3_kernel(const Tail3Args a) {
    extern __shared__ __align__(16) double sm[];
    const int r0 = a.r0, r1 = a.r1, r2 = a.r2, rt = a.rt;
    const int R01 = r0 * r1, R12 = r1 * r2;
    const int n2 = static_cast<int>(a.n2);
    double* U2s = sm;                               // [n2][kU2Pitch]
    double* Zs = U2s + n2 * kU2Pitch;               // [a0 + r0 (a1 + r1 a2)]
    __shared__ double red[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int64_t s = blockIdx.x;

    for (int e = tid; e < n2 * kU2Pitch; e += kThreads) {
        const int i2 = e / kU2Pitch, c = e - i2 * kU2Pitch;
        U2s[e] = c < r2 ? a.U2[i2 + static_cast<int64_t>(n2) * c] : 0.0;
    }
    __syncthreads();

    // ---- phase A: Z_s(p, a2), M = R01 (p), N = r2, K = n2 ----
    const double* W = a.wslab + s * n2 * static_cast<int64_t>(R01);
    const int mtA = (R01 + 7) / 8, ntA = (r2 + 7) / 8;
    for (int base = warp; base < mtA; base += kWarps * kGroup) {
        double acc[kGroup][3][2];
#pragma unroll
        for (int i = 0; i < kGroup; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        auto loadA = [&](int k, double (&av)[kGroup]) {
#pragma unroll
            for (int i = 0; i < kGroup; ++i) {
                const int mt = base + kWarps * i;
                const int p = 8 * mt + g4;
                av[i] = (mt < mtA && p < R01 && k < n2) ? __ldg(W + static_cast<int64_t>(k) * R01 + p) : 0.0;
            }
        };
        double anext[kGroup];
        loadA(t4, anext);
#pragma unroll 2
        for (int k0 = 0; k0 < n2; k0 += 4) {
            const int k = k0 + t4;
            double av[kGroup];
#pragma unroll
            for (int i = 0; i < kGroup; ++i) av[i] = anext[i];
            loadA(k + 4, anext);  // next step's operands in flight during the MMAs
            double b[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) b[j] = (k < n2) ? U2s[k * kU2Pitch + 8 * j + g4] : 0.0;
#pragma unroll
            for (int i = 0; i < kGroup; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    if (j < ntA) dmma(acc[i][j], av[i], b[j]);
        }
#pragma unroll
        for (int i = 0; i < kGroup; ++i) {
            const int mt = base + kWarps * i;
            if (mt >= mtA) continue;
            const int p = 8 * mt + g4;
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int a2 = 8 * j + 2 * t4 + h;
                    if (p < R01 && a2 < r2) Zs[p + R01 * a2] = acc[i][j][h];
                }
        }
    }
    __syncthreads();

    // ---- phase B: latent_s(a0, b) = Z_s(a0, j) B(j, b), M = r0, N = rt, K = R12 ----
    const int mtB = (r0 + 7) / 8, ntB = (rt + 7) / 8;
    double lsq = 0.0;
    double* out = a.latent + s * static_cast<int64_t>(r0) * rt;
    for (int base = warp; base < ntB; base += kWarps * kGroup) {
        double acc[3][kGroup][2];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < kGroup; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        auto loadB = [&](int k, double (&bv)[kGroup]) {
#pragma unroll
            for (int j = 0; j < kGroup; ++j) {
                const int nt = base + kWarps * j;
                const int bcol = 8 * nt + g4;
                bv[j] = (nt < ntB && bcol < rt && k < R12) ? __ldg(a.B + k + static_cast<int64_t>(R12) * bcol) : 0.0;
            }
        };
        double bnext[kGroup];
        loadB(t4, bnext);
#pragma unroll 2
        for (int k0 = 0; k0 < R12; k0 += 4) {
            const int k = k0 + t4;
            double bv[kGroup];
#pragma unroll
            for (int j = 0; j < kGroup; ++j) bv[j] = bnext[j];
            loadB(k + 4, bnext);  // next step's operands in flight during the MMAs
            double av[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int a0 = 8 * i + g4;
                av[i] = (i < mtB && a0 < r0 && k < R12) ? Zs[a0 + r0 * k] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < kGroup; ++j)
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    if (i < mtB) dmma(acc[i][j], av[i], bv[j]);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < kGroup; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int nt = base + kWarps * j;
                    const int a0 = 8 * i + g4, bcol = 8 * nt + 2 * t4 + h;
                    if (i < mtB && nt < ntB && a0 < r0 && bcol < rt) {
                        const double v = acc[i][j][h];
                        out[a0 + static_cast<int64_t>(r0) * bcol] = v;
                        lsq = fma(v, v, lsq);
                    }
                }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsq += __shfl_xor_sync(0xffffffffu, lsq, o);
    if (lane == 0) red[warp] = lsq;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        a.latsq[s] = t;
    }
}

}  // namespace

bool tail3_supported(int r0, int r1, int r2, int rt, int64_t n2) {
    if (r0 < 1 || r1 < 1 || r2 < 1 || rt < 1 || r0 > 24 || r2 > 24) return false;
    const size_t smem = sizeof(double) * (static_cast<size_t>(n2) * kU2Pitch + static_cast<size_t>(r0) * r1 * r2);
    return smem <= 200 * 1024;
}

void launch_tail3(const Tail3Args& a, cudaStream_t s, int64_t* launches) {
    const size_t smem =
        sizeof(double) * (static_cast<size_t>(a.n2) * kU2Pitch + static_cast<size_t>(a.r0) * a.r1 * a.r2);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(tail3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        configured = smem;
    }
    tail3_kernel<<<static_cast<unsigned>(a.S), kThreads, smem, s>>>(a);
    ++*launches;
}

}  // namespace htr
