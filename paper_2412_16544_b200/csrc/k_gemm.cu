// Generic strided f64 contraction engine (see GemmDesc in kernels.cuh).
//
// Replaces the Eigen GEMMs behind mode_multiply / unfold (reference
// tensor.hpp:300-312, 150-172), the Gram of every unfolding that feeds a
// truncated SVD (truncated_svd.hpp:53, bht.hpp:284/325, ht_rise.hpp:144) and
// the explicit residual energy of project_mode (bht.hpp:357-365) — all
// without materialising an unfolding: the unfolding is an index map
// (k1, k2) / (n1, n2) over the canonical buffer.
//
// Tile 64x64x16, 256 threads, 4x4 f64 accumulators per thread, register
// prefetch of the next K tile, deterministic split-K through a workspace.
#include <algorithm>
#include <cstdio>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 128;

struct Flags {
    int a_kfast;
    int b_kfast;
    int energy;
};

__device__ __forceinline__ int64_t a_off(const GemmDesc& d, int64_t m, int64_t k) {
    const int64_t k2 = k / d.K1;
    const int64_t k1 = k - k2 * d.K1;
    return m * d.sam + k1 * d.sak1 + k2 * d.sak2;
}
__device__ __forceinline__ int64_t b_off(const GemmDesc& d, int64_t k, int64_t n) {
    const int64_t k2 = k / d.K1;
    const int64_t k1 = k - k2 * d.K1;
    const int64_t n2 = n / d.N1;
    const int64_t n1 = n - n2 * d.N1;
    return k1 * d.sbk1 + k2 * d.sbk2 + n1 * d.sbn1 + n2 * d.sbn2;
}
__device__ __forceinline__ int64_t c_off(const GemmDesc& d, int64_t m, int64_t n) {
    const int64_t n2 = n / d.N1;
    const int64_t n1 = n - n2 * d.N1;
    return m * d.scm + n1 * d.scn1 + n2 * d.scn2;
}

// FP64 tensor-core tile: 64x64 outputs per CTA, 4 warps each owning a
// 32x32 quadrant as 4x4 DMMA 8x8 accumulators, K staged 16 at a time through
// shared memory (row pitch 68 doubles: conflict-free fragment reads).
constexpr int PITCH = BM + 4;

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(NT) gemm_kernel(const GemmDesc d, const int64_t kchunk, double* partial,
                                                  const Flags fl) {
    __shared__ __align__(16) double As[2][BK][PITCH];
    __shared__ __align__(16) double Bs[2][BK][PITCH];
    __shared__ double red[NT / 32];

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    const int64_t M = d.M, N = d.N1 * d.N2, K = d.K1 * d.K2;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
    const int64_t kbeg = static_cast<int64_t>(blockIdx.z) * kchunk;
    const int64_t kend = min(K, kbeg + kchunk);

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    constexpr int PER = BM * BK / NT;  // 8 elements of each operand per thread
    double ra[PER], rb[PER];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            int kk, mm;
            if (fl.a_kfast) { kk = t & 15; mm = (t >> 4) + 8 * j; }
            else { mm = t & 63; kk = (t >> 6) + 2 * j; }
            const int64_t m = m0 + mm, k = k0 + kk;
            ra[j] = (m < M && k < kend) ? __ldg(d.A + a_off(d, m, k)) : 0.0;
            int nn;
            if (fl.b_kfast) { kk = t & 15; nn = (t >> 4) + 8 * j; }
            else { nn = t & 63; kk = (t >> 6) + 2 * j; }
            const int64_t n = n0 + nn, k2 = k0 + kk;
            rb[j] = (n < N && k2 < kend) ? __ldg(d.B + b_off(d, k2, n)) : 0.0;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            if (fl.a_kfast) As[buf][t & 15][(t >> 4) + 8 * j] = ra[j];
            else As[buf][(t >> 6) + 2 * j][t & 63] = ra[j];
            if (fl.b_kfast) Bs[buf][t & 15][(t >> 4) + 8 * j] = rb[j];
            else Bs[buf][(t >> 6) + 2 * j][t & 63] = rb[j];
        }
    };

    int buf = 0;
    if (kbeg < kend) {
        load(kbeg);
        stash(0);
    }
    __syncthreads();
    for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
        const bool more = k0 + BK < kend;
        if (more) load(k0 + BK);  // global loads in flight during the MMAs
#pragma unroll
        for (int ks = 0; ks < BK; ks += 4) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][ks + t4][wm + 8 * i + g4];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[buf][ks + t4][wn + 8 * j + g4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j], a[i], b[j]);
        }
        if (more) stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }

    if (fl.energy) {
        double e = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t m = m0 + wm + 8 * i + g4, n = n0 + wn + 8 * j + 2 * t4 + h;
                    if (m < M && n < N) {
                        const double r = d.D[c_off(d, m, n)] - acc[i][j][h];
                        e = fma(r, r, e);
                    }
                }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (lane == 0) red[warp] = e;
        __syncthreads();
        if (t == 0) {
            double s = 0.0;
            for (int w = 0; w < NT / 32; ++w) s += red[w];
            d.energy_partials[blockIdx.x + static_cast<int64_t>(gridDim.x) * blockIdx.y] = s;
        }
        return;
    }

#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t m = m0 + wm + 8 * i + g4, n = n0 + wn + 8 * j + 2 * t4 + h;
                if (m < M && n < N) {
                    if (partial) {
                        partial[(static_cast<int64_t>(blockIdx.z) * M + m) * N + n] = acc[i][j][h];
                    } else {
                        double* c = d.C + c_off(d, m, n);
                        *c = d.beta == 0.0 ? d.alpha * acc[i][j][h] : fma(d.alpha, acc[i][j][h], d.beta * *c);
                    }
                }
            }
}

__global__ void splitk_reduce_kernel(const GemmDesc d, const double* partial, int splits) {
    const int64_t M = d.M, N = d.N1 * d.N2, MN = M * N;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < MN;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += partial[z * MN + idx];
        const int64_t m = idx / N, n = idx - m * N;
        double* c = d.C + c_off(d, m, n);
        *c = d.beta == 0.0 ? d.alpha * s : fma(d.alpha, s, d.beta * *c);
    }
}

struct Plan {
    int64_t tiles_n, tiles_m, splits, kchunk;
};

Plan plan_for(const GemmDesc& d, int num_sms) {
    Plan p;
    const int64_t N = d.N1 * d.N2, K = d.K1 * d.K2;
    p.tiles_n = (N + BN - 1) / BN;
    p.tiles_m = (d.M + BM - 1) / BM;
    const int64_t tiles = p.tiles_n * p.tiles_m;
    const int64_t ktiles = (K + BK - 1) / BK;
    p.splits = 1;
    if (d.energy_partials == nullptr && tiles < 2 * num_sms && ktiles >= 16) {
        p.splits = std::min<int64_t>((2 * num_sms + tiles - 1) / tiles, ktiles / 8);
        p.splits = std::max<int64_t>(1, std::min<int64_t>(p.splits, 4096));
    }
    const int64_t per = (ktiles + p.splits - 1) / p.splits;
    p.kchunk = std::max<int64_t>(per, 1) * BK;
    p.splits = (K + p.kchunk - 1) / p.kchunk;
    if (p.splits < 1) p.splits = 1;
    return p;
}

}  // namespace

int64_t gemm_workspace_doubles(const GemmDesc& d, int num_sms) {
    const Plan p = plan_for(d, num_sms);
    return p.splits > 1 ? p.splits * d.M * d.N1 * d.N2 : 0;
}

int launch_gemm(const GemmDesc& d, double* workspace, int num_sms, cudaStream_t s, int64_t* launches) {
    const int64_t N = d.N1 * d.N2, K = d.K1 * d.K2;
    if (d.M <= 0 || N <= 0) return 0;
    if (K <= 0) return 0;  // extents are >= 1 by construction
    const Plan p = plan_for(d, num_sms);
    const bool a_kc = d.K1 > 1 ? d.sak1 == 1 : d.sak2 == 1;
    const bool b_kc = d.K1 > 1 ? d.sbk1 == 1 : d.sbk2 == 1;
    const bool b_nc = d.N1 > 1 ? d.sbn1 == 1 : d.sbn2 == 1;
    Flags fl;
    fl.a_kfast = a_kc ? 1 : (d.sam == 1 ? 0 : 1);
    fl.b_kfast = b_kc ? 1 : (b_nc ? 0 : 1);
    fl.energy = d.energy_partials != nullptr;
    const dim3 grid(static_cast<unsigned>(p.tiles_n), static_cast<unsigned>(p.tiles_m),
                    static_cast<unsigned>(p.splits));
    double* partial = p.splits > 1 ? workspace : nullptr;
    gemm_kernel<<<grid, NT, 0, s>>>(d, p.kchunk, partial, fl);
    ++*launches;
    if (p.splits > 1) {
        const int64_t MN = d.M * N;
        const int blocks = static_cast<int>(std::min<int64_t>((MN + 255) / 256, 4 * num_sms));
        splitk_reduce_kernel<<<blocks, 256, 0, s>>>(d, partial, static_cast<int>(p.splits));
        ++*launches;
    }
    return fl.energy ? static_cast<int>(p.tiles_n * p.tiles_m) : 0;
}

}  // namespace htr
