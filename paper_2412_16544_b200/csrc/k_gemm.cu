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

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

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

__global__ void __launch_bounds__(NT) gemm_kernel(const GemmDesc d, const int64_t kchunk, double* partial,
                                                  const Flags fl) {
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BN + 1];
    __shared__ double red[NT / 32];

    const int t = threadIdx.x;
    const int tx = t & 15, ty = t >> 4;
    const int64_t M = d.M, N = d.N1 * d.N2, K = d.K1 * d.K2;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
    const int64_t kbeg = static_cast<int64_t>(blockIdx.z) * kchunk;
    const int64_t kend = min(K, kbeg + kchunk);

    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    double ra[4], rb[4];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int kk, mm;
            if (fl.a_kfast) { kk = t & 15; mm = (t >> 4) + 16 * j; }
            else { mm = t & 63; kk = (t >> 6) + 4 * j; }
            const int64_t m = m0 + mm, k = k0 + kk;
            ra[j] = (m < M && k < kend) ? __ldg(d.A + a_off(d, m, k)) : 0.0;
            int nn;
            if (fl.b_kfast) { kk = t & 15; nn = (t >> 4) + 16 * j; }
            else { nn = t & 63; kk = (t >> 6) + 4 * j; }
            const int64_t n = n0 + nn, k2 = k0 + kk;
            rb[j] = (n < N && k2 < kend) ? __ldg(d.B + b_off(d, k2, n)) : 0.0;
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (fl.a_kfast) As[t & 15][(t >> 4) + 16 * j] = ra[j];
            else As[(t >> 6) + 4 * j][t & 63] = ra[j];
            if (fl.b_kfast) Bs[t & 15][(t >> 4) + 16 * j] = rb[j];
            else Bs[(t >> 6) + 4 * j][t & 63] = rb[j];
        }
    };

    if (kbeg < kend) load(kbeg);
    for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
        stash();
        __syncthreads();
        if (k0 + BK < kend) load(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }

    if (fl.energy) {
        double e = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
                if (m < M && n < N) {
                    const double r = d.D[c_off(d, m, n)] - acc[i][j];
                    e = fma(r, r, e);
                }
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if ((t & 31) == 0) red[t >> 5] = e;
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
        for (int j = 0; j < 4; ++j) {
            const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
            if (m < M && n < N) {
                if (partial) {
                    partial[(static_cast<int64_t>(blockIdx.z) * M + m) * N + n] = acc[i][j];
                } else {
                    double* c = d.C + c_off(d, m, n);
                    *c = d.beta == 0.0 ? d.alpha * acc[i][j] : fma(d.alpha, acc[i][j], d.beta * *c);
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
