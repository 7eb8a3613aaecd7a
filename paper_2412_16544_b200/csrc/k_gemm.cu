// Generic strided f64 contraction engine on the FP64 tensor cores (DMMA).
//
// Replaces the Eigen GEMMs behind mode_multiply / unfold (reference
// tensor.hpp:300-312, 150-172), the Gram of every unfolding that feeds a
// truncated SVD (truncated_svd.hpp:53, bht.hpp:284/325, ht_rise.hpp:144) and
// the explicit residual energy of project_mode (bht.hpp:357-365) — all
// without materialising an unfolding: the unfolding is an index map
// (k1, k2) / (n1, n2) over the canonical buffer (see GemmDesc).
//
// CTA tiles of BM x BN outputs (64x64, 64x32 or 32x64, picked per problem to
// minimise padding), 4 warps each holding (BM/2)x(BN/2) as 8x8 DMMA
// accumulators, K staged 16 at a time through a 4-stage cp.async pipeline in
// shared memory (pitch = tile + 4 doubles: conflict-free fragment reads;
// zero-fill outside the problem). Operand offsets
// along m / n are precomputed per thread; the k offset needs one 32-bit
// multiply-shift division at most. Deterministic split-K and batching.
#include <algorithm>
#include <cstdio>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int BK = 16, NT = 128;

/// n / d for n < 2^31 via multiply-high (Granlund-Montgomery round-up).
struct FastDiv {
    uint32_t d = 1, magic = 0, shift = 0;
    FastDiv() = default;
    explicit FastDiv(uint32_t dv) : d(dv) {
        shift = 0;
        while ((uint64_t{1} << shift) < dv) ++shift;
        magic = static_cast<uint32_t>(((uint64_t{1} << 32) * ((uint64_t{1} << shift) - dv)) / dv + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        const uint64_t hi = __umulhi(n, magic);
        return static_cast<uint32_t>((hi + n) >> shift);
    }
};

struct Launch {
    int a_kfast, b_kfast, energy;
    int kmode;  // 0: K1 == 1 (k -> k2), 1: K2 == 1 (k -> k1), 2: general
    FastDiv k1div, n1div;
    int64_t splits;
};

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ int64_t k_part(const Launch& L, int64_t k, int64_t s1, int64_t s2, int64_t K1) {
    if (L.kmode == 0) return k * s2;
    if (L.kmode == 1) return k * s1;
    const int64_t k2 = L.k1div.div(static_cast<uint32_t>(k));
    return (k - k2 * K1) * s1 + k2 * s2;
}

__device__ __forceinline__ int64_t n_part(const Launch& L, int64_t n, int64_t s1, int64_t s2, int64_t N1) {
    const int64_t n2 = L.n1div.div(static_cast<uint32_t>(n));
    return (n - n2 * N1) * s1 + n2 * s2;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}

constexpr int NSTAGE = 4;

template <int BM, int BN>
constexpr size_t gemm_smem_bytes() {
    return sizeof(double) * NSTAGE * BK * ((BM + 4) + (BN + 4));
}

template <int BM, int BN>
__global__ void __launch_bounds__(NT, 3) gemm_kernel(const GemmDesc d, const int64_t kchunk, double* partial,
                                                     const Launch L) {
    constexpr int WM = BM / 2, WN = BN / 2, FM = WM / 8, FN = WN / 8;
    constexpr int PA = BM + 4, PB = BN + 4;
    constexpr int EA = BM * BK / NT, EB = BN * BK / NT;  // elements per thread per tile
    extern __shared__ __align__(16) double gsm[];
    double* As = gsm;                        // [NSTAGE][BK][PA]
    double* Bs = gsm + NSTAGE * BK * PA;     // [NSTAGE][BK][PB]
    __shared__ double red[NT / 32];

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int wm = (warp & 1) * WM, wn = (warp >> 1) * WN;
    const int64_t M = d.M, N = d.N1 * d.N2, K = d.K1 * d.K2;
    const int64_t zb = blockIdx.z / L.splits, zs = blockIdx.z - zb * L.splits;
    const double* A = d.A + zb * d.sab;
    const double* B = d.B + zb * d.sbb;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
    const int64_t kbeg = zs * kchunk;
    const int64_t kend = min(K, kbeg + kchunk);
    const int ntiles = static_cast<int>((kend - kbeg + BK - 1) / BK);

    // per-thread operand coordinates: the m / n parts never change with k
    auto akk = [&](int j) { return L.a_kfast ? (t & 15) : t / BM + (NT / BM) * j; };
    auto amm = [&](int j) { return L.a_kfast ? (t >> 4) + (NT / 16) * j : t % BM; };
    auto bkk = [&](int j) { return L.b_kfast ? (t & 15) : t / BN + (NT / BN) * j; };
    auto bnn = [&](int j) { return L.b_kfast ? (t >> 4) + (NT / 16) * j : t % BN; };
    int64_t aoff[EA], boff[EB];
#pragma unroll
    for (int j = 0; j < EA; ++j) {
        const int64_t m = m0 + amm(j);
        aoff[j] = m < M ? m * d.sam : -1;
    }
#pragma unroll
    for (int j = 0; j < EB; ++j) {
        const int64_t n = n0 + bnn(j);
        boff[j] = n < N ? n_part(L, n, d.sbn1, d.sbn2, d.N1) : -1;
    }

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // async copy of K tile `kt` into stage `st` (zero-fill outside the problem)
    auto issue = [&](int kt, int st) {
        const int64_t k0 = kbeg + static_cast<int64_t>(kt) * BK;
        double* as = As + st * BK * PA;
        double* bs = Bs + st * BK * PB;
#pragma unroll
        for (int j = 0; j < EA; ++j) {
            const int64_t k = k0 + akk(j);
            const bool ok = aoff[j] >= 0 && k < kend;
            cp_async8(as + akk(j) * PA + amm(j), ok ? A + aoff[j] + k_part(L, k, d.sak1, d.sak2, d.K1) : A, ok);
        }
#pragma unroll
        for (int j = 0; j < EB; ++j) {
            const int64_t k = k0 + bkk(j);
            const bool ok = boff[j] >= 0 && k < kend;
            cp_async8(bs + bkk(j) * PB + bnn(j), ok ? B + boff[j] + k_part(L, k, d.sbk1, d.sbk2, d.K1) : B, ok);
        }
    };

#pragma unroll
    for (int st = 0; st < NSTAGE - 1; ++st) {
        if (st < ntiles) issue(st, st);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int kt = 0; kt < ntiles; ++kt) {
        asm volatile("cp.async.wait_group %0;" ::"n"(NSTAGE - 2) : "memory");
        __syncthreads();
        // the stage consumed in the previous iteration is free again
        if (kt + NSTAGE - 1 < ntiles) issue(kt + NSTAGE - 1, (kt + NSTAGE - 1) % NSTAGE);
        asm volatile("cp.async.commit_group;" ::: "memory");
        const double* as = As + (kt % NSTAGE) * BK * PA;
        const double* bs = Bs + (kt % NSTAGE) * BK * PB;
#pragma unroll
        for (int ks = 0; ks < BK; ks += 4) {
            double a[FM], b[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) a[i] = as[(ks + t4) * PA + wm + 8 * i + g4];
#pragma unroll
            for (int j = 0; j < FN; ++j) b[j] = bs[(ks + t4) * PB + wn + 8 * j + g4];
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma884(acc[i][j], a[i], b[j]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");

    if (L.energy) {
        const double* D = d.D + zb * d.scb;
        double e = 0.0;
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t m = m0 + wm + 8 * i + g4, n = n0 + wn + 8 * j + 2 * t4 + h;
                    if (m < M && n < N) {
                        const double r = D[m * d.scm + n_part(L, n, d.scn1, d.scn2, d.N1)] - acc[i][j][h];
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
            d.energy_partials[blockIdx.x +
                              static_cast<int64_t>(gridDim.x) * (blockIdx.y + static_cast<int64_t>(gridDim.y) * blockIdx.z)] =
                s;
        }
        return;
    }

    double* C = d.C + zb * d.scb;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t m = m0 + wm + 8 * i + g4, n = n0 + wn + 8 * j + 2 * t4 + h;
                if (m < M && n < N) {
                    if (partial) {
                        partial[(static_cast<int64_t>(blockIdx.z) * M + m) * N + n] = acc[i][j][h];
                    } else {
                        double* c = C + m * d.scm + n_part(L, n, d.scn1, d.scn2, d.N1);
                        *c = d.beta == 0.0 ? d.alpha * acc[i][j][h] : fma(d.alpha, acc[i][j][h], d.beta * *c);
                    }
                }
            }
}

__global__ void splitk_reduce_kernel(const GemmDesc d, const double* partial, int64_t splits, const Launch L) {
    const int64_t M = d.M, N = d.N1 * d.N2, MN = M * N, total = MN * d.batch;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t zb = idx / MN, r = idx - zb * MN;
        double s = 0.0;
        for (int64_t z = 0; z < splits; ++z) s += partial[(zb * splits + z) * MN + r];
        const int64_t m = r / N, n = r - m * N;
        double* c = d.C + zb * d.scb + m * d.scm + n_part(L, n, d.scn1, d.scn2, d.N1);
        *c = d.beta == 0.0 ? d.alpha * s : fma(d.alpha, s, d.beta * *c);
    }
}

struct Plan {
    int bm, bn;
    int64_t tiles_n, tiles_m, splits, kchunk;
};

Plan plan_for(const GemmDesc& d, int num_sms) {
    Plan p;
    const int64_t N = d.N1 * d.N2, K = d.K1 * d.K2;
    // tile shape with the least padded area (ties: the square tile)
    const int shapes[3][2] = {{64, 64}, {64, 32}, {32, 64}};
    int64_t best = -1;
    for (const auto& sh : shapes) {
        const int64_t area = ((d.M + sh[0] - 1) / sh[0]) * sh[0] * ((N + sh[1] - 1) / sh[1]) * sh[1];
        if (best < 0 || area < best) {
            best = area;
            p.bm = sh[0];
            p.bn = sh[1];
        }
    }
    p.tiles_n = (N + p.bn - 1) / p.bn;
    p.tiles_m = (d.M + p.bm - 1) / p.bm;
    const int64_t tiles = p.tiles_n * p.tiles_m * d.batch;
    const int64_t ktiles = (K + BK - 1) / BK;
    p.splits = 1;
    if (d.energy_partials == nullptr && tiles < 2 * num_sms && ktiles >= 16) {
        p.splits = std::min<int64_t>((4 * num_sms + tiles - 1) / tiles, ktiles / 8);
        p.splits = std::max<int64_t>(1, std::min<int64_t>(p.splits, 4096));
    }
    const int64_t per = (ktiles + p.splits - 1) / p.splits;
    p.kchunk = std::max<int64_t>(per, 1) * BK;
    p.splits = std::max<int64_t>(1, (K + p.kchunk - 1) / p.kchunk);
    return p;
}

}  // namespace

int64_t gemm_workspace_doubles(const GemmDesc& d, int num_sms) {
    const Plan p = plan_for(d, num_sms);
    return p.splits > 1 ? p.splits * d.batch * d.M * d.N1 * d.N2 : 0;
}

int64_t gemm_energy_partials(const GemmDesc& d, int num_sms) {
    const Plan p = plan_for(d, num_sms);
    return p.tiles_n * p.tiles_m * d.batch;
}

int launch_gemm(const GemmDesc& d, double* workspace, int num_sms, cudaStream_t s, int64_t* launches) {
    const int64_t N = d.N1 * d.N2, K = d.K1 * d.K2;
    if (d.M <= 0 || N <= 0 || d.batch <= 0) return 0;
    if (K <= 0) return 0;  // extents are >= 1 by construction
    const Plan p = plan_for(d, num_sms);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(gemm_kernel<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(gemm_smem_bytes<64, 64>()));
        cudaFuncSetAttribute(gemm_kernel<64, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(gemm_smem_bytes<64, 32>()));
        cudaFuncSetAttribute(gemm_kernel<32, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(gemm_smem_bytes<32, 64>()));
        configured = true;
    }
    const bool a_kc = d.K1 > 1 ? d.sak1 == 1 : d.sak2 == 1;
    const bool b_kc = d.K1 > 1 ? d.sbk1 == 1 : d.sbk2 == 1;
    const bool b_nc = d.N1 > 1 ? d.sbn1 == 1 : d.sbn2 == 1;
    Launch L;
    L.a_kfast = a_kc ? 1 : (d.sam == 1 ? 0 : 1);
    L.b_kfast = b_kc ? 1 : (b_nc ? 0 : 1);
    L.energy = d.energy_partials != nullptr;
    L.kmode = d.K1 == 1 ? 0 : (d.K2 == 1 ? 1 : 2);
    L.k1div = FastDiv(static_cast<uint32_t>(d.K1));
    L.n1div = FastDiv(static_cast<uint32_t>(d.N1));
    L.splits = p.splits;
    const dim3 grid(static_cast<unsigned>(p.tiles_n), static_cast<unsigned>(p.tiles_m),
                    static_cast<unsigned>(p.splits * d.batch));
    double* partial = p.splits > 1 ? workspace : nullptr;
    if (p.bm == 64 && p.bn == 64) gemm_kernel<64, 64><<<grid, NT, gemm_smem_bytes<64, 64>(), s>>>(d, p.kchunk, partial, L);
    else if (p.bm == 64) gemm_kernel<64, 32><<<grid, NT, gemm_smem_bytes<64, 32>(), s>>>(d, p.kchunk, partial, L);
    else gemm_kernel<32, 64><<<grid, NT, gemm_smem_bytes<32, 64>(), s>>>(d, p.kchunk, partial, L);
    ++*launches;
    if (p.splits > 1) {
        const int64_t total = d.M * N * d.batch;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * num_sms));
        splitk_reduce_kernel<<<blocks, 256, 0, s>>>(d, partial, p.splits, L);
        ++*launches;
    }
    return L.energy ? static_cast<int>(p.tiles_n * p.tiles_m * d.batch) : 0;
}

}  // namespace htr
