// Projection of two adjacent modes in one read of the tensor, on the FP64
// tensor cores: for Y viewed as [n0, n1, n2, S] (canonical, n0 fastest)
//
//     C[i0, a1, a2, s] = sum_{i1, i2} Y[i0, i1, i2, s] U1[i1, a1] U2[i2, a2]
//
// i.e. mode_multiply by U1^T then by U2^T (tensor.hpp:300-312) -- BHT-l2r's
// deepest-layer projections (bht.hpp:290-293: the leaves of (1,(2,3)) trees,
// modes 1 and 2) and the re-projection after an expansion (ht_rise.hpp:160-
// 162). The generic engine runs them as two strided GEMMs with the [n0, r1,
// n2, S] intermediate in HBM; here the intermediate never leaves the SM.
//
// One CTA per (8-row block of i0, sample s), 8 warps. Warp w takes the slabs
// i2 = w, w + 8, ... of its sample: a TMA copy of X = Y[i0b : i0b + 8, :, i2, s]
// (8 x n1, two stages per warp), then Q = X U1 (8 x r1) with m8n8k4 DMMAs
// (k = i1). The 8 warps' Q of one round go to shared memory (double
// buffered, one CTA barrier per round) and every warp accumulates its own
// a1 rows of Z[(i0, a1), a2] += sum_{i2 of the round} Q_i2[(i0, a1)] U2[i2, a2]
// with DMMAs over k = i2 (4 slabs per k-step). Deterministic: fixed
// summation order, no atomics.
#include <algorithm>
#include <cudaTypedefs.h>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kP2Warps = 8;
constexpr int kP2Stages = 2;
constexpr int kP2Pad = 24;  // ranks padded to three 8-column tiles in shared memory

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(saddr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar)), "l"(policy)
        : "memory");
}

template <int NT1, int NT2>
__global__ void __launch_bounds__(kP2Warps * 32, 1) proj2_kernel(const Proj2Args a, const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full[kP2Warps][kP2Stages];
    const int n1 = a.n1, n2 = a.n2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int nb0 = a.n0 / 8;
    const int b0 = blockIdx.x % nb0;
    const int64_t s = blockIdx.x / nb0;
    const int stage_doubles = 8 * n1;
    double* stages = smem;                                                  // [warp][stage][n1][8]
    double* U1s = stages + kP2Warps * kP2Stages * stage_doubles;            // [n1][24]
    const int n2p = (n2 + 7) / 8 * 8;
    double* U2s = U1s + n1 * kP2Pad;                                        // [n2 rounded to 8][24]
    double* Qs = U2s + n2p * kP2Pad;                                        // [2][warp][8 * 8 * NT1]
    constexpr int QW = 64 * NT1;
    double* my_stages = stages + warp * kP2Stages * stage_doubles;
    uint64_t* my_full = full[warp];
    const int rounds = (n2 + kP2Warps - 1) / kP2Warps;
    const uint64_t policy = evict_first_policy();
    auto issue = [&](int r) {  // lane 0: slab i2 = warp + 8 r into stage r % 2
        const int i2 = warp + kP2Warps * r;
        if (i2 >= n2) return;
        const int st = r % kP2Stages;
        mbar_expect_tx(&my_full[st], static_cast<uint32_t>(stage_doubles * 8));
        tma_load_3d(my_stages + st * stage_doubles, &map, 8 * b0, 0, static_cast<int>(i2 + static_cast<int64_t>(n2) * s),
                    &my_full[st], policy);
    };
    if (lane == 0) {
        for (int k = 0; k < kP2Stages; ++k) mbar_init(&my_full[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < kP2Stages && k < rounds; ++k) issue(k);
    }
    for (int e = tid; e < n1 * kP2Pad; e += kP2Warps * 32) {
        const int i1 = e / kP2Pad, a1 = e % kP2Pad;
        U1s[e] = a1 < a.r1 ? a.U1[i1 + static_cast<int64_t>(n1) * a1] : 0.0;
    }
    for (int e = tid; e < n2p * kP2Pad; e += kP2Warps * 32) {
        const int i2 = e / kP2Pad, a2 = e % kP2Pad;
        U2s[e] = (i2 < n2 && a2 < a.r2) ? a.U2[i2 + static_cast<int64_t>(n2) * a2] : 0.0;
    }
    __syncthreads();

    double z[NT1][NT2][2];  // rows (i0 = g, a1 = w + 8 m), columns a2 = 8 nt + 2 t + h
#pragma unroll
    for (int m = 0; m < NT1; ++m)
#pragma unroll
        for (int nt = 0; nt < NT2; ++nt) z[m][nt][0] = z[m][nt][1] = 0.0;

    for (int r = 0; r < rounds; ++r) {
        const int i2 = warp + kP2Warps * r;
        double q[NT1][2];
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt) q[nt][0] = q[nt][1] = 0.0;
        if (i2 < n2) {
            const int st = r % kP2Stages;
            mbar_wait(&my_full[st], static_cast<uint32_t>((r / kP2Stages) & 1));
            const double* X = my_stages + st * stage_doubles;  // [i1][8]
            for (int ks = 0; ks < n1 / 4; ++ks) {
                const double av = X[(4 * ks + t) * 8 + g];
#pragma unroll
                for (int nt = 0; nt < NT1; ++nt) dmma(q[nt], av, U1s[(4 * ks + t) * kP2Pad + 8 * nt + g]);
            }
            __syncwarp();
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (r + kP2Stages < rounds) issue(r + kP2Stages);
            }
        }
        // Q of this warp's slab: row rho = i0 + 8 a1, a1 = 8 nt + 2 t + h
        double* qw = Qs + ((r & 1) * kP2Warps + warp) * QW;
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) qw[g + 8 * (8 * nt + 2 * t + h)] = q[nt][h];
        __syncthreads();
        // Z rows of a1 = warp + 8 m over the round's 8 slabs (2 k-steps)
        const double* qr = Qs + (r & 1) * kP2Warps * QW;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const int slab = 4 * ks + t;
            const double* u2 = U2s + (kP2Warps * r + slab) * kP2Pad;
            double bv[NT2];
#pragma unroll
            for (int nt = 0; nt < NT2; ++nt) bv[nt] = u2[8 * nt + g];
#pragma unroll
            for (int m = 0; m < NT1; ++m) {
                const double av = qr[slab * QW + g + 8 * (warp + 8 * m)];
#pragma unroll
                for (int nt = 0; nt < NT2; ++nt) dmma(z[m][nt], av, bv[nt]);
            }
        }
    }
    // C[i0b + g, a1, a2, s]
#pragma unroll
    for (int m = 0; m < NT1; ++m) {
        const int a1 = warp + 8 * m;
        if (a1 >= a.r1) continue;
#pragma unroll
        for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a2 = 8 * nt + 2 * t + h;
                if (a2 < a.r2)
                    a.C[(8 * b0 + g) + static_cast<int64_t>(a.n0) * (a1 + static_cast<int64_t>(a.r1) * (a2 + static_cast<int64_t>(a.r2) * s))] =
                        z[m][nt][h];
            }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

size_t proj2_smem(int64_t n1, int64_t n2, int nt1) {
    const int64_t n2p = (n2 + 7) / 8 * 8;
    return sizeof(double) * static_cast<size_t>(kP2Warps * kP2Stages * 8 * n1 + n1 * kP2Pad + n2p * kP2Pad +
                                                2 * kP2Warps * 64 * nt1);
}

template <int NT1, int NT2>
void launch_t(const Proj2Args& a, const CUtensorMap& map, int64_t grid, size_t smem, cudaStream_t s) {
    ensure_smem_limit(reinterpret_cast<const void*>(proj2_kernel<NT1, NT2>), smem);
    proj2_kernel<NT1, NT2><<<static_cast<unsigned>(grid), kP2Warps * 32, smem, s>>>(a, map);
}

template <int NT1>
void launch_nt1(const Proj2Args& a, const CUtensorMap& map, int64_t grid, size_t smem, cudaStream_t s) {
    switch ((a.r2 + 7) / 8) {
        case 1: launch_t<NT1, 1>(a, map, grid, smem, s); break;
        case 2: launch_t<NT1, 2>(a, map, grid, smem, s); break;
        default: launch_t<NT1, 3>(a, map, grid, smem, s); break;
    }
}

}  // namespace

bool proj2_supported(const Proj2Args& a) {
    if (a.n0 < 8 || a.n0 % 8 || a.n1 < 4 || a.n1 % 4 || a.n1 > 256 || a.n2 < 1 || a.S < 1) return false;
    if (a.r1 < 1 || a.r1 > kP2Pad || a.r2 < 1 || a.r2 > kP2Pad) return false;
    if ((reinterpret_cast<uintptr_t>(a.Y) & 15u) || a.n2 * a.S >= (int64_t{1} << 31)) return false;
    if ((a.n0 / 8) * a.S >= (int64_t{1} << 31)) return false;
    return proj2_smem(a.n1, a.n2, (a.r1 + 7) / 8) <= 220 * 1024;
}

int launch_proj2(const Proj2Args& a, cudaStream_t s, int64_t* launches) {
    if (!proj2_supported(a)) return -1;
    auto enc = encoder();
    if (!enc) return -1;
    CUtensorMap map;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.n0), static_cast<cuuint64_t>(a.n1),
                          static_cast<cuuint64_t>(a.n2 * a.S)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(a.n0 * 8), static_cast<cuuint64_t>(a.n0 * a.n1 * 8)};
    cuuint32_t box[3] = {8, static_cast<cuuint32_t>(a.n1), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(a.Y), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
    const int nt1 = static_cast<int>((a.r1 + 7) / 8);
    const size_t smem = proj2_smem(a.n1, a.n2, nt1);
    const int64_t grid = (a.n0 / 8) * a.S;
    switch (nt1) {
        case 1: launch_nt1<1>(a, map, grid, smem, s); break;
        case 2: launch_nt1<2>(a, map, grid, smem, s); break;
        default: launch_nt1<3>(a, map, grid, smem, s); break;
    }
    ++*launches;
    return static_cast<int>(grid);
}

}  // namespace htr
