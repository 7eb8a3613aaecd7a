// Streaming Gram of a mode unfolding, G = Y_(k) Y_(k)^T (the input of every
// truncation: truncated_svd of unfold(c, k), truncated_svd.hpp:53 via
// bht.hpp:284 / ht_rise.hpp:158), for modes k >= 1 of a large tensor.
//
// View the tensor as Y[K, M, B] (K = prod of the extents before mode k,
// contiguous; M = n_k; B = the rest): G[m, m'] = sum_b sum_k Y[k,m,b] Y[k,m',b].
// Each CTA owns a contiguous range of (b, 16-row k chunk) units. One producer
// warp streams the chunks by TMA (cp.async.bulk.tensor.3d, box 16 x M, 128-byte
// swizzle) into an 8-deep shared-memory ring; the consumer warps each own one
// 32 x 32 block of the lower triangle of G and accumulate it on DMMA 8x8x4
// (A and B fragments are both rows of the same chunk; the swizzle makes the
// fragment reads conflict-free). Diagonal blocks skip their upper tiles, so
// the MMA work is that of the lower triangle (136 of 256 tiles at M = 128).
// Every CTA writes its partial G; a fixed-order reduction sums the partials
// and mirrors the triangle. Deterministic for a given grid.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kGStages = 4;
constexpr int kGChunk = 16;  // k rows per TMA box (128 B: the swizzle span)
constexpr int kGBoxes = 2;   // boxes per stage: 32 k rows between two barrier hand-overs
constexpr int kGUnit = kGChunk * kGBoxes;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                      uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar)), "l"(policy)
        : "memory");
}

// element (row m, k) of a swizzled chunk [M][16 doubles]
__device__ __forceinline__ int swz(int m, int k) { return m * kGChunk + ((((k >> 1) ^ (m & 7))) << 1) + (k & 1); }

template <int MB>
__host__ __device__ constexpr int consumer_warps() {
    return MB * (MB + 1) / 2;
}

/// Lower-triangle block (mb >= nb) of consumer warp w. The FP64 tensor pipe is
/// fed per scheduler (warp % 4), a diagonal block issues 10 of an off-diagonal
/// block's 16 DMMAs per k-step, and the row-major order would give the four
/// schedulers 42/36/26/32 DMMAs per k-step at MB = 4; this order gives
/// 36/36/32/32 (warp 10, the TMA producer, shares scheduler 2).
template <int MB>
__device__ __forceinline__ void block_of_warp(int w, int& mb, int& nb) {
    if constexpr (MB == 4) {
        // warps 0,4,8 | 1,5,9 | 2,6 | 3,7
        // mb = {1, 2, 2, 3, 0, 2, 3, 3, 1, 3}, nb = {0, 0, 1, 1, 0, 2, 0, 2, 1, 3}, two bits per warp
        mb = (0xdf8e9u >> (2 * w)) & 3;
        nb = (0xd8850u >> (2 * w)) & 3;
    } else {
        mb = 0;
        nb = w;
        while (nb > mb) {
            nb -= mb + 1;
            ++mb;
        }
    }
}

template <int MB>
__global__ void __launch_bounds__((consumer_warps<MB>() + 1) * 32, 1)
    gram_stream_kernel(int64_t units, int64_t kchunks, int M, double* __restrict__ partials,
                       const __grid_constant__ CUtensorMap tmap) {
    constexpr int CW = consumer_warps<MB>();
    constexpr int MP = 32 * MB;  // padded rows per chunk
    extern __shared__ __align__(1024) unsigned char gsm_raw[];
    // 1024-byte aligned ring (the swizzle's span); the offset is applied to the
    // shared array itself so the compiler keeps the shared address space (LDS)
    const uint32_t pad = (1024u - (saddr(gsm_raw) & 1023u)) & 1023u;
    double* ring = reinterpret_cast<double*>(gsm_raw + pad);
    constexpr int SD = kGBoxes * MP * kGChunk;  // doubles per stage
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kGStages * SD);
    uint64_t* empty = full + kGStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kGStages; ++s) {
            bar_init(full + s, 1);
            bar_init(empty + s, CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == CW) {
        // producer: one lane issues the chunk copies kGStages ahead
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            const uint32_t bytes = static_cast<uint32_t>(SD * sizeof(double));
            for (int64_t u = u0, i = 0; u < u1; ++u, ++i) {
                const int s = static_cast<int>(i % kGStages);
                if (i >= kGStages) bar_wait(empty + s, static_cast<uint32_t>(((i / kGStages) - 1) & 1));
                bar_expect_tx(full + s, bytes);
                const int64_t b = u / kchunks, kc = u - b * kchunks;
#pragma unroll
                for (int x = 0; x < kGBoxes; ++x)  // (rows beyond K are zero-filled)
                    tma3d(ring + s * SD + x * MP * kGChunk, &tmap, static_cast<int>(kc * kGUnit + x * kGChunk), 0,
                          static_cast<int>(b), full + s, pol);
            }
        }
        return;
    }
    // consumer warp -> lower-triangle block (mb >= nb)
    int mb, nb;
    block_of_warp<MB>(warp, mb, nb);
    const bool diag = mb == nb;
    const int g4 = lane >> 2, t4 = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int64_t u = u0, i = 0; u < u1; ++u, ++i) {
        const int s = static_cast<int>(i % kGStages);
        bar_wait(full + s, static_cast<uint32_t>((i / kGStages) & 1));
#pragma unroll
        for (int ks8 = 0; ks8 < kGUnit / 4; ++ks8) {
            const double* ch = ring + s * SD + (ks8 / (kGChunk / 4)) * MP * kGChunk;
            const int k = 4 * (ks8 % (kGChunk / 4)) + t4;
            double af[4], bf[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) af[t] = ch[swz(32 * mb + 8 * t + g4, k)];
            if (diag) {
#pragma unroll
                for (int t = 0; t < 4; ++t) bf[t] = af[t];
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t) bf[t] = ch[swz(32 * nb + 8 * t + g4, k)];
            }
#pragma unroll
            for (int ti = 0; ti < 4; ++ti)
#pragma unroll
                for (int tj = 0; tj < 4; ++tj)
                    if (!diag || tj <= ti) dmma(acc[ti][tj], af[ti], bf[tj]);
        }
        __syncwarp();
        if (lane == 0) bar_arrive(empty + s);
    }
    double* out = partials + static_cast<int64_t>(blockIdx.x) * MP * MP;
#pragma unroll
    for (int ti = 0; ti < 4; ++ti)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj) {
            if (diag && tj > ti) continue;
            const int m = 32 * mb + 8 * ti + g4, n = 32 * nb + 8 * tj + 2 * t4;
            out[m + MP * n] = acc[ti][tj][0];
            out[m + MP * (n + 1)] = acc[ti][tj][1];
        }
    (void)M;
}

// Gram of mode 0 (rows contiguous: X = Y viewed as [M, C], M <= 128): column
// chunks of 32 staged in shared memory with a row pitch of M + 8 (the
// fragment reads of lanes (g, t) -- row 8 i + g, column 4 s + t -- land on 32
// distinct banks), double buffered with cp.async; one warp per 32 x 32
// lower-triangle block as in gram_stream_kernel. Per-CTA partials, then
// gram_reduce_kernel.
constexpr int kG0Cols = 32;

template <int MB>
__global__ void __launch_bounds__(consumer_warps<MB>() * 32, 1)
    gram_mode0_kernel(const double* __restrict__ X, int M, int64_t C, double* __restrict__ partials) {
    constexpr int MP = 32 * MB;
    constexpr int PITCH = MP + 8;
    constexpr int NT = consumer_warps<MB>() * 32;
    extern __shared__ __align__(16) double g0s[];  // [2][kG0Cols][PITCH]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int64_t nch = (C + kG0Cols - 1) / kG0Cols;
    const int64_t c0 = nch * blockIdx.x / gridDim.x, c1 = nch * (blockIdx.x + 1) / gridDim.x;
    // stage chunk q into buffer b: 16-byte copies (M even), zero rows >= M and columns >= C
    auto stage = [&](int64_t q, int b) {
        double* dst = g0s + b * kG0Cols * PITCH;
        const int halves = MP / 2;
        for (int e = tid; e < kG0Cols * halves; e += NT) {
            const int col = e / halves, h = e - col * halves, m = 2 * h;
            const int64_t cg = q * kG0Cols + col;
            double* d = dst + col * PITCH + m;
            if (cg < C && m < M) {
                const double* src = X + cg * M + m;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(d))),
                             "l"(src)
                             : "memory");
            } else {
                d[0] = 0.0;
                d[1] = 0.0;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int mb, nb;
    block_of_warp<MB>(warp, mb, nb);
    const bool diag = mb == nb;
    const int g4 = lane >> 2, t4 = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (c0 < c1) stage(c0, 0);
    for (int64_t q = c0; q < c1; ++q) {
        const int b = static_cast<int>((q - c0) & 1);
        if (q + 1 < c1) {
            stage(q + 1, b ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* ch = g0s + b * kG0Cols * PITCH;
#pragma unroll
        for (int ks = 0; ks < kG0Cols / 4; ++ks) {
            const double* col = ch + (4 * ks + t4) * PITCH;
            double af[4], bf[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) af[t] = col[32 * mb + 8 * t + g4];
            if (diag) {
#pragma unroll
                for (int t = 0; t < 4; ++t) bf[t] = af[t];
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t) bf[t] = col[32 * nb + 8 * t + g4];
            }
#pragma unroll
            for (int ti = 0; ti < 4; ++ti)
#pragma unroll
                for (int tj = 0; tj < 4; ++tj)
                    if (!diag || tj <= ti) dmma(acc[ti][tj], af[ti], bf[tj]);
        }
        __syncthreads();  // the buffer is refilled two chunks later
    }
    double* out = partials + static_cast<int64_t>(blockIdx.x) * MP * MP;
#pragma unroll
    for (int ti = 0; ti < 4; ++ti)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj) {
            if (diag && tj > ti) continue;
            const int m = 32 * mb + 8 * ti + g4, n = 32 * nb + 8 * tj + 2 * t4;
            out[m + MP * n] = acc[ti][tj][0];
            out[m + MP * (n + 1)] = acc[ti][tj][1];
        }
}

template <int MB>
int launch_mode0_mb(const double* X, int64_t M, int64_t C, double* partials, double* G, int num_sms, cudaStream_t s) {
    constexpr int MP = 32 * MB;
    const int64_t nch = (C + kG0Cols - 1) / kG0Cols;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms, nch)));
    const size_t smem = sizeof(double) * 2 * kG0Cols * (MP + 8);
    ensure_smem_limit(reinterpret_cast<const void*>(gram_mode0_kernel<MB>), smem);
    gram_mode0_kernel<MB><<<grid, consumer_warps<MB>() * 32, smem, s>>>(X, static_cast<int>(M), C, partials);
    return grid;
}

// G[m, m'] = G[m', m] = sum over CTAs (in order) of the lower-triangle partial
__global__ void gram_reduce_kernel(const double* __restrict__ partials, int nparts, int MP, int M,
                                   double* __restrict__ G) {
    const int64_t total = static_cast<int64_t>(M) * M;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(e % M), n = static_cast<int>(e / M);
        const int r = m >= n ? m : n, c = m >= n ? n : m;  // lower-triangle source
        double s = 0.0;
        for (int p = 0; p < nparts; ++p) s += partials[static_cast<int64_t>(p) * MP * MP + r + static_cast<int64_t>(MP) * c];
        G[m + static_cast<int64_t>(M) * n] = s;
    }
}

// Gram of a mode with at most 8 rows (c4's 8-extent modes): every (k, b)
// column x = Y[k, :, b] is read once by one thread, which accumulates the
// lower triangle of x x^T in registers; warp, CTA and grid sums in a fixed
// order (partials per CTA, then gram_small_finish_kernel).
constexpr int kSmallThreads = 256;

template <int M>
__global__ void __launch_bounds__(kSmallThreads) gram_small_kernel(const double* __restrict__ Y, uint32_t K,
                                                                   uint32_t units, double* __restrict__ partials) {
    constexpr int L = M * (M + 1) / 2;
    double acc[L];
#pragma unroll
    for (int e = 0; e < L; ++e) acc[e] = 0.0;
    for (uint32_t u = blockIdx.x * kSmallThreads + threadIdx.x; u < units; u += gridDim.x * kSmallThreads) {
        const uint32_t b = u / K, k = u - b * K;
        const double* col = Y + k + static_cast<uint64_t>(K) * M * b;
        double x[M];
#pragma unroll
        for (int m = 0; m < M; ++m) x[m] = __ldg(col + static_cast<uint64_t>(K) * m);
        int e = 0;
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
            for (int i = j; i < M; ++i, ++e) acc[e] = fma(x[i], x[j], acc[e]);
    }
    __shared__ double red[kSmallThreads / 32][L];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < L; ++e) {
        double v = acc[e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp][e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < L; e += kSmallThreads) {
        double v = 0.0;
        for (int w = 0; w < kSmallThreads / 32; ++w) v += red[w][e];
        partials[static_cast<int64_t>(blockIdx.x) * L + e] = v;
    }
}

__global__ void gram_small_finish_kernel(const double* __restrict__ partials, int nparts, int M,
                                         double* __restrict__ G) {
    // one warp per lower-triangle entry e (enumerated column by column):
    // fixed lane striding and shuffle tree
    const int L = M * (M + 1) / 2, e = blockIdx.x;
    double v = 0.0;
    for (int p = threadIdx.x; p < nparts; p += 32) v += partials[static_cast<int64_t>(p) * L + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) {
        int j = 0, rem = e;
        while (rem >= M - j) {
            rem -= M - j;
            ++j;
        }
        const int i = j + rem;
        G[i + M * j] = v;
        G[j + M * i] = v;
    }
}

// Gram of a mode with 9..32 rows (c1's 16-row leaves, c3's 32-row mode 0,
// any mode incl. 0): Y viewed as [K, M, B], columns (k, b) taken 4 at a
// time as the k dimension of m8n8k4 DMMAs. Lane (g, t) loads rows 8 mt + g
// of column 4 q + t once; that value is both the A fragment of row tile mt
// and the B fragment of column tile mt, so the lower-triangle blocks
// (mt >= nt) accumulate in registers. Per-CTA partials in a fixed order,
// then gram_small_finish_kernel.
constexpr int kMidWarps = 8;

template <int MT>
__global__ void __launch_bounds__(kMidWarps * 32) gram_mid_kernel(const double* __restrict__ Y, uint32_t K,
                                                                  uint32_t M, uint32_t units4, uint32_t units,
                                                                  double* __restrict__ partials) {
    constexpr int NB = MT * (MT + 1) / 2;
    double acc[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b][0] = acc[b][1] = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const uint32_t gw = blockIdx.x * kMidWarps + warp, nw = gridDim.x * kMidWarps;
    for (uint32_t q = gw; q < units4; q += nw) {
        const uint32_t u = 4 * q + t;  // column (k, b) = (u % K, u / K)
        double a[MT];
        if (u < units) {
            const uint32_t bb = u / K, k = u - bb * K;
            const double* col = Y + k + static_cast<uint64_t>(K) * M * bb;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const uint32_t m = 8 * mt + g;
                a[mt] = m < M ? __ldg(col + static_cast<uint64_t>(K) * m) : 0.0;
            }
        } else {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) a[mt] = 0.0;
        }
        int b = 0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt <= mt; ++nt, ++b) dmma(acc[b], a[mt], a[nt]);
    }
    // lower triangle (i >= j) of the M x M Gram, enumerated column by column
    // as in gram_small (entry e of column j, row i)
    __shared__ double red[kMidWarps][32 * 33 / 2];
    const int L = static_cast<int>(M * (M + 1) / 2);
    for (int e = lane; e < L; e += 32) red[warp][e] = 0.0;
    __syncwarp();
    int b = 0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt <= mt; ++nt, ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = 8 * mt + g, j = 8 * nt + 2 * t + h;
                if (i < static_cast<int>(M) && j <= i) {
                    const int e = j * static_cast<int>(M) - (j * (j - 1)) / 2 + (i - j);
                    red[warp][e] = acc[b][h];
                }
            }
    __syncthreads();
    for (int e = threadIdx.x; e < L; e += kMidWarps * 32) {
        double v = 0.0;
        for (int w = 0; w < kMidWarps; ++w) v += red[w][e];
        partials[static_cast<int64_t>(blockIdx.x) * L + e] = v;
    }
}

template <int MT>
int launch_mid_mt(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, double* G, int num_sms,
                  cudaStream_t s) {
    const int64_t units = K * B, units4 = (units + 3) / 4;
    const int grid = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(2 * num_sms, (units4 + kMidWarps - 1) / kMidWarps)));
    gram_mid_kernel<MT><<<grid, kMidWarps * 32, 0, s>>>(Y, static_cast<uint32_t>(K), static_cast<uint32_t>(M),
                                                       static_cast<uint32_t>(units4), static_cast<uint32_t>(units),
                                                       partials);
    gram_small_finish_kernel<<<static_cast<unsigned>(M * (M + 1) / 2), 32, 0, s>>>(partials, grid,
                                                                                   static_cast<int>(M), G);
    return grid;
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

template <int MB>
size_t gram_smem_bytes() {
    return sizeof(double) * kGStages * kGBoxes * 32 * MB * kGChunk + 2 * kGStages * sizeof(uint64_t) + 1024;
}

template <int MB>
int launch_mb(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, int grid, const CUtensorMap& map,
              cudaStream_t s) {
    const int64_t kchunks = (K + kGUnit - 1) / kGUnit;
    const size_t smem = gram_smem_bytes<MB>();
    ensure_smem_limit(reinterpret_cast<const void*>(gram_stream_kernel<MB>), smem);
    gram_stream_kernel<MB><<<grid, (consumer_warps<MB>() + 1) * 32, smem, s>>>(B * kchunks, kchunks, static_cast<int>(M),
                                                                               partials, map);
    (void)Y;
    return grid;
}

template <int M>
int launch_small_m(const double* Y, int64_t K, int64_t B, double* partials, double* G, int num_sms, cudaStream_t s) {
    const int64_t units = K * B;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4 * num_sms, (units + kSmallThreads - 1) / kSmallThreads)));
    gram_small_kernel<M><<<grid, kSmallThreads, 0, s>>>(Y, static_cast<uint32_t>(K), static_cast<uint32_t>(units), partials);
    gram_small_finish_kernel<<<M * (M + 1) / 2, 32, 0, s>>>(partials, grid, M, G);
    return grid;
}

}  // namespace

bool gram_small_supported(int64_t K, int64_t M, int64_t B) {
    return M >= 1 && M <= 8 && K >= 1 && B >= 1 && K * B < (int64_t{1} << 31) && K * M * B < (int64_t{1} << 40);
}

int64_t gram_small_partials(int num_sms) { return static_cast<int64_t>(4 * num_sms) * 36; }

bool gram_mid_supported(int64_t K, int64_t M, int64_t B) {
    return M >= 9 && M <= 32 && K >= 1 && B >= 1 && K * B < (int64_t{1} << 31) - 8 && K * M * B < (int64_t{1} << 40);
}

int64_t gram_mid_partials(int num_sms) { return static_cast<int64_t>(2 * num_sms) * (32 * 33 / 2); }

int launch_gram_mid(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, double* G, int num_sms,
                    cudaStream_t s, int64_t* launches) {
    if (!gram_mid_supported(K, M, B)) return -1;
    int grid;
    switch ((M + 7) / 8) {
        case 2: grid = launch_mid_mt<2>(Y, K, M, B, partials, G, num_sms, s); break;
        case 3: grid = launch_mid_mt<3>(Y, K, M, B, partials, G, num_sms, s); break;
        default: grid = launch_mid_mt<4>(Y, K, M, B, partials, G, num_sms, s); break;
    }
    *launches += 2;
    return grid;
}

int launch_gram_small(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, double* G, int num_sms,
                      cudaStream_t s, int64_t* launches) {
    if (!gram_small_supported(K, M, B)) return -1;
    int grid;
    switch (M) {
        case 1: grid = launch_small_m<1>(Y, K, B, partials, G, num_sms, s); break;
        case 2: grid = launch_small_m<2>(Y, K, B, partials, G, num_sms, s); break;
        case 3: grid = launch_small_m<3>(Y, K, B, partials, G, num_sms, s); break;
        case 4: grid = launch_small_m<4>(Y, K, B, partials, G, num_sms, s); break;
        case 5: grid = launch_small_m<5>(Y, K, B, partials, G, num_sms, s); break;
        case 6: grid = launch_small_m<6>(Y, K, B, partials, G, num_sms, s); break;
        case 7: grid = launch_small_m<7>(Y, K, B, partials, G, num_sms, s); break;
        default: grid = launch_small_m<8>(Y, K, B, partials, G, num_sms, s); break;
    }
    *launches += 2;
    return grid;
}

bool gram_stream_supported(const double* Y, int64_t K, int64_t M, int64_t B) {
    return M >= 1 && M <= 128 && K >= 2 && (K & 1) == 0 && B >= 1 && B < (int64_t{1} << 31) &&
           K < (int64_t{1} << 31) && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 && encoder() != nullptr;
}

int64_t gram_stream_partials(int64_t M, int num_sms) {
    const int64_t MP = (M + 31) / 32 * 32;
    return static_cast<int64_t>(num_sms) * MP * MP;
}

bool gram_mode0_supported(const double* X, int64_t M, int64_t C) {
    return M >= 2 && M <= 128 && (M % 2) == 0 && C >= 1 && (reinterpret_cast<uintptr_t>(X) & 15u) == 0;
}

int launch_gram_mode0(const double* X, int64_t M, int64_t C, double* partials, double* G, int num_sms, cudaStream_t s,
                      int64_t* launches) {
    if (!gram_mode0_supported(X, M, C)) return -1;
    const int MB = static_cast<int>((M + 31) / 32);
    int grid;
    if (MB == 1) grid = launch_mode0_mb<1>(X, M, C, partials, G, num_sms, s);
    else if (MB == 2) grid = launch_mode0_mb<2>(X, M, C, partials, G, num_sms, s);
    else if (MB == 3) grid = launch_mode0_mb<3>(X, M, C, partials, G, num_sms, s);
    else grid = launch_mode0_mb<4>(X, M, C, partials, G, num_sms, s);
    gram_reduce_kernel<<<std::max(1, std::min(num_sms, static_cast<int>((M * M + 255) / 256))), 256, 0, s>>>(
        partials, grid, 32 * MB, static_cast<int>(M), G);
    *launches += 2;
    return grid;
}

int launch_gram_stream(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, double* G, int num_sms,
                       cudaStream_t s, int64_t* launches) {
    if (!gram_stream_supported(Y, K, M, B)) return -1;
    const int MB = static_cast<int>((M + 31) / 32);
    const int MP = 32 * MB;
    alignas(64) CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(B)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(K * 8), static_cast<cuuint64_t>(K * M * 8)};
    cuuint32_t box[3] = {kGChunk, static_cast<cuuint32_t>(MP), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(Y), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
    const int64_t units = B * ((K + kGUnit - 1) / kGUnit);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms, units)));
    if (MB == 1) launch_mb<1>(Y, K, M, B, partials, grid, map, s);
    else if (MB == 2) launch_mb<2>(Y, K, M, B, partials, grid, map, s);
    else if (MB == 3) launch_mb<3>(Y, K, M, B, partials, grid, map, s);
    else launch_mb<4>(Y, K, M, B, partials, grid, map, s);
    gram_reduce_kernel<<<std::max(1, std::min(num_sms, static_cast<int>((M * M + 255) / 256))), 256, 0, s>>>(
        partials, grid, MP, static_cast<int>(M), G);
    *launches += 2;
    return grid;
}

}  // namespace htr
