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
// the r0 r1 r2 / (N0 N1 n2)-size Z.
//
// Structure (one CTA per SM, no CTA barriers in the main loop). A CTA owns a
// contiguous range of slabs X = Y[:, :, i2, s] (N0 x N1, contiguous). Its 12
// warps take whole slabs in rounds (warp w: slabs w, w + 12, ...); the last
// partial round (fewer than 12 slabs) is split evenly over all warps at
// column-pair granularity (16 columns), so no warp has more than 1/8 slab
// more work than another at any batch size (c5 per-rank shards at 8 GPUs:
// 27-28 slabs per CTA). A slab split between warps has its partial W pieces
// summed in warp order at the end of the kernel (deterministic).
// Each warp walks its slabs in steps of 16 columns x 32 rows; each step
// arrives by two TMA tensor copies (cp.async.bulk.tensor.3d over a
// [N0, N1, slabs] tensor map, 16x16 boxes, 128-byte swizzle) into the warp's
// own 4-deep shared-memory ring, issued by one lane three steps ahead and
// completed on a per-stage mbarrier. The MMA's
// column order is permuted (n-index g -> physical column pi(g)) so that the
// swizzled fragment reads are bank-conflict-free; step 2 undoes the
// permutation through the order of the U1 fragments;
//   * step 1  P = U0^T X    DMMA 8x8x4 with U0^T fragments from shared memory;
//   * step 2  W += P U1     P's accumulator fragments re-used in registers as
//                           the A operand (MMA k index permuted to the C layout);
//   * per slab the warp writes W (r0 x r1) to global memory; a DMMA GEMM
//     then contracts the slab axis with U2:  Z_s = sum_i2 W_(s,i2) (x) U2[i2,:].
// Everything is deterministic: no atomics, fixed reduction trees.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kWarps = 12;
constexpr int kThreads = kWarps * 32;
constexpr int kStages = 3;         // per-warp ring depth
constexpr int kRows = 32;          // rows (i0) per step
constexpr int kCols = 16;          // columns (i1) per step = 2 DMMA n-tiles
constexpr int kBoxRows = 16;      // TMA box: 16 doubles (128 B, the swizzle span) x 16 columns
constexpr int kBoxDoubles = kBoxRows * kCols;
constexpr int kStageDoubles = kCols * kRows;  // two boxes
constexpr uint32_t kStageBytes = kCols * kRows * sizeof(double);

// physical column (within an 8-column MMA n-tile) of MMA n-index g: lanes
// g and g+1 of a quarter-warp land in columns differing in bit 2, whose
// 128-byte swizzle XOR sends them to disjoint 16-byte bank groups
__host__ __device__ __forceinline__ int col_perm(int g) { return (g >> 1) + 4 * (g & 1); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// global -> shared tensor copy (TMA engine), completion counted on `bar`;
// the batch is read exactly once, so it is marked evict-first in L2
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

struct RangeInfo {
    int64_t T;  // total slabs = n2 * S
    int n0, n1; // slab extents (<= the kernel's N0, N1; n0 even)
};

__host__ __device__ __forceinline__ int64_t cta_begin(int64_t T, int64_t b, int64_t B) { return (T * b) / B; }

// EXACT: the slabs are N0 x N1 (all step counts compile-time). Otherwise the
// slabs are n0 x n1 with n0 <= N0 (even), n1 <= N1: the tensor map carries
// the true extents, TMA zero-fills the out-of-range part of a box, the basis
// fragments are zero beyond n0 / n1, and only the steps that touch the slab
// are walked (n0 = 96 on the 128-row kernel: 3 of 4 row quarters).
template <int N0, int N1, int MT0, int MT1, bool EXACT, int ST = kStages>
__global__ void __launch_bounds__(kThreads, 1)
    fused3_kernel(const Fused3Args a, const RangeInfo ri, const __grid_constant__ CUtensorMap tmap) {
    constexpr int NC = N0 / 8;      // 8-row chunks per column block
    const int n0 = EXACT ? N0 : ri.n0, n1 = EXACT ? N1 : ri.n1;
    const int NQ = EXACT ? N0 / kRows : (ri.n0 + kRows - 1) / kRows;  // steps per column pair
    const int NP = EXACT ? N1 / kCols : (ri.n1 + kCols - 1) / kCols;  // column pairs per slab
    const int IPS = NP * NQ;        // steps per slab
    extern __shared__ __align__(1024) double smem_raw[];
    // stages first: the 128-byte swizzle needs 1024-byte aligned boxes
    double* stages = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u) / sizeof(double);  // [warp][stage][box][col][16]
    double2* U0f = reinterpret_cast<double2*>(stages + kWarps * ST * kStageDoubles);  // [NC][MT0][32]
    double2* U1f = U0f + NC * MT0 * 32;                                              // [N1/8][MT1][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(U1f + (N1 / 8) * MT1 * 32);  // [warp][stage]
    __shared__ double red[kWarps];
    __shared__ int64_t piece_slab[kWarps][2];  // slab of a warp's partial head / tail piece, or -1

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int R01 = a.r0 * a.r1;

    if (tid < 2 * kWarps) piece_slab[tid >> 1][tid & 1] = -1;

    const int64_t B = gridDim.x, b = blockIdx.x;
    const int64_t tb = cta_begin(ri.T, b, B), te = cta_begin(ri.T, b + 1, B);
    // whole-slab rounds, then this warp's share [u0, u1) of the last partial
    // round's (slab, column pair) units
    // (slab indices fit in 32 bits: make_batch_map rejects T >= 2^31)
    const int tb32 = static_cast<int>(tb);
    const int rounds = static_cast<int>(te - tb) / kWarps;
    const int tr = tb32 + rounds * kWarps;  // first slab of the partial round
    const int units = (static_cast<int>(te) - tr) * NP;
    const int u0 = units * warp / kWarps, u1 = units * (warp + 1) / kWarps;
    const int whole = rounds * IPS;         // steps in whole slabs
    const int total = whole + (u1 - u0) * NQ;
    // step i -> slab, column pair, row quarter; unit index u (partial round only)
    auto coords = [&](int i, int& t, int& pair, int& q, int& u) {
        if (i < whole) {
            const int j = i / IPS;
            const int rem = i - j * IPS;
            pair = rem / NQ;
            q = rem - pair * NQ;
            t = tb32 + warp + kWarps * j;
            u = -1;
        } else {
            const int k = i - whole;
            u = u0 + k / NQ;
            q = k % NQ;
            pair = u % NP;
            t = tr + u / NP;
        }
    };
    double* my_stages = stages + warp * ST * kStageDoubles;
    uint64_t* my_full = full + warp * ST;
    const uint64_t policy = evict_first_policy();
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");

    auto issue = [&](int i) {  // lane 0 only
        const int st = i % ST;
        int t, u, pair, q;
        coords(i, t, pair, q, u);
        mbar_expect_tx(&my_full[st], kStageBytes);
        double* dst = my_stages + st * kStageDoubles;
        tma_load_3d(dst, &tmap, kRows * q, kCols * pair, t, &my_full[st], policy);
        tma_load_3d(dst + kBoxDoubles, &tmap, kRows * q + kBoxRows, kCols * pair, t, &my_full[st], policy);
    };
    // lane 0 sets up its warp's ring and starts the stream before the basis
    // fragments are staged (the first loads' latency overlaps the staging)
    if (lane == 0) {
        for (int k = 0; k < ST; ++k) mbar_init(&my_full[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < ST; ++k)
            if (k < total) issue(k);
    }
    // ---- stage basis fragments (zero-padded to 8-multiples) ----
    for (int idx = tid; idx < NC * MT0 * 32; idx += kThreads) {
        const int l = idx & 31, mt = (idx >> 5) % MT0, c = idx / (32 * MT0);
        const int i0 = 8 * c + 2 * (l & 3), col = 8 * mt + (l >> 2);
        double2 v;
        const bool ok = col < a.r0 && i0 < n0;  // (n0 even: i0 + 1 < n0 too)
        v.x = ok ? a.U0[i0 + static_cast<int64_t>(n0) * col] : 0.0;
        v.y = ok ? a.U0[i0 + 1 + static_cast<int64_t>(n0) * col] : 0.0;
        U0f[idx] = v;
    }
    for (int idx = tid; idx < (N1 / 8) * MT1 * 32; idx += kThreads) {
        const int l = idx & 31, mt = (idx >> 5) % MT1, nt = idx / (32 * MT1);
        const int i1x = 8 * nt + col_perm(2 * (l & 3)), i1y = 8 * nt + col_perm(2 * (l & 3) + 1);
        const int col = 8 * mt + (l >> 2);
        double2 v;
        v.x = (col < a.r1 && i1x < n1) ? a.U1[i1x + static_cast<int64_t>(n1) * col] : 0.0;
        v.y = (col < a.r1 && i1y < n1) ? a.U1[i1y + static_cast<int64_t>(n1) * col] : 0.0;
        U1f[idx] = v;
    }
    __syncthreads();
    // the skip-path tail is launched as a programmatic dependent: it may be
    // scheduled as this grid's CTAs retire and stages its bases before
    // waiting for this grid's results (griddepcontrol.wait in tail3)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    double ysq0 = 0.0, ysq1 = 0.0, ysq2 = 0.0, ysq3 = 0.0;
    double wacc[MT0][MT1][2];
    double pacc[MT0][2][2];
#pragma unroll
    for (int i = 0; i < MT0; ++i)
#pragma unroll
        for (int j = 0; j < MT1; ++j) wacc[i][j][0] = wacc[i][j][1] = 0.0;

    for (int i = 0; i < total; ++i) {
        const int st = i % ST;
        int t, u, pair, q;
        coords(i, t, pair, q, u);
        if (q == 0) {
#pragma unroll
            for (int x = 0; x < MT0; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) pacc[x][y][0] = pacc[x][y][1] = 0.0;
        }
        mbar_wait(&my_full[st], static_cast<uint32_t>((i / ST) & 1));
        const double* sb = my_stages + st * kStageDoubles;
        const int pc0 = col_perm(g4), pc1 = 8 + col_perm(g4);
#pragma unroll
        for (int cc = 0; cc < kRows / 8; ++cc) {
            const int c = q * (kRows / 8) + cc;
            const int box = cc >> 1, chunk = 4 * (cc & 1) + t4;  // 16-byte chunk within the 128-byte column
            const double* bb = sb + box * kBoxDoubles;
            const double2 x0 = *reinterpret_cast<const double2*>(bb + pc0 * kBoxRows + 2 * (chunk ^ (pc0 & 7)));
            const double2 x1 = *reinterpret_cast<const double2*>(bb + pc1 * kBoxRows + 2 * (chunk ^ (pc1 & 7)));
            double2 u[MT0];
#pragma unroll
            for (int ma = 0; ma < MT0; ++ma) u[ma] = U0f[(c * MT0 + ma) * 32 + lane];
            ysq0 = fma(x0.x, x0.x, ysq0);
            ysq1 = fma(x0.y, x0.y, ysq1);
            ysq2 = fma(x1.x, x1.x, ysq2);
            ysq3 = fma(x1.y, x1.y, ysq3);
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
        // the stage is consumed (its values fed warp-collective MMAs): order
        // the generic-proxy reads before the async-proxy refill
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (i + ST < total) issue(i + ST);
        }

        if (q == NQ - 1) {
            // step 2: W += P U1 over this pair's 16 columns
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int ntile = 2 * pair + nt;
                double2 u[MT1];
#pragma unroll
                for (int mb = 0; mb < MT1; ++mb) u[mb] = U1f[(ntile * MT1 + mb) * 32 + lane];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int mb = 0; mb < MT1; ++mb)
#pragma unroll
                        for (int ma = 0; ma < MT0; ++ma)
                            dmma(wacc[ma][mb], pacc[ma][nt][h], h ? u[mb].y : u[mb].x);
            }
            if (pair == NP - 1 || (u >= 0 && u == u1 - 1)) {
                // this warp's piece of the slab done: publish W (compact
                // a0 + r0 a1) and reset; a partial piece (the slab is shared
                // with a neighbouring warp) goes to the warp's head/tail slot
                const bool from_start = u < 0 || u - pair >= u0;  // the piece includes column pair 0
                double* wdst = a.wslab + static_cast<int64_t>(t) * R01;
                if (!(from_start && pair == NP - 1)) {
                    const int which = from_start ? 1 : 0;
                    wdst = a.wpart + ((static_cast<int64_t>(b) * kWarps + warp) * 2 + which) * R01;
                    if (lane == 0) piece_slab[warp][which] = t;
                }
#pragma unroll
                for (int ma = 0; ma < MT0; ++ma)
#pragma unroll
                    for (int mb = 0; mb < MT1; ++mb)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int a0 = 8 * ma + g4, a1 = 8 * mb + 2 * t4 + h;
                            if (a0 < a.r0 && a1 < a.r1) wdst[a0 + a.r0 * a1] = wacc[ma][mb][h];
                            wacc[ma][mb][h] = 0.0;
                        }
            }
        }
    }

    __syncthreads();
    // slabs split between warps: W = the pieces summed in warp order
    __shared__ int64_t split[2 * kWarps];
    __shared__ int nsplit;
    if (tid == 0) {
        int n = 0;
        for (int k = 0; k < 2 * kWarps; ++k) {
            const int64_t t = piece_slab[k >> 1][k & 1];
            bool seen = t < 0;
            for (int m = 0; m < n && !seen; ++m) seen = split[m] == t;
            if (!seen) split[n++] = t;
        }
        nsplit = n;
    }
    __syncthreads();
    const double* parts = a.wpart + static_cast<int64_t>(b) * kWarps * 2 * R01;
#pragma unroll 2
    for (int idx = tid; idx < nsplit * R01; idx += kThreads) {
        const int m = idx / R01, e = idx - m * R01;
        const int64_t t = split[m];
        double v = 0.0;
        for (int k = 0; k < 2 * kWarps; ++k)
            if (piece_slab[k >> 1][k & 1] == t) v += __ldcg(parts + static_cast<int64_t>(k) * R01 + e);
        a.wslab[t * R01 + e] = v;
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

template <int N0, int N1, int MT0, int MT1, int ST>
size_t smem_bytes() {
    return sizeof(double) * (static_cast<size_t>(N0 / 8) * MT0 * 64 + static_cast<size_t>(N1 / 8) * MT1 * 64 +
                             static_cast<size_t>(kWarps) * ST * kStageDoubles) +
           sizeof(uint64_t) * kWarps * ST + 1024;  // + alignment slack
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

/// [N0, N1, T] view of the batch (T = n2 * S slabs), 16 x 16 x 1 boxes.
bool make_batch_map(CUtensorMap* map, const double* Y, int64_t N0, int64_t N1, int64_t T) {
    auto enc = tensor_map_encoder();
    if (!enc || (reinterpret_cast<uintptr_t>(Y) & 15) || T > (int64_t{1} << 31)) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(N0), static_cast<cuuint64_t>(N1), static_cast<cuuint64_t>(T)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(N0 * 8), static_cast<cuuint64_t>(N0 * N1 * 8)};
    cuuint32_t box[3] = {kBoxRows, kCols, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(Y), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N0, int N1, int MT0, int MT1, bool EXACT, int ST = kStages>
int launch_impl(int64_t n0, int64_t n1, const Fused3Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    const int64_t T = a.n2 * a.S;
    const int64_t B = std::min<int64_t>(num_sms, T);
    RangeInfo ri{T, static_cast<int>(n0), static_cast<int>(n1)};
    Fused3Args args = a;
    args.wpart = a.ysq_partials + B;  // B * kWarps * 2 * r0 r1 doubles (fused3_workspace_doubles)
    alignas(64) CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (!make_batch_map(&map, a.Y, n0, n1, T)) return -1;
    const size_t smem = smem_bytes<N0, N1, MT0, MT1, ST>();
    auto kfn = fused3_kernel<N0, N1, MT0, MT1, EXACT, ST>;
    ensure_smem_limit(reinterpret_cast<const void*>(kfn), smem);
    kfn<<<static_cast<unsigned>(B), kThreads, smem, s>>>(args, ri, map);
    ++*launches;
    if (!a.slab_gemm) return static_cast<int>(B);
    // Z_s[p, a2] = sum_i2 W[(s, i2), p] U2[i2, a2]: the slab-axis (mode 2)
    // contraction, one small GEMM per sample
    GemmDesc d;
    const int64_t R01 = static_cast<int64_t>(a.r0) * a.r1;
    d.M = R01;
    d.N1 = a.r2;
    d.K1 = a.n2;
    d.batch = a.S;
    d.A = a.wslab;
    d.sam = 1;
    d.sak1 = R01;
    d.sab = R01 * a.n2;
    d.B = a.U2;
    d.sbk1 = 1;
    d.sbn1 = a.n2;
    d.C = a.Z;
    d.scm = 1;
    d.scn1 = R01;
    d.scb = R01 * a.r2;
    launch_gemm(d, nullptr, num_sms, s, launches);
    return static_cast<int>(B);
}

template <int N0, int N1, bool EXACT, int ST = kStages>
int dispatch_mt(int mt, int64_t n0, int64_t n1, const Fused3Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    switch (mt) {
        case 1: return launch_impl<N0, N1, 1, 1, EXACT, ST>(n0, n1, a, num_sms, s, launches);
        case 2: return launch_impl<N0, N1, 2, 2, EXACT, ST>(n0, n1, a, num_sms, s, launches);
        case 3: return launch_impl<N0, N1, 3, 3, EXACT, ST>(n0, n1, a, num_sms, s, launches);
        default: return -1;
    }
}

}  // namespace

bool fused3_supported(int64_t n0, int64_t n1, int64_t n2, int r0, int r1, int r2) {
    (void)n2;
    // slabs up to 256 x 256; n0 even (16-byte rows for the tensor map) and a
    // slab large enough that the 16 x 32 steps are not mostly padding
    if (n0 < 16 || n1 < 16 || n0 > 256 || n1 > 256 || (n0 & 1)) return false;
    if (r0 < 1 || r1 < 1 || r2 < 1 || r0 > 24 || r1 > 24) return false;
    return true;
}

int64_t fused3_workspace_doubles(int64_t n0, int64_t n1, int64_t n2, int64_t S, int r0, int r1, int r2,
                                 int num_sms) {
    (void)n0;
    (void)n1;
    (void)r2;
    const int64_t T = n2 * S;
    const int64_t B = std::min<int64_t>(num_sms, T);
    // per-slab W + ||Y||^2 partials + split-slab pieces (2 per warp)
    return T * static_cast<int64_t>(r0) * r1 + B + B * kWarps * 2 * static_cast<int64_t>(r0) * r1;
}

int launch_fused3(int64_t n0, int64_t n1, const Fused3Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    const int mt = (std::max(a.r0, a.r1) + 7) / 8;
    if (n0 == 128 && n1 == 128) return dispatch_mt<128, 128, true>(mt, n0, n1, a, num_sms, s, launches);
    if (n0 == 64 && n1 == 64) return dispatch_mt<64, 64, true>(mt, n0, n1, a, num_sms, s, launches);
    if (n0 == 128 && n1 == 64) return dispatch_mt<128, 64, true>(mt, n0, n1, a, num_sms, s, launches);
    if (n0 == 64 && n1 == 128) return dispatch_mt<64, 128, true>(mt, n0, n1, a, num_sms, s, launches);
    if (n0 == 32 && n1 == 32) return dispatch_mt<32, 32, true>(mt, n0, n1, a, num_sms, s, launches);
    // any other slab: the smallest kernel that holds it (the basis fragments
    // in shared memory are sized by the kernel's extents)
    if (n0 < 2 || n0 > 256 || n1 < 1 || n1 > 256 || (n0 & 1)) return -1;
    // above 128: the 256 x 256 kernel with two-stage rings (the basis
    // fragments of both modes take 96 KB of shared memory at ranks 17..24)
    if (n0 > 128 || n1 > 128) return dispatch_mt<256, 256, false, 2>(mt, n0, n1, a, num_sms, s, launches);
    if (n0 <= 32 && n1 <= 32) return dispatch_mt<32, 32, false>(mt, n0, n1, a, num_sms, s, launches);
    if (n0 <= 64 && n1 <= 64) return dispatch_mt<64, 64, false>(mt, n0, n1, a, num_sms, s, launches);
    if (n0 <= 64) return dispatch_mt<64, 128, false>(mt, n0, n1, a, num_sms, s, launches);
    if (n1 <= 64) return dispatch_mt<128, 64, false>(mt, n0, n1, a, num_sms, s, launches);
    return dispatch_mt<128, 128, false>(mt, n0, n1, a, num_sms, s, launches);
}

}  // namespace htr
