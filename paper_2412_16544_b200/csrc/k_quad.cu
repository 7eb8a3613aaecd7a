// Skip-path encode of a balanced 4-leaf subtree in one read of the batch.
//
// Replaces, for a subtree whose leaves are four consecutive modes m..m+3 of
// extent 8 with ranks 4 (config 4: an 8-way 8^8 batch on balanced(8), every
// rank 4), the leaf projections of encode (bht.hpp:381-383 -> project_mode
// 357-365), the two layer-2 transfer projections and the subtree root's
// transfer projection (bht.hpp:385-399): every 8^4 block of the batch (the
// subtree's modes, 32 KB) becomes the subtree's 4 outputs. Two launches give
// the latent of an 8-way batch: the first over y (modes 0-3 contiguous,
// 537 MB read once, 2 MB written as [8^4 (modes 4-7), 4, N] so that the
// second subtree's blocks are contiguous too), the second over that result,
// which also finishes ||y||^2 and ||latent||^2 (last CTA, fixed order) like
// the 3-way tail.
//
// One warp per block (8 warps per CTA, a 3-deep ring of 4 KB TMA bulk
// chunks per warp, no CTA barriers in the loop):
//   stage 0+1  per chunk (one e3 slice): p0 = U0^T x per fibre,
//              P1 += p0 (x) U1[e1, :]; ||x||^2 on the side;
//   stage 2    mode e2 per chunk; stage 3 mode e3 per block;
//   stage 4-6  the three 16 x 4 transfer projections.
// The finishing launch (few blocks) runs one CTA per block, a chunk per warp.
// All FP64 FMAs (DFMA; the contractions are 8 -> 4, far too thin for DMMA
// tiles): ~36k FMA per 4096-element block. Measured (c4): 128 us over the
// 537 MB batch = 4.2 TB/s, issue/latency-bound at 2 warps per scheduler
// (190 registers), profiles/r1_quad_ncu_summary.txt.
#include <algorithm>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int QN = 8, QR = 4;
constexpr int kQBlock = QN * QN * QN * QN;  // elements per subtree block

// Each warp streams its blocks through a ring of 4 KB chunks in shared
// memory with TMA bulk copies
// (cp.async.bulk, one per chunk, mbarrier completion): chunk k of a block is
// e3 = k (8 columns e2 of 64 contiguous doubles). Lane (e2 = lane / 4,
// j = lane % 4) takes fibres e1 = j and j + 4; a per-lane rotation of the
// 16-byte parts it reads keeps the shared-memory reads conflict-free (U0
// rows are read with the same rotation). P1 partials are reduced over the 4
// j-lanes by shuffles, then mode e2 runs per chunk and modes e3 + the
// transfers per block, as above.
constexpr int kQ2Warps = 8;   // finishing launch (one chunk per warp in the split mode)
constexpr int kQ1Warps = 12;  // streaming pass over y
constexpr int kQ1Stages = 2;
constexpr int kQ2Threads = kQ2Warps * 32;
constexpr int kQ2Stages = 3;
constexpr int kQ2Chunk = 512;                        // doubles (4 KB): one e3 slice of a block
constexpr int kQ2Scratch = 128 + 512 + 256 + 64 + 16;  // S1 (one chunk), S2, S3, V01, V

__device__ __forceinline__ uint32_t q_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <bool FINISH, bool SPLIT, int NW, int NST>
__global__ void __launch_bounds__(NW * 32, 1) quad_stream_kernel(const QuadArgs a) {
    // SPLIT (few blocks: the finishing launch): one CTA per block, warp w
    // takes chunk w (e3 = w); warp 0 finishes the block after a CTA barrier
    static_assert(!SPLIT || NW == QN, "one chunk per warp");
    __shared__ double Us[4][QN * QR];
    __shared__ double Ts[3][QR * QR * QR];
    __shared__ double red[NW];
    __shared__ __align__(8) uint64_t full[NW][NST];
    extern __shared__ __align__(128) double dyn[];  // [warp][stage][512] then [warp][scratch]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < 4 * QN * QR; e += (NW * 32)) {
        const int m = e / (QN * QR), r = e % (QN * QR), j = r / QR, q = r % QR;
        Us[m][r] = a.U[m][j + QN * q];
    }
    for (int e = tid; e < 3 * QR * QR * QR; e += (NW * 32)) {
        const int m = e / (QR * QR * QR), r = e % (QR * QR * QR), k = r / QR, b = r % QR;
        const double* T = m == 0 ? a.T01 : (m == 1 ? a.T23 : a.T);
        Ts[m][r] = T[k + QR * QR * b];
    }
    double* ring = dyn + warp * NST * kQ2Chunk;
    double* S1 = dyn + NW * NST * kQ2Chunk + warp * kQ2Scratch;  // [k16][e2]
    double* S2 = (SPLIT ? dyn + NW * NST * kQ2Chunk : S1) + 128;  // [k16][a2][e3] (CTA-shared in SPLIT)
    double* S3 = S2 + 512;   // [(a0,a1,a2)][a3]
    double* V01 = S3 + 256;
    double* V = V01 + 64;
    uint64_t* bar = full[warp];

    const int64_t units = a.O;
    // every CTA owns an equal contiguous share of the blocks (+-1), dealt
    // round-robin to its warps: the partly filled last round is spread over
    // all SMs (a grid-strided deal gave 34 of the 148 SMs a full extra round
    // at c4's 16384 blocks: 120 blocks against 108 on the others)
    const int64_t lo = units * blockIdx.x / gridDim.x, hi = units * (blockIdx.x + 1) / gridDim.x;
    const int64_t gw = lo + warp;
    constexpr int64_t nw = NW;
    const int64_t my_units = gw < hi ? (hi - gw + nw - 1) / nw : 0;
    const int64_t chunks = SPLIT ? (blockIdx.x < units ? 1 : 0) : my_units * QN;
    auto issue = [&](int64_t g) {  // lane 0: chunk g of this warp's sequence
        const int st = static_cast<int>(g % NST);
        const int64_t o = SPLIT ? static_cast<int64_t>(blockIdx.x) : gw + (g / QN) * nw;
        const double* src = a.X + kQBlock * o + kQ2Chunk * (SPLIT ? warp : static_cast<int>(g % QN));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(q_smem(&bar[st])),
                     "r"(kQ2Chunk * 8)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                q_smem(ring + st * kQ2Chunk)),
            "l"(src), "r"(kQ2Chunk * 8), "r"(q_smem(&bar[st]))
            : "memory");
    };
    if constexpr (FINISH) {
        // launched as a programmatic dependent of the streaming pass: the
        // bases above were staged while that grid drained; its output (this
        // launch's input) and ||y||^2 partials are complete past this point
        asm volatile("griddepcontrol.wait;" ::: "memory");
    } else {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (lane == 0) {
        for (int k = 0; k < NST; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(q_smem(&bar[k])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < NST && k < chunks; ++k) issue(k);
    }
    __syncthreads();

    const int e2 = lane >> 2, j = lane & 3;
    // rotation of the 16-byte parts read (conflict-free: the 8 lanes of a
    // quarter-warp cover the 8 16-byte slots of a 128-byte window); the lane's
    // copy of U0 is held in registers in the same rotated order
    const int rot = ((j >> 1) | ((e2 & 1) << 1)) & 3;
    double ur[QN / 2][2][QR];  // [step v][e0 parity][q] for part (v + rot) & 3
#pragma unroll
    for (int v = 0; v < QN / 2; ++v) {
        const int part = (v + rot) & 3;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < QR; ++q) ur[v][h][q] = Us[0][(2 * part + h) * QR + q];
    }
    double ysv[QN / 2] = {0.0, 0.0, 0.0, 0.0};  // independent chains
    // modes e3 and the three transfers of a completed block (one warp)
    auto finish_block = [&](int64_t ob) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int jj = lane + 32 * t;
            double acc[QR] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int e3 = 0; e3 < QN; ++e3) {
                const double v = S2[jj + 64 * e3];
#pragma unroll
                for (int q = 0; q < QR; ++q) acc[q] = fma(Us[3][e3 * QR + q], v, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < QR; ++q) S3[jj + 64 * q] = acc[q];
        }
        __syncwarp();
        {
            const int b = lane & 3, m0 = lane >> 2;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int m = m0 + 8 * t;
                double v = 0.0;
#pragma unroll
                for (int k = 0; k < 16; ++k) v = fma(Ts[0][k * QR + b], S3[k + 16 * m], v);
                V01[b + QR * m] = v;
            }
        }
        __syncwarp();
        if (lane < 16) {
            const int b01 = lane & 3, b23 = lane >> 2;
            double v = 0.0;
#pragma unroll
            for (int m = 0; m < 16; ++m) v = fma(Ts[1][m * QR + b23], V01[b01 + QR * m], v);
            V[b01 + QR * b23] = v;
        }
        __syncwarp();
        if (lane < QR) {
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < 16; ++k) v = fma(Ts[2][k * QR + lane], V[k], v);
            a.out[(ob % a.P) + a.P * (lane + QR * (ob / a.P))] = v;
            if constexpr (FINISH) ysv[0] = fma(v, v, ysv[0]);
        }
        __syncwarp();
    };

    // ring slot / phase and the chunk's e3 advance incrementally (no 64-bit
    // division per chunk)
    int st = 0, k3 = SPLIT ? warp : 0;
    uint32_t parity = 0;
    int64_t o = SPLIT ? static_cast<int64_t>(blockIdx.x) : gw;  // block of the current chunk
    for (int64_t g = 0; g < chunks; ++g) {
        asm volatile(
            "{\n\t.reg .pred p;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n}\n" ::"r"(
                q_smem(&bar[st])),
            "r"(parity)
            : "memory");
        const double* ch = ring + st * kQ2Chunk + 64 * e2;
        double p1[QR][QR];
#pragma unroll
        for (int x0 = 0; x0 < QR; ++x0)
#pragma unroll
            for (int x1 = 0; x1 < QR; ++x1) p1[x0][x1] = 0.0;
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const int e1 = j + 4 * f;
            double p0[QR] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int v = 0; v < QN / 2; ++v) {
                const int part = (v + rot) & 3;  // e0 = 2 part, 2 part + 1
                const double2 x2 = *reinterpret_cast<const double2*>(ch + QN * e1 + 2 * part);
#pragma unroll
                for (int q = 0; q < QR; ++q) {
                    p0[q] = fma(ur[v][0][q], x2.x, p0[q]);
                    p0[q] = fma(ur[v][1][q], x2.y, p0[q]);
                }
                if constexpr (!FINISH) {
                    ysv[v] = fma(x2.x, x2.x, ysv[v]);
                    ysv[v] = fma(x2.y, x2.y, ysv[v]);
                }
            }
            const double2 w01 = *reinterpret_cast<const double2*>(&Us[1][e1 * QR]);
            const double2 w23 = *reinterpret_cast<const double2*>(&Us[1][e1 * QR + 2]);
            const double w[QR] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
            for (int x0 = 0; x0 < QR; ++x0)
#pragma unroll
                for (int x1 = 0; x1 < QR; ++x1) p1[x0][x1] = fma(p0[x0], w[x1], p1[x0][x1]);
        }
        // the stage is consumed: refill it (generic-proxy reads before the
        // async-proxy write)
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (g + NST < chunks) issue(g + NST);
        }
        // reduce-scatter P1 over the 4 j-lanes of this e2 (fixed order): lane
        // j ends with the sums of row x0 = j, which is what it stores.
        // Level 1 (partner j ^ 1): keep rows with x0 & 1 == j & 1.
        const bool odd = (j & 1) != 0, up = (j & 2) != 0;
        double h[2][QR];  // rows x0 = (j & 1) and (j & 1) + 2
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int x1 = 0; x1 < QR; ++x1) {
                const double keep = odd ? p1[2 * t + 1][x1] : p1[2 * t][x1];
                const double send = odd ? p1[2 * t][x1] : p1[2 * t + 1][x1];
                h[t][x1] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
            }
        // level 2 (partner j ^ 2): keep row x0 = j
#pragma unroll
        for (int x1 = 0; x1 < QR; ++x1) {
            const double keep = up ? h[1][x1] : h[0][x1];
            const double send = up ? h[0][x1] : h[1][x1];
            S1[(j + QR * x1) + 16 * e2] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        __syncwarp();
        // mode e2 for this e3: S2[k16 + 16 (a2 + 4 e3)] (64 outputs, 2 per lane)
        {
            const int k16 = lane & 15, a2h = lane >> 4;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int a2 = 2 * a2h + t;
                double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                for (int ee = 0; ee < QN; ee += 2) {
                    acc0 = fma(Us[2][ee * QR + a2], S1[k16 + 16 * ee], acc0);
                    acc1 = fma(Us[2][(ee + 1) * QR + a2], S1[k16 + 16 * (ee + 1)], acc1);
                }
                S2[k16 + 16 * (a2 + QR * k3)] = acc0 + acc1;
            }
        }
        __syncwarp();
        if constexpr (SPLIT) continue;  // the block is finished after the loop
        const bool block_done = k3 == QN - 1;
        if (++st == NST) {
            st = 0;
            parity ^= 1u;
        }
        if (!block_done) {
            ++k3;
            continue;
        }
        k3 = 0;
        finish_block(o);
        o += nw;
    }
    if constexpr (SPLIT) {
        __syncthreads();  // every warp's e3 slice of S2 is in place
        if (warp == 0 && blockIdx.x < units) finish_block(static_cast<int64_t>(blockIdx.x));
    }
    // FINISH: the partials are of ||out||^2 (ysv[0] of lanes 0-3)
    double ys = (ysv[0] + ysv[1]) + (ysv[2] + ysv[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ys += __shfl_xor_sync(0xffffffffu, ys, off);
    if (lane == 0) red[warp] = ys;
    __syncthreads();
    __shared__ bool last;
    if (tid == 0) {
        double sum = 0.0;
        for (int w = 0; w < NW; ++w) sum += red[w];
        a.partials[blockIdx.x] = sum;
        if constexpr (FINISH) {
            __threadfence();
            last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
        }
    }
    if constexpr (FINISH) {
        __syncthreads();
        if (!last) return;
        __threadfence();
        // last CTA: ||y||^2 from the first launch's partials and ||latent||^2
        // from this launch's: loads in parallel, a fixed reduction tree
        // (lane-strided sums, shuffle tree, warps in order)
        double y2 = 0.0, l2 = 0.0;
        for (int64_t k = tid; k < a.n_ysq; k += (NW * 32)) y2 += __ldcg(a.ysq_partials + k);
        for (unsigned k = tid; k < gridDim.x; k += (NW * 32)) l2 += __ldcg(a.partials + k);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            y2 += __shfl_xor_sync(0xffffffffu, y2, off);
            l2 += __shfl_xor_sync(0xffffffffu, l2, off);
        }
        __shared__ double red2[2][NW];
        if (lane == 0) {
            red2[0][warp] = y2;
            red2[1][warp] = l2;
        }
        __syncthreads();
        if (tid == 0) {
            y2 = 0.0;
            l2 = 0.0;
            for (int w = 0; w < NW; ++w) {
                y2 += red2[0][w];
                l2 += red2[1][w];
            }
            a.sc[0] = y2;
            a.sc[2] = l2;
            if (a.host_out) {
                a.host_out[0] = y2;
                a.host_out[2] = l2;
            }
            *a.ticket = 0u;
        }
    }
}

}  // namespace

bool quad_supported(int64_t extent, int64_t rank) { return extent == QN && rank == QR; }

int launch_quad(const QuadArgs& a, bool finish, int num_sms, cudaStream_t s, int64_t* launches) {
    if ((reinterpret_cast<uintptr_t>(a.X) & 15u) != 0) return -1;  // TMA bulk copies need 16-byte alignment
    // few blocks (the finishing launch): one CTA per block, a chunk per warp
    const bool split = finish && a.O <= num_sms;
    const int grid = split ? static_cast<int>(a.O)
                           : static_cast<int>(std::max<int64_t>(
                                 1, std::min<int64_t>(num_sms, (a.O + kQ2Warps - 1) / kQ2Warps)));
    if (!finish) {
        // the streaming pass over y: 12 warps with two-stage rings (more
        // warps in flight per SM to cover the per-chunk dependency chains)
        constexpr int NW = kQ1Warps, NST = kQ1Stages;
        const int grid1 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms, (a.O + NW - 1) / NW)));
        const size_t smem = sizeof(double) * NW * (NST * kQ2Chunk + kQ2Scratch);
        auto kfn = quad_stream_kernel<false, false, NW, NST>;
        ensure_smem_limit(reinterpret_cast<const void*>(kfn), smem);
        kfn<<<grid1, NW * 32, smem, s>>>(a);
        ++*launches;
        return grid1;
    }
    const size_t smem = sizeof(double) * kQ2Warps * (kQ2Stages * kQ2Chunk + kQ2Scratch);
    auto kfn = split ? quad_stream_kernel<true, true, kQ2Warps, kQ2Stages>
                     : quad_stream_kernel<true, false, kQ2Warps, kQ2Stages>;
    ensure_smem_limit(reinterpret_cast<const void*>(kfn), smem);
    // programmatic dependent launch after the streaming pass (griddepcontrol.wait in the kernel)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kQ2Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kfn, a);
    ++*launches;
    return grid;
}

}  // namespace htr
