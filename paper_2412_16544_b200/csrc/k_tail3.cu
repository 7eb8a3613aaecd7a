// Skip-path tail for 3-way trees (1,(2,3)): one CTA per sample s computes
//
//   Z_s[a0, a1, a2]  = sum_i2 W[(s,i2), a0 + r0 a1] U2[i2, a2]      (slab-axis contraction)
//   latent_s[a0, b]  = sum_{a1,a2} Z_s[a0, a1, a2] B[a1 + r1 a2, b]  (transfer projection,
//                                                                     bht.hpp:385-399)
//   ||latent_s||^2
//
// on the FP64 tensor cores, with Z_s kept in shared memory between the two
// contractions. W is the per-slab output of fused3_kernel, B the transfer
// node's basis matrix (r1 r2 x rt), streamed from L2.
//
// Work split (every DMMA issued is a useful tile; no predicated padding):
//   phase A  M = r0 r1 (m-tiles dealt round-robin to warps, processed in
//            groups of 4/2/1 sharing the W fragments), N = r2 (NT <= 3
//            tiles, compile time), K = n2, operands prefetched two k-steps
//            ahead;
//   phase B  M = r0 (MT <= 3 tiles, compile time), N = rt in pairs of
//            n-tiles per warp (each Z fragment feeds two DMMAs), whole pairs
//            in full rounds over the warps and the remainder split over
//            K = r1 r2 so all warps carry equal work; B fragments loaded in
//            chunks of 8 k-steps one chunk ahead (L2 latency); partial tiles
//            summed in a fixed order through shared memory (deterministic).
// The last CTA to finish (ticket counter) also reduces ||y||^2 (fused3's
// per-CTA partials) and ||latent||^2 in a fixed order. Replaces two generic
// GEMM launches, the latent norm pass and two scalar reductions.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace htr {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kU2Pitch = 28;  // doubles: conflict-free B-fragment reads (<= 24 columns)
constexpr int kChunk = 8;     // phase-B k-steps per prefetch chunk
constexpr int kRedDoubles = kWarps * 3 * 2 * 64;  // phase-B partial tiles (K split)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

// Z tiles for G m-tiles (mt0, mt0 + stride, ...) x NT n-tiles, stored into
// this CTA's Zs and (cluster split) into every peer CTA's copy.
template <int G, int NT, bool CL>
__device__ __forceinline__ void phase_a_group(const double* __restrict__ W, const double* U2s, double* Zs,
                                              int R01, int r2, int n2, int mt0, int stride_rt, int g4, int t4,
                                              int csize) {
    const int stride = CL ? stride_rt : kWarps;
    double acc[G][NT][2];
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    auto load = [&](int k, double (&av)[G]) {
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const int p = 8 * (mt0 + stride * i) + g4;
            av[i] = (p < R01 && k < n2) ? __ldg(W + static_cast<int64_t>(k) * R01 + p) : 0.0;
        }
    };
    double cur[G], nxt[G];
    load(t4, cur);
    load(t4 + 4, nxt);
    for (int k0 = 0; k0 < n2; k0 += 4) {
        double fut[G];
        load(k0 + 8 + t4, fut);
        const int k = k0 + t4;
        double b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = (k < n2) ? U2s[k * kU2Pitch + 8 * j + g4] : 0.0;
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
    cg::cluster_group cluster = cg::this_cluster();
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int p = 8 * (mt0 + stride * i) + g4;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a2 = 8 * j + 2 * t4 + h;
                if (p < R01 && a2 < r2) {
                    const int idx = p + R01 * a2;
                    Zs[idx] = acc[i][j][h];
                    if constexpr (CL) {
                        for (int q = 1; q < csize; ++q) {  // distributed shared memory of the peers
                            const unsigned peer = (cluster.block_rank() + q) % csize;
                            cluster.map_shared_rank(Zs, peer)[idx] = acc[i][j][h];
                        }
                    }
                }
            }
    }
}

template <int NT, int MT, bool CL>
__global__ void __launch_bounds__(kThreads, 2) tail3_kernel(const Tail3Args a) {
    extern __shared__ __align__(16) double sm[];
    const int r0 = a.r0, r1 = a.r1, r2 = a.r2, rt = a.rt;
    const int R01 = r0 * r1, R12 = r1 * r2;
    const int n2 = static_cast<int>(a.n2);
    double* U2s = sm;  // [n2][kU2Pitch], later the phase-B reduction buffer
    double* Zs = U2s + max(n2 * kU2Pitch, kRedDoubles);  // [a0 + r0 (a1 + r1 a2)]
    __shared__ double red[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    // cluster split (small batches): the csize CTAs of a cluster share one
    // sample; each computes 1/csize of Z (all-gathered into every CTA's
    // shared memory) and 1/csize of the latent's column pairs
    const int C = CL ? a.csize : 1;
    const int crank = CL ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
    const int64_t s = blockIdx.x / C;

    for (int e = tid; e < n2 * kU2Pitch; e += kThreads) {
        const int i2 = e / kU2Pitch, c = e - i2 * kU2Pitch;
        U2s[e] = c < r2 ? a.U2[i2 + static_cast<int64_t>(n2) * c] : 0.0;
    }
    __syncthreads();
    // launched as a programmatic dependent of the fused leaf kernel: its W
    // and ||y||^2 partials are complete and visible after this (a no-op for a
    // plain launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- phase A: Z_s(p, a2), M = R01 (p), N = r2, K = n2 ----
    {
        const double* W = a.wslab + s * n2 * static_cast<int64_t>(R01);
        const int mtA = (R01 + 7) / 8;
        const int gw = crank * kWarps + warp, stride = C * kWarps;
        const int cnt = gw < mtA ? (mtA - gw + stride - 1) / stride : 0;
        int t = 0;
        for (; cnt - t >= 4; t += 4)
            phase_a_group<4, NT, CL>(W, U2s, Zs, R01, r2, n2, gw + stride * t, stride, g4, t4, C);
        if (cnt - t >= 2) {
            phase_a_group<2, NT, CL>(W, U2s, Zs, R01, r2, n2, gw + stride * t, stride, g4, t4, C);
            t += 2;
        }
        if (cnt - t >= 1) phase_a_group<1, NT, CL>(W, U2s, Zs, R01, r2, n2, gw + stride * t, stride, g4, t4, C);
    }
    if constexpr (CL)
        cg::this_cluster().sync();  // every CTA's Z complete (no DSMEM access after this)
    else
        __syncthreads();

    // ---- phase B: latent_s(a0, b) = Z_s(a0, j) B(j, b), M = r0, N = rt, K = R12 ----
    // work item = a pair of n-tiles over a K range: per k-step 3 Z and 2 B
    // fragment loads feed 2 MT DMMAs. Whole pairs are dealt to the warps in
    // full rounds; the remaining npairs % kWarps pairs are split over K so
    // every warp gets the same share, and their partial tiles are summed in
    // a fixed order through shared memory (deterministic).
    const int ntB = (rt + 7) / 8;
    const int npairs_all = (ntB + 1) / 2;
    // this CTA's contiguous range of column pairs [pb0, pb0 + npairs)
    const int pb0 = static_cast<int>(static_cast<int64_t>(npairs_all) * crank / C);
    // an identity transfer basis (a full-rank node: rt = r1 r2, B = I) makes
    // the latent Z_s itself, in the same layout: no pairs to project
    const int npairs = a.identity_transfer
                           ? 0
                           : static_cast<int>(static_cast<int64_t>(npairs_all) * (crank + 1) / C) - pb0;
    const int full = npairs / kWarps * kWarps;
    const int rem = npairs - full;
    const int kparts = rem ? kWarps / rem : 1;
    const int KS = (R12 + 3) / 4;
    const int sp = (KS + kparts - 1) / kparts;
    double* out = a.latent + s * static_cast<int64_t>(r0) * rt;
    double* redbuf = U2s;
    double lsq = 0.0;
    if (a.identity_transfer) {
        // latent[a0 + r0 b] = Z_s[a0 + r0 (a1 + r1 a2)]: this CTA's share of the copy
        const int total = r0 * rt;
        const int c0 = static_cast<int>(static_cast<int64_t>(total) * crank / C);
        const int c1 = static_cast<int>(static_cast<int64_t>(total) * (crank + 1) / C);
        for (int e = c0 + tid; e < c1; e += kThreads) {
            const double v = Zs[e];
            out[e] = v;
            lsq = fma(v, v, lsq);
        }
    }
    auto pair_tiles = [&](int pr, int ks0, int ks1, double (&acc)[MT][2][2]) {
        pr += pb0;
        const int kend = min(R12, 4 * ks1);
        const double* Bc[2];
        bool colok[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int bcol = 8 * (2 * pr + j) + g4;
            colok[j] = bcol < rt;
            Bc[j] = a.B + static_cast<int64_t>(R12) * (colok[j] ? bcol : 0);
        }
        auto load = [&](int ks, double (&bv)[kChunk][2]) {
#pragma unroll
            for (int c = 0; c < kChunk; ++c) {
                const int k = 4 * (ks + c) + t4;
#pragma unroll
                for (int j = 0; j < 2; ++j) bv[c][j] = (colok[j] && k < kend) ? __ldg(Bc[j] + k) : 0.0;
            }
        };
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        double bc[kChunk][2];
        load(ks0, bc);
        bool rowok[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) rowok[i] = 8 * i + g4 < r0;
        for (int ks = ks0; ks < ks1; ks += kChunk) {
            double bn[kChunk][2];
            load(ks + kChunk, bn);
            if (ks + kChunk <= ks1 && 4 * (ks + kChunk) <= R12) {
                // whole chunk in range: no per-step branch, so the Z loads of
                // later steps can be issued ahead of earlier steps' MMAs
#pragma unroll
                for (int c = 0; c < kChunk; ++c) {
                    const int k = 4 * (ks + c) + t4;
                    double av[MT];
#pragma unroll
                    for (int i = 0; i < MT; ++i) av[i] = rowok[i] ? Zs[8 * i + g4 + r0 * k] : 0.0;
#pragma unroll
                    for (int i = 0; i < MT; ++i)
#pragma unroll
                        for (int j = 0; j < 2; ++j) dmma(acc[i][j], av[i], bc[c][j]);
                }
            } else {
#pragma unroll
                for (int c = 0; c < kChunk; ++c) {
                    if (ks + c < ks1) {  // warp-uniform
                        const int k = 4 * (ks + c) + t4;
                        double av[MT];
#pragma unroll
                        for (int i = 0; i < MT; ++i) av[i] = (rowok[i] && k < R12) ? Zs[8 * i + g4 + r0 * k] : 0.0;
#pragma unroll
                        for (int i = 0; i < MT; ++i)
#pragma unroll
                            for (int j = 0; j < 2; ++j) dmma(acc[i][j], av[i], bc[c][j]);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < kChunk; ++c) {
                bc[c][0] = bn[c][0];
                bc[c][1] = bn[c][1];
            }
        }
    };
    for (int pr = warp; pr < full; pr += kWarps) {
        double acc[MT][2][2];
        pair_tiles(pr, 0, KS, acc);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int a0 = 8 * i + g4, b = 8 * (2 * (pb0 + pr) + j) + 2 * t4 + h;
                    if (a0 < r0 && b < rt) {
                        const double v = acc[i][j][h];
                        out[a0 + static_cast<int64_t>(r0) * b] = v;
                        lsq = fma(v, v, lsq);
                    }
                }
    }
    if (rem) {
        if (warp < rem * kparts) {
            const int pr = full + warp % rem, q = warp / rem;
            double acc[MT][2][2];
            pair_tiles(pr, q * sp, min(KS, (q + 1) * sp), acc);
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    double* dst = redbuf + (((q * rem + warp % rem) * MT + i) * 2 + j) * 64 + 2 * lane;
                    dst[0] = acc[i][j][0];
                    dst[1] = acc[i][j][1];
                }
        }
        __syncthreads();
        const int per_part = rem * MT * 2 * 64;
        for (int e = tid; e < per_part; e += kThreads) {
            const int tile = e / 64, ln = (e & 63) >> 1, h = e & 1;
            const int j = tile % 2, i = (tile / 2) % MT, pr = pb0 + full + tile / (2 * MT);
            const int a0 = 8 * i + (ln >> 2), b = 8 * (2 * pr + j) + 2 * (ln & 3) + h;
            if (a0 >= r0 || b >= rt) continue;
            double v = 0.0;
            for (int q = 0; q < kparts; ++q) v += redbuf[q * per_part + e];
            out[a0 + static_cast<int64_t>(r0) * b] = v;
            lsq = fma(v, v, lsq);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsq += __shfl_xor_sync(0xffffffffu, lsq, o);
    if (lane == 0) red[warp] = lsq;
    __syncthreads();
    __shared__ bool last;
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        a.latsq[s * C + crank] = t;
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
    for (int64_t i = tid; i < a.S * C; i += kThreads) ls += __ldcg(a.latsq + i);
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

// ---- identity transfer basis: the latent is Z itself -----------------------
// A full-rank transfer node carries the identity basis (BHT-l2r's Cholesky
// certificate; config 5: rt = r1 r2 = 400), so the tail is phase A alone and
// Z_s needs no shared-memory staging. Work units (sample, 16 rows p of Z_s =
// two m-tiles) are dealt round-robin to every warp of a grid two CTAs per SM
// deep. W arrives by TMA: a [R01, n2, S] tensor map, 16 x 16 boxes (128-byte
// rows, 128-byte swizzle) into the warp's own four-stage ring, one lane
// issuing the copies and an mbarrier per stage, so a warp keeps 8 KB of W in
// flight without holding the loads in registers (register prefetch is capped
// by the six scoreboards of a warp: a variant with sixteen loads per lane in
// flight measured 69 us). Per stage 4 k-steps x 2 x NT DMMAs; the tiles are
// stored straight into the latent; per-CTA ||latent||^2 partials, the final
// reductions by the last CTA. c5: 42.7 us against 53.7 us for the
// one-CTA-per-sample kernel. (Writing W in 16-row blocks from fused3 so that a
// unit is one contiguous range was measured too: the scattered 128-byte
// writes cost fused3 5 % and the tail gained nothing.)
constexpr int kIdStages = 4;
constexpr int kIdBox = 16;                    // rows p and steps k per box
constexpr int kIdStageDoubles = kIdBox * kIdBox;

__device__ __forceinline__ uint32_t id_saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// element (k, p) of a swizzled 16 x 16 box (rows k of 128 bytes)
__device__ __forceinline__ int id_swz(int k, int p) { return k * kIdBox + ((((p >> 1) ^ (k & 7))) << 1) + (p & 1); }

template <int NT>
__global__ void __launch_bounds__(kThreads, 2)
    tail3_identity_kernel(const Tail3Args a, const __grid_constant__ CUtensorMap wmap) {
    extern __shared__ __align__(1024) unsigned char idsm_raw[];
    const int r0 = a.r0, r1 = a.r1, r2 = a.r2;
    const int R01 = r0 * r1;
    const int n2 = static_cast<int>(a.n2);
    const int spu = (n2 + kIdBox - 1) / kIdBox;  // stages per unit
    const int n2p = spu * kIdBox;
    // rings first (1024-byte aligned for the swizzle), then U2 (zero rows beyond n2)
    const uint32_t pad = (1024u - (id_saddr(idsm_raw) & 1023u)) & 1023u;
    double* rings = reinterpret_cast<double*>(idsm_raw + pad);  // [warp][stage][16][16]
    double* U2s = rings + kWarps * kIdStages * kIdStageDoubles;  // [n2p][kU2Pitch]
    __shared__ __align__(8) uint64_t full[kWarps][kIdStages];
    __shared__ double red[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;

    const int mtA = (R01 + 7) / 8;
    const int upg = (mtA + 1) / 2;  // units (pairs of m-tiles) per sample
    const int64_t units = a.S * upg;
    const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + warp, nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int64_t my_units = gw < units ? (units - gw + nw - 1) / nw : 0;
    const int64_t total = my_units * spu;  // stages this warp consumes
    double* ring = rings + warp * kIdStages * kIdStageDoubles;
    uint64_t* bar = full[warp];
    auto issue = [&](int64_t i) {  // lane 0: stage i of this warp's sequence
        const int st = static_cast<int>(i % kIdStages);
        const int64_t u = gw + (i / spu) * nw;
        const int kc = static_cast<int>(i % spu);
        const int64_t s = u / upg;
        const int p0 = static_cast<int>(u - s * upg) * kIdBox;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(id_saddr(&bar[st])),
                     "r"(static_cast<uint32_t>(kIdStageDoubles * sizeof(double)))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(id_saddr(ring + st * kIdStageDoubles)),
            "l"(reinterpret_cast<uint64_t>(&wmap)), "r"(p0), "r"(kc * kIdBox), "r"(static_cast<int>(s)),
            "r"(id_saddr(&bar[st]))
            : "memory");
    };
    if (lane == 0) {
        for (int k = 0; k < kIdStages; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(id_saddr(&bar[k])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = tid; e < n2p * kU2Pitch; e += kThreads) {
        const int i2 = e / kU2Pitch, c = e - i2 * kU2Pitch;
        U2s[e] = (c < r2 && i2 < n2) ? a.U2[i2 + static_cast<int64_t>(n2) * c] : 0.0;
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // fused3's W and ||y||^2 partials are complete
    if (lane == 0)
        for (int64_t i = 0; i < kIdStages && i < total; ++i) issue(i);

    double lsq = 0.0;
    int64_t i = 0;
    for (int64_t uu = 0; uu < my_units; ++uu) {
        const int64_t u = gw + uu * nw;
        const int64_t s = u / upg;
        const int mt0 = static_cast<int>(u - s * upg) * 2;
        double acc[2][NT][2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[x][j][0] = acc[x][j][1] = 0.0;
        for (int kc = 0; kc < spu; ++kc, ++i) {
            const int st = static_cast<int>(i % kIdStages);
            const uint32_t parity = static_cast<uint32_t>((i / kIdStages) & 1);
            asm volatile(
                "{\n\t.reg .pred p;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n}\n" ::"r"(
                    id_saddr(&bar[st])),
                "r"(parity)
                : "memory");
            const double* box = ring + st * kIdStageDoubles;
#pragma unroll
            for (int ks = 0; ks < kIdBox / 4; ++ks) {
                const int kk = 4 * ks + t4;
                const double a0 = box[id_swz(kk, g4)], a1 = box[id_swz(kk, 8 + g4)];
                const double* u2 = U2s + (kc * kIdBox + kk) * kU2Pitch + g4;
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const double b = u2[8 * j];
                    dmma(acc[0][j], a0, b);
                    dmma(acc[1][j], a1, b);
                }
            }
            // the stage is consumed: refill it (generic-proxy reads before the async-proxy write)
            __syncwarp();
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (i + kIdStages < total) issue(i + kIdStages);
            }
        }
        double* out = a.latent + s * static_cast<int64_t>(R01) * r2;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            const int p = 8 * (mt0 + x) + g4;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int a2 = 8 * j + 2 * t4 + h;
                    if (p < R01 && a2 < r2) {
                        const double v = acc[x][j][h];
                        out[p + static_cast<int64_t>(R01) * a2] = v;
                        lsq = fma(v, v, lsq);
                    }
                }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsq += __shfl_xor_sync(0xffffffffu, lsq, o);
    if (lane == 0) red[warp] = lsq;
    __syncthreads();
    __shared__ bool last;
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        a.latsq[blockIdx.x] = t;
        __threadfence();
        last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double ys = 0.0, ls = 0.0;
    for (int64_t k = tid; k < a.n_ysq; k += kThreads) ys += __ldcg(a.ysq_partials + k);
    for (int64_t k = tid; k < gridDim.x; k += kThreads) ls += __ldcg(a.latsq + k);
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

PFN_cuTensorMapEncodeTiled_v12000 id_encoder() {
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

int tail3_identity_grid(const Tail3Args& a) {
    const int64_t mtA = (static_cast<int64_t>(a.r0) * a.r1 + 7) / 8;
    const int64_t units = a.S * ((mtA + 1) / 2);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(2 * a.num_sms, (units + kWarps - 1) / kWarps)));
}

size_t tail3_identity_smem(int64_t n2) {
    const int64_t n2p = (n2 + kIdBox - 1) / kIdBox * kIdBox;
    return sizeof(double) * static_cast<size_t>(kWarps * kIdStages * kIdStageDoubles + n2p * kU2Pitch) + 1024;
}

/// Launches the identity-transfer tail; false (nothing launched) when the
/// operands do not fit it (odd r0 r1, unaligned W, no tensor-map encoder).
bool launch_identity(const Tail3Args& a, cudaStream_t s) {
    const int64_t R01 = static_cast<int64_t>(a.r0) * a.r1;
    auto enc = id_encoder();
    if (!enc || (R01 & 1) || (reinterpret_cast<uintptr_t>(a.wslab) & 15u) || a.n2 > 4096 || a.S >= (int64_t{1} << 31))
        return false;
    const size_t smem = tail3_identity_smem(a.n2);
    if (smem > 100 * 1024) return false;  // two CTAs per SM
    alignas(64) CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(R01), static_cast<cuuint64_t>(a.n2), static_cast<cuuint64_t>(a.S)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(R01 * 8), static_cast<cuuint64_t>(R01 * a.n2 * 8)};
    cuuint32_t box[3] = {kIdBox, kIdBox, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(a.wslab), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(tail3_identity_grid(a)));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto run = [&](auto kfn) {
        if (smem > 46 * 1024) ensure_smem_limit(reinterpret_cast<const void*>(kfn), smem);
        cudaLaunchKernelEx(&cfg, kfn, a, map);
    };
    switch ((a.r2 + 7) / 8) {
        case 1: run(tail3_identity_kernel<1>); break;
        case 2: run(tail3_identity_kernel<2>); break;
        default: run(tail3_identity_kernel<3>); break;
    }
    return true;
}

// ---- sample-pair variant --------------------------------------------------
// One CTA per pair of samples (s0, s0 + 1), 10 warps:
//   phase A  Z_s = W_s U2 for both samples (as above), written transposed
//            into one shared-memory operand Z^T[j, n] with n = a0 + r0 * (s - s0);
//   phase B  latent^T[b, n] = sum_j B[j, b] Z^T[j, n]: M = rt (transfer basis
//            columns, streamed from L2 as the A operand), N = 2 r0 (c5: 40 = 5
//            whole n-tiles, so no MMA row is padding), K = r1 r2; each warp
//            owns groups of 5 m-tiles x all n-tiles (25 DMMAs per k-step on 5 A
//            and 5 B fragment loads), A prefetched two k-steps ahead.
// c5 per pair: phase A 2 x 4800 + phase B 25000 DMMAs (vs 2 x 19800 one
// sample per CTA, whose M = r0 = 20 pads to 24), in 128 CTAs.
constexpr int kPairWarps = 10;
constexpr int kPairThreads = kPairWarps * 32;
constexpr int kGroup = 5;  // phase-B m-tiles per warp work item

__host__ __device__ __forceinline__ int pair_pitch(int nb) { return (nb % 16 == 8) ? nb : nb + 8; }

// Z^T tiles of one sample for G m-tiles (mt0, mt0 + kPairWarps, ...) x NT n-tiles
template <int G, int NT>
__device__ __forceinline__ void phase_a_pair(const double* __restrict__ W, const double* U2s, double* Zt, int pitch,
                                             int r0, int r1, int r2, int n2, int sl, int mt0, int g4, int t4) {
    const int R01 = r0 * r1;
    double acc[G][NT][2];
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    auto load = [&](int k, double (&av)[G]) {
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const int p = 8 * (mt0 + kPairWarps * i) + g4;
            av[i] = (p < R01 && k < n2) ? __ldg(W + static_cast<int64_t>(k) * R01 + p) : 0.0;
        }
    };
    double cur[G], nxt[G];
    load(t4, cur);
    load(t4 + 4, nxt);
    for (int k0 = 0; k0 < n2; k0 += 4) {
        double fut[G];
        load(k0 + 8 + t4, fut);
        const int k = k0 + t4;
        double b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = (k < n2) ? U2s[k * kU2Pitch + 8 * j + g4] : 0.0;
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
        const int p = 8 * (mt0 + kPairWarps * i) + g4;
        const int a0 = p % r0, a1 = p / r0;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a2 = 8 * j + 2 * t4 + h;
                if (p < R01 && a2 < r2) Zt[(a0 + r0 * sl) + pitch * (a1 + r1 * a2)] = acc[i][j][h];
            }
    }
}

template <int NT, int NTB>
__global__ void __launch_bounds__(kPairThreads) tail3_pair_kernel(const Tail3Args a) {
    extern __shared__ __align__(16) double sm[];
    constexpr int NB = 8 * NTB;
    const int r0 = a.r0, r1 = a.r1, r2 = a.r2, rt = a.rt;
    const int R01 = r0 * r1, R12 = r1 * r2;
    const int n2 = static_cast<int>(a.n2);
    const int pitch = pair_pitch(NB);
    const int KS = (R12 + 3) / 4;
    double* U2s = sm;                   // [n2][kU2Pitch]
    double* Zt = U2s + n2 * kU2Pitch;   // [4 KS][pitch]
    __shared__ double red[kPairWarps][2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int64_t s0 = 2 * static_cast<int64_t>(blockIdx.x);
    const int ns = static_cast<int>(min(static_cast<int64_t>(2), a.S - s0));

    for (int e = tid; e < n2 * kU2Pitch; e += kPairThreads) {
        const int i2 = e / kU2Pitch, c = e - i2 * kU2Pitch;
        U2s[e] = c < r2 ? a.U2[i2 + static_cast<int64_t>(n2) * c] : 0.0;
    }
    for (int e = tid; e < 4 * KS * pitch; e += kPairThreads) Zt[e] = 0.0;
    __syncthreads();

    // ---- phase A: both samples' Z into Z^T ----
    const int mtA = (R01 + 7) / 8;
    const int cnt = warp < mtA ? (mtA - warp + kPairWarps - 1) / kPairWarps : 0;
    for (int sl = 0; sl < ns; ++sl) {
        const double* W = a.wslab + (s0 + sl) * n2 * static_cast<int64_t>(R01);
        int t = 0;
        for (; cnt - t >= 4; t += 4)
            phase_a_pair<4, NT>(W, U2s, Zt, pitch, r0, r1, r2, n2, sl, warp + kPairWarps * t, g4, t4);
        if (cnt - t >= 2) {
            phase_a_pair<2, NT>(W, U2s, Zt, pitch, r0, r1, r2, n2, sl, warp + kPairWarps * t, g4, t4);
            t += 2;
        }
        if (cnt - t >= 1) phase_a_pair<1, NT>(W, U2s, Zt, pitch, r0, r1, r2, n2, sl, warp + kPairWarps * t, g4, t4);
    }
    __syncthreads();

    // ---- phase B: latent^T = B^T Z^T ----
    const int MTB = (rt + 7) / 8;
    const int ngroups = (MTB + kGroup - 1) / kGroup;
    double lsq[2] = {0.0, 0.0};
    for (int g = warp; g < ngroups; g += kPairWarps) {
        const int mt0 = g * kGroup;
        double acc[kGroup][NTB][2];
#pragma unroll
        for (int i = 0; i < kGroup; ++i)
#pragma unroll
            for (int j = 0; j < NTB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const double* Bc[kGroup];
        bool ok[kGroup];
#pragma unroll
        for (int i = 0; i < kGroup; ++i) {
            const int bcol = 8 * (mt0 + i) + g4;
            ok[i] = bcol < rt;
            Bc[i] = a.B + static_cast<int64_t>(R12) * (ok[i] ? bcol : 0);
        }
        auto loadA = [&](int ks, double (&v)[kGroup]) {
            const int k = 4 * ks + t4;
#pragma unroll
            for (int i = 0; i < kGroup; ++i) v[i] = (ok[i] && k < R12) ? __ldg(Bc[i] + k) : 0.0;
        };
        double cur[kGroup];
        loadA(0, cur);
        for (int ks = 0; ks < KS; ++ks) {
            double nxt[kGroup];
            loadA(ks + 1, nxt);
            const double* zr = Zt + pitch * (4 * ks + t4) + g4;
            double bv[NTB];
#pragma unroll
            for (int j = 0; j < NTB; ++j) bv[j] = zr[8 * j];
#pragma unroll
            for (int i = 0; i < kGroup; ++i)
#pragma unroll
                for (int j = 0; j < NTB; ++j) dmma(acc[i][j], cur[i], bv[j]);
#pragma unroll
            for (int i = 0; i < kGroup; ++i) cur[i] = nxt[i];
        }
#pragma unroll
        for (int i = 0; i < kGroup; ++i)
#pragma unroll
            for (int j = 0; j < NTB; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int b = 8 * (mt0 + i) + g4, n = 8 * j + 2 * t4 + h;
                    const int sl = n >= r0 ? 1 : 0, a0 = n - r0 * sl;
                    if (b < rt && n < r0 * ns) {
                        const double v = acc[i][j][h];
                        a.latent[a0 + static_cast<int64_t>(r0) * b + static_cast<int64_t>(r0) * rt * (s0 + sl)] = v;
                        if (sl) lsq[1] = fma(v, v, lsq[1]);
                        else lsq[0] = fma(v, v, lsq[0]);
                    }
                }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lsq[q] += __shfl_xor_sync(0xffffffffu, lsq[q], o);
    if (lane == 0) {
        red[warp][0] = lsq[0];
        red[warp][1] = lsq[1];
    }
    __syncthreads();
    __shared__ bool last;
    if (tid == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < kPairWarps; ++w) {
            t0 += red[w][0];
            t1 += red[w][1];
        }
        a.latsq[s0] = t0;
        if (ns == 2) a.latsq[s0 + 1] = t1;
        __threadfence();
        last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double ys = 0.0, ls = 0.0;
    for (int64_t i = tid; i < a.n_ysq; i += kPairThreads) ys += __ldcg(a.ysq_partials + i);
    for (int64_t i = tid; i < a.S; i += kPairThreads) ls += __ldcg(a.latsq + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ys += __shfl_xor_sync(0xffffffffu, ys, o);
        ls += __shfl_xor_sync(0xffffffffu, ls, o);
    }
    __shared__ double red2[2][kPairWarps];
    if (lane == 0) {
        red2[0][warp] = ys;
        red2[1][warp] = ls;
    }
    __syncthreads();
    if (tid == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < kPairWarps; ++w) {
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

size_t tail3_pair_smem(int64_t n2, int r0, int r1, int r2) {
    const int nb = 8 * ((2 * r0 + 7) / 8);
    const int64_t ks = (static_cast<int64_t>(r1) * r2 + 3) / 4;
    return sizeof(double) * (static_cast<size_t>(n2) * kU2Pitch + static_cast<size_t>(4 * ks * pair_pitch(nb)));
}

template <int NT, int NTB>
void launch_pair_t(const Tail3Args& a, size_t smem, cudaStream_t s) {
    if (smem > 46 * 1024) ensure_smem_limit(reinterpret_cast<const void*>(tail3_pair_kernel<NT, NTB>), smem);
    tail3_pair_kernel<NT, NTB><<<static_cast<unsigned>((a.S + 1) / 2), kPairThreads, smem, s>>>(a);
}

template <int NT>
void launch_pair_nt(const Tail3Args& a, size_t smem, cudaStream_t s) {
    switch ((2 * a.r0 + 7) / 8) {
        case 1: return launch_pair_t<NT, 1>(a, smem, s);
        case 2: return launch_pair_t<NT, 2>(a, smem, s);
        case 3: return launch_pair_t<NT, 3>(a, smem, s);
        case 4: return launch_pair_t<NT, 4>(a, smem, s);
        case 5: return launch_pair_t<NT, 5>(a, smem, s);
        default: return launch_pair_t<NT, 6>(a, smem, s);
    }
}

size_t tail3_smem(int64_t n2, int r0, int r1, int r2) {
    return sizeof(double) * (std::max<size_t>(static_cast<size_t>(n2) * kU2Pitch, kRedDoubles) +
                             static_cast<size_t>(r0) * r1 * r2);
}

template <int NT, int MT>
void launch_t(const Tail3Args& a, size_t smem, cudaStream_t s) {
    const int cl = a.csize > 1 ? 1 : 0;
    if (smem > 46 * 1024)  // margin for the static arrays
        ensure_smem_limit(cl ? reinterpret_cast<const void*>(tail3_kernel<NT, MT, true>)
                             : reinterpret_cast<const void*>(tail3_kernel<NT, MT, false>),
                          smem);
    // programmatic dependent launch after the fused leaf kernel (see
    // griddepcontrol.wait in the kernel)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(a.S * a.csize));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(a.csize);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cl ? 2 : 1;
    if (cl)
        cudaLaunchKernelEx(&cfg, tail3_kernel<NT, MT, true>, a);
    else
        cudaLaunchKernelEx(&cfg, tail3_kernel<NT, MT, false>, a);
}

template <int NT>
void launch_nt(const Tail3Args& a, size_t smem, cudaStream_t s) {
    switch ((a.r0 + 7) / 8) {
        case 1: return launch_t<NT, 1>(a, smem, s);
        case 2: return launch_t<NT, 2>(a, smem, s);
        default: return launch_t<NT, 3>(a, smem, s);
    }
}

}  // namespace

int64_t tail3_latsq_entries(int64_t S, int num_sms) { return std::max<int64_t>(8 * S, 2 * static_cast<int64_t>(num_sms)); }

bool tail3_supported(int r0, int r1, int r2, int rt, int64_t n2) {
    if (r0 < 1 || r1 < 1 || r2 < 1 || rt < 1 || r0 > 24 || r2 > 24) return false;
    return tail3_smem(n2, r0, r1, r2) <= 200 * 1024;
}

void launch_tail3(const Tail3Args& a, cudaStream_t s, int64_t* launches) {
    // identity transfer basis: the unit-dealt TMA kernel at every batch size
    // (HTR_OPT_TAIL_KERNEL = 1 keeps the one-CTA-per-sample kernel); measured
    // on c5 shards of 128 / 64 / 32 samples against the cluster-split kernel:
    // 0.527 / 0.293 / 0.164 ms per step vs 0.534 / 0.298 / 0.173
    if (a.identity_transfer && a.variant == 0 && launch_identity(a, s)) {
        ++*launches;
        return;
    }
    if (a.variant == 2 && !a.identity_transfer) {
        const size_t psmem = tail3_pair_smem(a.n2, a.r0, a.r1, a.r2);
        if (psmem <= 220 * 1024) {
            switch ((a.r2 + 7) / 8) {
                case 1: launch_pair_nt<1>(a, psmem, s); break;
                case 2: launch_pair_nt<2>(a, psmem, s); break;
                default: launch_pair_nt<3>(a, psmem, s); break;
            }
            ++*launches;
            return;
        }
    }
    const size_t smem = tail3_smem(a.n2, a.r0, a.r1, a.r2);
    // small batches (per-rank shards of a multi-GPU run): when fewer than
    // half the SMs would hold a sample, split each sample over a cluster of up
    // to 8 CTAs (grid up to 2 CTAs per SM). Measured on c5 shards
    // (tools/shard_probe.py): S = 128 is fastest unsplit (the split adds the
    // all-gather and per-CTA staging without freeing pipe time), S = 64 with
    // 4-CTA and S = 32 with 4- or 8-CTA clusters (tail 69 -> 38 us at S = 32)
    Tail3Args b = a;
    b.csize = 1;
    if (a.variant != 1 && 2 * a.S <= static_cast<int64_t>(a.num_sms))
        while (b.csize < 8 && a.S * b.csize * 2 <= 2 * static_cast<int64_t>(a.num_sms) &&
               b.csize * 2 <= (a.rt + 15) / 16)  // at least one column pair per CTA
            b.csize *= 2;
    switch ((a.r2 + 7) / 8) {
        case 1: launch_nt<1>(b, smem, s); break;
        case 2: launch_nt<2>(b, smem, s); break;
        default: launch_nt<3>(b, smem, s); break;
    }
    ++*launches;
}

}  // namespace htr
