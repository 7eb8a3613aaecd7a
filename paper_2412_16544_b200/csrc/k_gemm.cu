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

// ---------------------------------------------------------------------------
// Fast path for plain contractions: single-level k and n maps, one operand
// dimension contiguous per operand, 16-byte aligned rows. 32x32 warp tiles
// (8 fragment loads feed 16 DMMAs per k-step), 16-byte cp.async staging into
// padded shared layouts (conflict-free fragment reads; k-contiguous operands
// read as 16-byte (k, k+1) pairs), 3 stages of 16 k. Optional
// per-CTA sum of squares of the stored outputs (sq_partials).
// ---------------------------------------------------------------------------
constexpr int FBK = 16;      // k per stage
constexpr int FSTAGE = 3;
// pitch of a k-contiguous row in shared memory: 16-byte fragment loads of
// (k, k+1) pairs from 8 rows x 4 pairs hit 8 distinct 16-byte bank groups
constexpr int FPK = FBK + 8;

struct FastArgs {
    int64_t M, N, K;
    int64_t sam, sak, sbk, sbn;  // single-level operand strides
    // two-level K whose inner extent k1 is a multiple of the k tile (a tile
    // never straddles the outer index): k = kr + k1 kq sits at kr sak + kq sak2
    // (A) / kr sbk + kq sbk2 (B); k1 = 0 for a single level
    int64_t k1, sak2, sbk2;
    int64_t kchunk, splits;
    double* partial;             // split-K partials or nullptr
    double* sq_partials;         // per-CTA sum of squares of C, or nullptr
    int staged;                  // C is n-contiguous, rows 16-byte aligned: coalesced epilogue
    int sym_lower;               // skip tiles strictly above the diagonal (mirrored afterwards)
};

template <int BM, int BN, bool AK>
__host__ __device__ constexpr int fast_a_doubles() {
    return AK ? BM * FPK : FBK * (BM + 4);
}
template <int BM, int BN, bool BKF>
__host__ __device__ constexpr int fast_b_doubles() {
    return BKF ? BN * FPK : FBK * (BN + 4);
}
template <int BM, int BN, bool AK, bool BKF>
constexpr size_t fast_smem_bytes() {
    return sizeof(double) * FSTAGE * (fast_a_doubles<BM, BN, AK>() + fast_b_doubles<BM, BN, BKF>());
}

__device__ __forceinline__ void cp_async16(double* dst, const double* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}

template <int BM, int BN, bool AK, bool BKF>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32, 2)
    gemm_fast_kernel(const GemmDesc d, const FastArgs f, const Launch L) {
    constexpr int WX = BM / 32, NTH = WX * (BN / 32) * 32;
    constexpr int SA = fast_a_doubles<BM, BN, AK>(), SB = fast_b_doubles<BM, BN, BKF>();
    constexpr int PAM = BM + 4, PBN = BN + 4;
    extern __shared__ __align__(16) double fsm[];
    double* As = fsm;                 // [FSTAGE][SA]
    double* Bs = fsm + FSTAGE * SA;   // [FSTAGE][SB]
    __shared__ double red[NTH / 32];

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int wm = (warp % WX) * 32, wn = (warp / WX) * 32;
    const int64_t zb = blockIdx.z / f.splits, zs = blockIdx.z - zb * f.splits;
    const double* A = d.A + zb * d.sab;
    const double* B = d.B + zb * d.sbb;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
    if (f.sym_lower && n0 >= m0 + BM) return;  // strictly above the diagonal: mirrored from the lower triangle
    const int64_t kbeg = zs * f.kchunk;
    const int64_t kend = min(f.K, kbeg + f.kchunk);
    const int ntiles = static_cast<int>((kend - kbeg + FBK - 1) / FBK);

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // stage fill: every operand row / column segment is copied in 16-byte
    // chunks (the contiguous extent is even, so a chunk is all in or all out)
    auto issue = [&](int kt, int st) {
        const int64_t k0 = kbeg + static_cast<int64_t>(kt) * FBK;
        double* as = As + st * SA;
        double* bs = Bs + st * SB;
        // operand offsets of the tile's first k (one or two K levels)
        int64_t ka = k0 * f.sak, kb = k0 * f.sbk;
        if (f.k1) {
            const int64_t kq = k0 / f.k1, kr = k0 - kq * f.k1;
            ka = kr * f.sak + kq * f.sak2;
            kb = kr * f.sbk + kq * f.sbk2;
        }
        if constexpr (AK) {
#pragma unroll
            for (int c = t; c < BM * (FBK / 2); c += NTH) {
                const int m = c / (FBK / 2), kk = 2 * (c % (FBK / 2));
                const bool ok = m0 + m < f.M && k0 + kk < kend;
                cp_async16(as + m * FPK + kk, ok ? A + (m0 + m) * f.sam + (ka + kk) : A, ok);
            }
        } else {
#pragma unroll
            for (int c = t; c < FBK * (BM / 2); c += NTH) {
                const int kk = c / (BM / 2), m = 2 * (c % (BM / 2));
                const bool ok = m0 + m < f.M && k0 + kk < kend;
                cp_async16(as + kk * PAM + m, ok ? A + ka + kk * f.sak + (m0 + m) : A, ok);
            }
        }
        if constexpr (BKF) {
#pragma unroll
            for (int c = t; c < BN * (FBK / 2); c += NTH) {
                const int n = c / (FBK / 2), kk = 2 * (c % (FBK / 2));
                const bool ok = n0 + n < f.N && k0 + kk < kend;
                cp_async16(bs + n * FPK + kk, ok ? B + (n0 + n) * f.sbn + (kb + kk) : B, ok);
            }
        } else {
#pragma unroll
            for (int c = t; c < FBK * (BN / 2); c += NTH) {
                const int kk = c / (BN / 2), n = 2 * (c % (BN / 2));
                const bool ok = n0 + n < f.N && k0 + kk < kend;
                cp_async16(bs + kk * PBN + n, ok ? B + kb + kk * f.sbk + (n0 + n) : B, ok);
            }
        }
    };

#pragma unroll
    for (int st = 0; st < FSTAGE - 1; ++st) {
        if (st < ntiles) issue(st, st);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int kt = 0; kt < ntiles; ++kt) {
        asm volatile("cp.async.wait_group %0;" ::"n"(FSTAGE - 2) : "memory");
        __syncthreads();
        if (kt + FSTAGE - 1 < ntiles) issue(kt + FSTAGE - 1, (kt + FSTAGE - 1) % FSTAGE);
        asm volatile("cp.async.commit_group;" ::: "memory");
        const double* as = As + (kt % FSTAGE) * SA;
        const double* bs = Bs + (kt % FSTAGE) * SB;
        // two k-steps per iteration; lane t4 carries k = ks + 2 t4 in the
        // first MMA and ks + 2 t4 + 1 in the second (the same split of the k
        // sum for A and B), so a k-contiguous operand is read as 16-byte pairs
        const int64_t kleft = kend - (kbeg + static_cast<int64_t>(kt) * FBK);  // valid k in this tile
#pragma unroll
        for (int ks = 0; ks < FBK; ks += 8) {
            if (ks >= kleft) break;  // warp-uniform: the zero-filled tail of the last tile
            double a0[4], a1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if constexpr (AK) {
                    const double2 v = *reinterpret_cast<const double2*>(as + (wm + 8 * i + g4) * FPK + ks + 2 * t4);
                    a0[i] = v.x;
                    a1[i] = v.y;
                } else {
                    a0[i] = as[(ks + 2 * t4) * PAM + wm + 8 * i + g4];
                    a1[i] = as[(ks + 2 * t4 + 1) * PAM + wm + 8 * i + g4];
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // B pairs loaded per column tile: fewer live registers
                double b0, b1;
                if constexpr (BKF) {
                    const double2 v = *reinterpret_cast<const double2*>(bs + (wn + 8 * j + g4) * FPK + ks + 2 * t4);
                    b0 = v.x;
                    b1 = v.y;
                } else {
                    b0 = bs[(ks + 2 * t4) * PBN + wn + 8 * j + g4];
                    b1 = bs[(ks + 2 * t4 + 1) * PBN + wn + 8 * j + g4];
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) dmma884(acc[i][j], a0[i], b0);
#pragma unroll
                for (int i = 0; i < 4; ++i) dmma884(acc[i][j], a1[i], b1);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");

    double* C = d.C + zb * d.scb;
    double sq = 0.0;
    if (f.staged && !f.partial) {
        // C rows are contiguous in n and 16-byte aligned: stage the tile in
        // shared memory and write it back in full 16-byte pairs (the direct
        // fragment layout leaves half of every 32-byte sector unwritten)
        constexpr int PC = BN + 2;
        double* cs = fsm;
        __syncthreads();  // every warp is done with the operand stages
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                double2 v;
                v.x = acc[i][j][0];
                v.y = acc[i][j][1];
                *reinterpret_cast<double2*>(cs + (wm + 8 * i + g4) * PC + wn + 8 * j + 2 * t4) = v;
            }
        __syncthreads();
#pragma unroll 4
        for (int e = t; e < BM * (BN / 2); e += NTH) {
            const int ml = e / (BN / 2), nl = 2 * (e % (BN / 2));
            const int64_t m = m0 + ml, n = n0 + nl;
            if (m >= f.M || n >= f.N) continue;
            double2 v = *reinterpret_cast<const double2*>(cs + ml * PC + nl);
            double* c = C + m * d.scm + n;
            if (n + 1 < f.N) {
                if (d.beta != 0.0) {
                    const double2 o = *reinterpret_cast<const double2*>(c);
                    v.x = fma(d.alpha, v.x, d.beta * o.x);
                    v.y = fma(d.alpha, v.y, d.beta * o.y);
                } else {
                    v.x *= d.alpha;
                    v.y *= d.alpha;
                }
                *reinterpret_cast<double2*>(c) = v;
                sq = fma(v.x, v.x, fma(v.y, v.y, sq));
            } else {
                const double x = d.beta == 0.0 ? d.alpha * v.x : fma(d.alpha, v.x, d.beta * *c);
                *c = x;
                sq = fma(x, x, sq);
            }
        }
    } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t m = m0 + wm + 8 * i + g4, n = n0 + wn + 8 * j + 2 * t4 + h;
                if (m < f.M && n < f.N) {
                    if (f.partial) {
                        f.partial[(static_cast<int64_t>(blockIdx.z) * f.M + m) * f.N + n] = acc[i][j][h];
                    } else {
                        double* c = C + m * d.scm + n_part(L, n, d.scn1, d.scn2, d.N1);
                        const double v = d.beta == 0.0 ? d.alpha * acc[i][j][h] : fma(d.alpha, acc[i][j][h], d.beta * *c);
                        *c = v;
                        sq = fma(v, v, sq);
                    }
                }
            }
    }
    if (f.sq_partials) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) red[warp] = sq;
        __syncthreads();
        if (t == 0) {
            double s2 = 0.0;
            for (int w = 0; w < NTH / 32; ++w) s2 += red[w];
            f.sq_partials[blockIdx.x + static_cast<int64_t>(gridDim.x) * (blockIdx.y + static_cast<int64_t>(gridDim.y) * blockIdx.z)] = s2;
        }
    }
}

// ---------------------------------------------------------------------------
// Persistent small-K expansion: out[i + I (q + Q o)] = sum_j M(q, j)
// t[i + I (j + J o)] with J <= 32, Q <= 128 (decode's leaf expansions,
// r -> n). M stays resident in shared memory; each CTA walks (o, 64-wide
// i-tile) items, double-buffering the t tiles (16-byte cp.async), computes
// the 128 x 64 tile on DMMA (32 x 32 warp tiles, (k, k+1) pair loads of M)
// and stores it from the fragments as 16-byte pairs (whole sectors). Two
// CTAs per SM overlap one tile's stores with the other's MMAs.
// ---------------------------------------------------------------------------
constexpr int XQ = 128, XN = 64, XJ = 32, XT = 256;
constexpr int XPA = XJ + 8;   // M row pitch ([q][j], pair loads conflict-free)
constexpr int XPB = XN + 4;   // t tile pitch ([j][i])
constexpr size_t expand_smem_bytes() { return sizeof(double) * (XQ * XPA + 2 * XJ * XPB); }

__global__ void __launch_bounds__(XT, 2) expand_kernel(const double* __restrict__ t, int64_t I, int J, int64_t O,
                                                       const double* __restrict__ Mp, int Q, int64_t smq,
                                                       int64_t smj, double* __restrict__ out) {
    extern __shared__ __align__(16) double xsm[];
    double* As = xsm;                      // [XQ][XPA]
    double* Bs = As + XQ * XPA;            // [2][XJ][XPB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
    const int JP = (J + 7) / 8 * 8;  // k processed in pairs of k-steps
    for (int e = tid; e < XQ * XJ; e += XT) {
        const int q = e / XJ, j = e % XJ;
        As[q * XPA + j] = (q < Q && j < J) ? Mp[q * smq + j * smj] : 0.0;
    }
    const int64_t tiles_i = (I + XN - 1) / XN;
    const int64_t items = tiles_i * O;
    // zero-filled k rows beyond J stay zero in both buffers
    for (int e = tid; e < 2 * XJ * XPB; e += XT) Bs[e] = 0.0;
    __syncthreads();

    auto issue = [&](int64_t item, int buf) {
        const int64_t o = item / tiles_i, i0 = (item - o * tiles_i) * XN;
        double* bs = Bs + buf * XJ * XPB;
        const double* src = t + I * static_cast<int64_t>(J) * o + i0;
        for (int c = tid; c < J * (XN / 2); c += XT) {
            const int j = c / (XN / 2), ii = 2 * (c % (XN / 2));
            const bool ok = i0 + ii < I;
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(bs + j * XPB + ii));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d),
                         "l"(ok ? src + I * j + ii : t), "r"(ok ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    int64_t item = blockIdx.x;
    int buf = 0;
    if (item < items) issue(item, 0);
    for (; item < items; item += gridDim.x, buf ^= 1) {
        const int64_t next = item + gridDim.x;
        if (next < items) {
            issue(next, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* bs = Bs + buf * XJ * XPB;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int ks = 0; ks < JP; ks += 8) {
            double a0[4], a1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double2 v = *reinterpret_cast<const double2*>(As + (wm + 8 * i + g4) * XPA + ks + 2 * t4);
                a0[i] = v.x;
                a1[i] = v.y;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double b0 = bs[(ks + 2 * t4) * XPB + wn + 8 * j + g4];
                const double b1 = bs[(ks + 2 * t4 + 1) * XPB + wn + 8 * j + g4];
#pragma unroll
                for (int i = 0; i < 4; ++i) dmma884(acc[i][j], a0[i], b0);
#pragma unroll
                for (int i = 0; i < 4; ++i) dmma884(acc[i][j], a1[i], b1);
            }
        }
        // 16-byte stores straight from the fragments: the 4 lanes of a row
        // write 64 contiguous bytes (whole sectors)
        const int64_t o = item / tiles_i, i0 = (item - o * tiles_i) * XN;
        double* dst = out + I * static_cast<int64_t>(Q) * o + i0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int q = wm + 8 * i + g4;
            if (q >= Q) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int ii = wn + 8 * j + 2 * t4;
                if (i0 + ii < I)
                    *reinterpret_cast<double2*>(dst + I * q + ii) = make_double2(acc[i][j][0], acc[i][j][1]);
            }
        }
        __syncthreads();  // this B buffer is refilled next-but-one item
    }
}

// C[m, n] = C[n, m] for n > m of a square single-level C (the symmetric
// contractions whose upper tiles were skipped)
__global__ void sym_mirror_kernel(double* C, int64_t n, int64_t scm, int64_t scn) {
    const int64_t total = n * n;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t m = idx % n, c = idx / n;
        if (c > m) C[m * scm + c * scn] = C[c * scm + m * scn];
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
    bool fast = false, ak = false, bkf = false;
    int64_t sam = 0, sak = 0, sbk = 0, sbn = 0;
    int64_t k1 = 0, sak2 = 0, sbk2 = 0;  // two-level K (fast kernel), see FastArgs
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

/// Single-level operand maps with one contiguous, even dimension per operand
/// and 16-byte aligned rows: eligible for gemm_fast_kernel.
bool fast_eligible(const GemmDesc& d, Plan& p) {
    if (d.energy_partials) return false;
    const int64_t M = d.M, N = d.N1 * d.N2, K = d.K1 * d.K2;
    if (d.K2 == 1) {
        p.sak = d.sak1;
        p.sbk = d.sbk1;
    } else if (d.K1 == 1) {
        p.sak = d.sak2;
        p.sbk = d.sbk2;
    } else if (d.sak2 == d.K1 * d.sak1 && d.sbk2 == d.K1 * d.sbk1) {
        p.sak = d.sak1;
        p.sbk = d.sbk1;
    } else if (d.K1 % FBK == 0 && ((d.sak2 | d.sbk2) & 1) == 0) {
        // two K levels, the inner a whole number of k tiles (the transfer
        // Grams of a projected layer: K = leading extent x batch)
        p.sak = d.sak1;
        p.sbk = d.sbk1;
        p.k1 = d.K1;
        p.sak2 = d.sak2;
        p.sbk2 = d.sbk2;
    } else {
        return false;
    }
    if (d.N2 == 1) p.sbn = d.sbn1;
    else if (d.N1 == 1) p.sbn = d.sbn2;
    else if (d.sbn2 == d.N1 * d.sbn1) p.sbn = d.sbn1;
    else return false;
    p.sam = d.sam;
    p.ak = p.sak == 1;
    p.bkf = p.sbk == 1;
    if (!p.ak && p.sam != 1) return false;
    if (!p.bkf && p.sbn != 1) return false;
    if (!aligned16(d.A) || !aligned16(d.B) || (d.batch > 1 && ((d.sab | d.sbb) & 1))) return false;
    if (p.ak ? ((K | p.sam) & 1) : ((M | p.sak) & 1)) return false;
    if (p.bkf ? ((K | p.sbn) & 1) : ((N | p.sbk) & 1)) return false;
    return M < (int64_t{1} << 31) && N < (int64_t{1} << 31) && K < (int64_t{1} << 31);
}

Plan plan_for(const GemmDesc& d, int num_sms) {
    Plan p;
    const int64_t N = d.N1 * d.N2, K = d.K1 * d.K2;
    p.fast = fast_eligible(d, p);
    // tile shape with the least padded area (ties: the first listed)
    const int slow_shapes[3][2] = {{64, 64}, {64, 32}, {32, 64}};
    const int fast_shapes[3][2] = {{128, 64}, {64, 128}, {64, 64}};
    const auto& shapes = p.fast ? fast_shapes : slow_shapes;
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

template <int BM, int BN, bool AK, bool BKF>
void launch_fast_t(const GemmDesc& d, const FastArgs& f, const Launch& L, dim3 grid, cudaStream_t s) {
    constexpr size_t smem = fast_smem_bytes<BM, BN, AK, BKF>();
    static_assert(sizeof(double) * BM * (BN + 2) <= smem, "C staging tile must fit the operand stages");
    ensure_smem_limit(reinterpret_cast<const void*>(gemm_fast_kernel<BM, BN, AK, BKF>), smem);
    gemm_fast_kernel<BM, BN, AK, BKF><<<grid, (BM / 32) * (BN / 32) * 32, smem, s>>>(d, f, L);
}

template <int BM, int BN>
void launch_fast_tile(const Plan& p, const GemmDesc& d, const FastArgs& f, const Launch& L, dim3 grid,
                      cudaStream_t s) {
    if (p.ak && p.bkf) launch_fast_t<BM, BN, true, true>(d, f, L, grid, s);
    else if (p.ak) launch_fast_t<BM, BN, true, false>(d, f, L, grid, s);
    else if (p.bkf) launch_fast_t<BM, BN, false, true>(d, f, L, grid, s);
    else launch_fast_t<BM, BN, false, false>(d, f, L, grid, s);
}

void launch_fast(const Plan& p, const GemmDesc& d, const FastArgs& f, const Launch& L, dim3 grid, cudaStream_t s) {
    if (p.bm == 128) launch_fast_tile<128, 64>(p, d, f, L, grid, s);
    else if (p.bn == 128) launch_fast_tile<64, 128>(p, d, f, L, grid, s);
    else launch_fast_tile<64, 64>(p, d, f, L, grid, s);
}

}  // namespace

int64_t gemm_workspace_doubles(const GemmDesc& d, int num_sms) {
    const Plan p = plan_for(d, num_sms);
    return p.splits > 1 ? p.splits * d.batch * d.M * d.N1 * d.N2 : 0;
}

bool gemm_is_fast(const GemmDesc& d, int num_sms) { return plan_for(d, num_sms).fast && plan_for(d, num_sms).splits == 1; }

int64_t gemm_energy_partials(const GemmDesc& d, int num_sms) {
    const Plan p = plan_for(d, num_sms);
    return p.tiles_n * p.tiles_m * d.batch;
}

int launch_expand(const double* t, int64_t I, int64_t J, int64_t O, const double* M, int64_t Q, int64_t smq,
                  int64_t smj, double* out, int num_sms, cudaStream_t s, int64_t* launches) {
    // 16-byte rows: I even, aligned bases; J, Q within the resident tile
    if (J > XJ || Q > XQ || Q < 1 || J < 1 || (I & 1) || !aligned16(t) || !aligned16(out)) return -1;
    ensure_smem_limit(reinterpret_cast<const void*>(expand_kernel), expand_smem_bytes());
    const int64_t items = (I + XN - 1) / XN * O;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(items, 2 * num_sms)));
    expand_kernel<<<grid, XT, expand_smem_bytes(), s>>>(t, I, static_cast<int>(J), O, M, static_cast<int>(Q), smq, smj,
                                                        out);
    ++*launches;
    return grid;
}

int launch_gemm(const GemmDesc& d, double* workspace, int num_sms, cudaStream_t s, int64_t* launches,
                double* sq_partials) {
    const int64_t N = d.N1 * d.N2, K = d.K1 * d.K2;
    if (d.M <= 0 || N <= 0 || d.batch <= 0) return 0;
    if (K <= 0) return 0;  // extents are >= 1 by construction
    const Plan p = plan_for(d, num_sms);
    ensure_smem_limit(reinterpret_cast<const void*>(gemm_kernel<64, 64>), gemm_smem_bytes<64, 64>());
    ensure_smem_limit(reinterpret_cast<const void*>(gemm_kernel<64, 32>), gemm_smem_bytes<64, 32>());
    ensure_smem_limit(reinterpret_cast<const void*>(gemm_kernel<32, 64>), gemm_smem_bytes<32, 64>());
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
    if (p.fast) {
        // coalesced epilogue: C single-level and contiguous in n, 16-byte rows
        const bool c_flat = d.N2 == 1 || d.N1 == 1 ? true : d.scn2 == d.N1 * d.scn1;
        const int64_t c_sn = d.N2 == 1 ? d.scn1 : (d.N1 == 1 ? d.scn2 : d.scn1);
        const int staged = c_flat && c_sn == 1 && aligned16(d.C) && (d.scm % 2 == 0) &&
                           (d.batch == 1 || d.scb % 2 == 0);
        // symmetric results: lower tiles only (square, single-level C, no
        // accumulation into C, no per-CTA sums of squares)
        const int sym = d.symmetric && d.M == N && d.batch == 1 && d.beta == 0.0 && !sq_partials && (d.N2 == 1 || d.N1 == 1);
        FastArgs f{d.M, N, K, p.sam, p.sak, p.sbk, p.sbn, p.k1, p.sak2, p.sbk2, p.kchunk, p.splits, partial, sq_partials, staged, sym};
        launch_fast(p, d, f, L, grid, s);
        ++*launches;
        if (p.splits > 1) {
            const int64_t total = d.M * N * d.batch;
            const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * num_sms));
            splitk_reduce_kernel<<<blocks, 256, 0, s>>>(d, partial, p.splits, L);
            ++*launches;
        }
        if (sym) {
            const int64_t scn = d.N2 == 1 ? d.scn1 : d.scn2;
            const int blocks = static_cast<int>(std::min<int64_t>((d.M * d.M + 255) / 256, 8 * num_sms));
            sym_mirror_kernel<<<blocks, 256, 0, s>>>(d.C, d.M, d.scm, scn);
            ++*launches;
        }
        return 0;
    }
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
