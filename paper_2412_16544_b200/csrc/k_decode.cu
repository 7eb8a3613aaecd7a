// Fused two-leaf reconstruction (decode's last step, bht.hpp:437-455):
//
//   X[i0 + n0 (i1 + n1 t)] = sum_{a0,a1} U0[i0, a0] U1[i1, a1] W[a0 + r0 (a1 + r1 t)]
//
// for every slab t (the remaining modes and the samples, already expanded
// into W). One warp owns a slab at a time and never writes an intermediate:
//
//   step A (DMMA, M = i1, N = a0, K = a1):  T[i1, a0] = sum_a1 U1[i1, a1] W[a0, a1]
//   step B (DMMA, M = i1, N = i0, K = a0):  X[i0, i1] = sum_a0 T[i1, a0] U0[i0, a0]
//
// Step B takes its A operand straight from step A's accumulators: a C
// fragment holds T[i1 = g][a0 = 8 nt + 2 t + h] on lane (g, t), which is the A
// fragment of a k-step whose k index is permuted to (nt, h); U0's fragments
// are pre-permuted to the same k order in shared memory. A rank that ends in
// a half tile (r0 mod 8 in 1..4) gets one plain k-step built with two
// shuffles, so the contraction runs over ceil(r0/4) k-steps instead of
// 2 ceil(r0/8) — the ranks are contraction dimensions in both steps, padded
// to 4, not to 8. The output tile is stored from the fragments as 16-byte
// pairs (four lanes cover 64 contiguous bytes of a row). The slabs' W blocks
// are double-buffered per warp with cp.async.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kDecWarps = 8;
constexpr int kDecMaxR = 24;
constexpr int kDecMaxN1 = 128;
constexpr int kDecWS = kDecMaxR * kDecMaxR;  // W block per buffer (doubles)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

template <int N0T, int MT0>
constexpr size_t decode2_smem_doubles() {
    return static_cast<size_t>(N0T) * MT0 * 64 + (kDecMaxN1 / 8) * 3 * 64 + kDecWarps * 2 * kDecWS;
}

struct DecodeFinal {
    double* out;           // residual mode: the total sum (X - Y)^2, or null (partials only)
    double* host_out;      // optional mapped-host copy
    unsigned int* ticket;  // zero on entry, left zero
};

// N0T: n0 / 8 (i0 n-tiles); MT0: ceil(r0 / 8) (a0 tiles of step A's output)
// RESID: instead of storing X, accumulate sum (X - Y)^2 (relative_test_error,
// metrics.hpp:218-237) into one partial per warp; the reconstruction is never
// written.
template <int N0T, int MT0, bool RESID>
__global__ void __launch_bounds__(kDecWarps * 32, 1)
    decode2_kernel(const double* __restrict__ W, int64_t T, int r0, int r1, int n1, const double* __restrict__ U0,
                   const double* __restrict__ U1, double* __restrict__ X, const double* __restrict__ Y,
                   double* __restrict__ partials, const DecodeFinal fin) {
    constexpr int HT = N0T > 8 ? 8 : N0T;  // n-tiles per pass (accumulator budget)
    constexpr int NH = N0T / HT;
    constexpr int n0 = 8 * N0T;
    extern __shared__ __align__(16) double dsm[];
    double* U0p = dsm;                           // [N0T][MT0][32 lanes][2]
    double* U1p = U0p + N0T * MT0 * 64;          // [n1/8][3][32 lanes][2]
    double* Wb = U1p + (kDecMaxN1 / 8) * 3 * 64;  // [warps][2][kDecWS]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;

    // k-step plan for the a0 contraction: F full (permuted) tiles, then one
    // half-tile step if r0 mod 8 is 1..4 (5..7 pad the tile instead)
    int F = r0 / 8, rem = r0 % 8;
    if (rem > 4) {
        ++F;
        rem = 0;
    }
    const int KB0 = 2 * F + (rem > 0 ? 1 : 0);
    const int KS1 = (r1 + 3) / 4;

    for (int e = tid; e < N0T * MT0 * 64; e += blockDim.x) {
        const int h = e & 1, ln = (e >> 1) & 31, kp = (e >> 6) % MT0, j = (e >> 6) / MT0;
        const int kk = 2 * kp + h, g = ln >> 2, t = ln & 3;
        int a0 = kDecMaxR;
        if (kk < 2 * F) a0 = 8 * (kk >> 1) + 2 * t + (kk & 1);
        else if (kk == 2 * F && rem > 0) a0 = 8 * F + t;
        U0p[e] = a0 < r0 ? U0[(8 * j + g) + static_cast<int64_t>(n0) * a0] : 0.0;
    }
    for (int e = tid; e < (n1 / 8) * 3 * 64; e += blockDim.x) {
        const int h = e & 1, ln = (e >> 1) & 31, kp = (e >> 6) % 3, mt = (e >> 6) / 3;
        const int a1 = 4 * (2 * kp + h) + (ln & 3), i1 = 8 * mt + (ln >> 2);
        U1p[e] = a1 < r1 ? U1[i1 + static_cast<int64_t>(n1) * a1] : 0.0;
    }
    __syncthreads();

    const int64_t gw = static_cast<int64_t>(blockIdx.x) * kDecWarps + warp;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kDecWarps;
    const int wsz = r0 * r1;
    double* wbuf = Wb + warp * 2 * kDecWS;
    auto issue = [&](int64_t t, int buf) {
        const double* src = W + static_cast<int64_t>(wsz) * t;
        for (int e = lane; e < wsz; e += 32) cp_async8(wbuf + buf * kDecWS + e, src + e);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (gw < T) issue(gw, 0);
    int buf = 0;
    const int np = n1 / 16;
    const int src_lane = (lane & ~3) | (t4 >> 1);
    double rs = 0.0;
    for (int64_t t = gw; t < T; t += nw, buf ^= 1) {
        if (t + nw < T) {
            issue(t + nw, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        const double* wb = wbuf + buf * kDecWS;
        // step A's B operand: W[a0 = 8 nt + g][a1 = 4 ks + t]
        double wf[MT0][6];
#pragma unroll
        for (int nt = 0; nt < MT0; ++nt)
#pragma unroll
            for (int ks = 0; ks < 6; ++ks) {
                const int a0 = 8 * nt + g4, a1 = 4 * ks + t4;
                wf[nt][ks] = (a0 < r0 && a1 < r1) ? wb[a0 + r0 * a1] : 0.0;
            }
        __syncwarp();  // this buffer is refilled two slabs later
        const int64_t xoff = static_cast<int64_t>(n0) * n1 * t;
        for (int p = 0; p < np; ++p) {
            double ca[2][MT0][2];
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int nt = 0; nt < MT0; ++nt) ca[m][nt][0] = ca[m][nt][1] = 0.0;
#pragma unroll
            for (int kp = 0; kp < 3; ++kp) {
                if (2 * kp >= KS1) break;
                double2 u[2];
#pragma unroll
                for (int m = 0; m < 2; ++m)
                    u[m] = *reinterpret_cast<const double2*>(U1p + (((2 * p + m) * 3 + kp) * 32 + lane) * 2);
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int nt = 0; nt < MT0; ++nt) dmma(ca[m][nt], u[m].x, wf[nt][2 * kp]);
                if (2 * kp + 1 < KS1) {
#pragma unroll
                    for (int m = 0; m < 2; ++m)
#pragma unroll
                        for (int nt = 0; nt < MT0; ++nt) dmma(ca[m][nt], u[m].y, wf[nt][2 * kp + 1]);
                }
            }
            // step B's A operand, k order (nt, h) then the half-tile step
            double af[2][2 * MT0];
#pragma unroll
            for (int m = 0; m < 2; ++m) {
#pragma unroll
                for (int kk = 0; kk < 2 * MT0; ++kk) af[m][kk] = ca[m][kk >> 1][kk & 1];
                if (rem > 0) {
#pragma unroll
                    for (int nt = 0; nt < MT0; ++nt)
                        if (nt == F) {
                            const double lo = __shfl_sync(0xffffffffu, ca[m][nt][0], src_lane);
                            const double hi = __shfl_sync(0xffffffffu, ca[m][nt][1], src_lane);
                            af[m][2 * nt] = (t4 & 1) ? hi : lo;
                        }
                }
            }
#pragma unroll
            for (int hh = 0; hh < NH; ++hh) {
                const int64_t rowoff[2] = {xoff + static_cast<int64_t>(n0) * (16 * p + g4) + 8 * hh * HT + 2 * t4,
                                           xoff + static_cast<int64_t>(n0) * (16 * p + 8 + g4) + 8 * hh * HT + 2 * t4};
                double2 yv[RESID ? 2 : 1][RESID ? HT : 1];
                if constexpr (RESID) {
#pragma unroll
                    for (int m = 0; m < 2; ++m)
#pragma unroll
                        for (int j = 0; j < HT; ++j)
                            asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                                         : "=d"(yv[m][j].x), "=d"(yv[m][j].y)
                                         : "l"(Y + rowoff[m] + 8 * j));
                }
                double acc[2][HT][2];
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int j = 0; j < HT; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
#pragma unroll
                for (int kp = 0; kp < MT0; ++kp) {
                    if (2 * kp >= KB0) break;
                    const bool second = 2 * kp + 1 < KB0;
#pragma unroll
                    for (int j = 0; j < HT; ++j) {
                        const double2 b =
                            *reinterpret_cast<const double2*>(U0p + (((hh * HT + j) * MT0 + kp) * 32 + lane) * 2);
#pragma unroll
                        for (int m = 0; m < 2; ++m) dmma(acc[m][j], af[m][2 * kp], b.x);
                        if (second) {
#pragma unroll
                            for (int m = 0; m < 2; ++m) dmma(acc[m][j], af[m][2 * kp + 1], b.y);
                        }
                    }
                }
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int j = 0; j < HT; ++j) {
                        if constexpr (RESID) {
                            const double d0 = acc[m][j][0] - yv[m][j].x, d1 = acc[m][j][1] - yv[m][j].y;
                            rs = fma(d0, d0, fma(d1, d1, rs));
                        } else {
                            *reinterpret_cast<double2*>(X + rowoff[m] + 8 * j) = make_double2(acc[m][j][0], acc[m][j][1]);
                        }
                    }
            }
        }
    }
    if constexpr (RESID) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
        if (lane == 0) partials[gw] = rs;
        if (fin.out == nullptr) return;
        // the last CTA to finish (ticket counter) sums every warp's partial in
        // a fixed order and publishes the total, also into mapped host memory
        // when given: the stream API's explicit loss needs neither a reduction
        // launch nor a device-to-host copy
        __shared__ bool last;
        __shared__ double fred[kDecWarps];
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            last = atomicAdd(fin.ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (!last) return;
        __threadfence();
        const int64_t np = static_cast<int64_t>(gridDim.x) * kDecWarps;
        double t = 0.0;
        for (int64_t i = tid; i < np; i += kDecWarps * 32) t += __ldcg(partials + i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) fred[warp] = t;
        __syncthreads();
        if (tid == 0) {
            double sum = 0.0;
            for (int w = 0; w < kDecWarps; ++w) sum += fred[w];
            fin.out[0] = sum;
            if (fin.host_out) fin.host_out[0] = sum;
            *fin.ticket = 0u;
        }
    }
}

template <int N0T, int MT0, bool RESID>
int launch_t(const Decode2Args& a, int num_sms, cudaStream_t s) {
    constexpr size_t smem = sizeof(double) * decode2_smem_doubles<N0T, MT0>();
    ensure_smem_limit(reinterpret_cast<const void*>(decode2_kernel<N0T, MT0, RESID>), smem);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms, (a.T + kDecWarps - 1) / kDecWarps)));
    decode2_kernel<N0T, MT0, RESID><<<grid, kDecWarps * 32, smem, s>>>(a.W, a.T, a.r0, a.r1, static_cast<int>(a.n1),
                                                                        a.U0, a.U1, a.X, a.Y, a.partials,
                                                                        DecodeFinal{a.final_out, a.final_host, a.ticket});
    return grid;
}

template <int N0T, bool RESID>
int launch_n0(const Decode2Args& a, int num_sms, cudaStream_t s) {
    const int mt0 = (a.r0 + 7) / 8;
    if (mt0 == 1) return launch_t<N0T, 1, RESID>(a, num_sms, s);
    if (mt0 == 2) return launch_t<N0T, 2, RESID>(a, num_sms, s);
    return launch_t<N0T, 3, RESID>(a, num_sms, s);
}

template <bool RESID>
int launch_r(const Decode2Args& a, int num_sms, cudaStream_t s) {
    if (a.n0 == 32) return launch_n0<4, RESID>(a, num_sms, s);
    if (a.n0 == 64) return launch_n0<8, RESID>(a, num_sms, s);
    return launch_n0<16, RESID>(a, num_sms, s);
}

// sum (x - y)^2 per block (the generic path's residual)
__global__ void __launch_bounds__(256) diff_sumsq_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                         int64_t n, double* __restrict__ partials) {
    __shared__ double sh[8];
    double s = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double d = x[i] - y[i];
        s = fma(d, d, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += sh[w];
        partials[blockIdx.x] = t;
    }
}

}  // namespace

bool decode2_supported(int64_t n0, int64_t n1, int64_t r0, int64_t r1) {
    return (n0 == 32 || n0 == 64 || n0 == 128) && n1 >= 16 && n1 <= kDecMaxN1 && n1 % 16 == 0 && r0 >= 1 &&
           r0 <= kDecMaxR && r1 >= 1 && r1 <= kDecMaxR && r0 <= n0 && r1 <= n1;
}

int launch_decode2(const Decode2Args& a, int num_sms, cudaStream_t s, int64_t* launches) {
    if (!decode2_supported(a.n0, a.n1, a.r0, a.r1) || a.T < 1) return -1;
    if ((!a.Y && (reinterpret_cast<uintptr_t>(a.X) & 15u) != 0) || (reinterpret_cast<uintptr_t>(a.W) & 7u) != 0) return -1;
    if (a.Y && (!a.partials || (reinterpret_cast<uintptr_t>(a.Y) & 15u) != 0)) return -1;
    if (a.final_out && !a.ticket) return -1;
    const int grid = a.Y ? launch_r<true>(a, num_sms, s) : launch_r<false>(a, num_sms, s);
    ++*launches;
    return grid;
}

int64_t decode2_partials(int64_t T, int num_sms) {
    return static_cast<int64_t>(std::max<int64_t>(1, std::min<int64_t>(num_sms, (T + kDecWarps - 1) / kDecWarps))) *
           kDecWarps;
}

int launch_diff_sumsq(const double* x, const double* y, int64_t n, double* partials, int num_sms, cudaStream_t s,
                      int64_t* launches) {
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4 * num_sms, (n + 255) / 256)));
    diff_sumsq_kernel<<<grid, 256, 0, s>>>(x, y, n, partials);
    ++*launches;
    return grid;
}

}  // namespace htr
