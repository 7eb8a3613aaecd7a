// Small deterministic kernels: norms, the truncation rank rule, basis column
// extraction, zero padding and fills.
#include <algorithm>

#include "kernels.cuh"

namespace htr {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-block sum of squares with a non-finite flag (frobenius_norm,
// tensor.hpp:269, fused with DenseTensor::all_finite, bht.hpp:208-211).
__global__ void __launch_bounds__(256) sumsq_kernel(const double* __restrict__ x, int64_t n,
                                                    double* __restrict__ partials) {
    __shared__ double sh[8];
    __shared__ int bad_sh[8];
    double s0 = 0.0, s1 = 0.0;
    int bad = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    if (aligned) {
        const int64_t n2 = n / 2;
        const double2* x2 = reinterpret_cast<const double2*>(x);
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2; i += stride) {
            double2 v;
            asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                         : "=d"(v.x), "=d"(v.y)
                         : "l"(x2 + i));
            s0 = fma(v.x, v.x, s0);
            s1 = fma(v.y, v.y, s1);
            bad |= !isfinite(v.x) | !isfinite(v.y);
        }
        if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
            const double v = x[n - 1];
            s0 = fma(v, v, s0);
            bad |= !isfinite(v);
        }
    } else {
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
            const double v = x[i];
            s0 = fma(v, v, s0);
            bad |= !isfinite(v);
        }
    }
    double s = warp_sum(s0 + s1);
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        sh[threadIdx.x >> 5] = s;
        bad_sh[threadIdx.x >> 5] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        int b = 0;
        for (int w = 0; w < 8; ++w) {
            t += sh[w];
            b |= bad_sh[w];
        }
        partials[2 * blockIdx.x] = t;
        partials[2 * blockIdx.x + 1] = b ? 1.0 : 0.0;
    }
}

__global__ void sumsq_finish_kernel(const double* partials, int nb, double* out) {
    // one warp, fixed lane striding and shuffle tree: deterministic
    double t = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nb; i += 32) {
        t += partials[2 * i];
        b = fmax(b, partials[2 * i + 1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, o);
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (threadIdx.x == 0) {
        out[0] = t;
        out[1] = b;
    }
}

__global__ void sum_partials_kernel(const double* partials, int64_t n, double* out) {
    // one warp, fixed lane striding and fixed shuffle tree: deterministic
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 32) s += partials[i];
    s = warp_sum(s);
    if (threadIdx.x == 0) out[0] = s;
}

constexpr int kDefectMax = 64;
struct DefectJobs {
    const double* U[kDefectMax];
    int64_t alpha[kDefectMax], r[kDefectMax];
};

__global__ void __launch_bounds__(256) basis_defect_kernel(DefectJobs jobs, double* out) {
    const double* U = jobs.U[blockIdx.x];
    const int64_t alpha = jobs.alpha[blockIdx.x], r = jobs.r[blockIdx.x];
    double acc = 0.0;
    // entries (a, b), a <= b, of U^T U - I; off-diagonal ones count twice
    for (int64_t ab = threadIdx.x; ab < r * r; ab += blockDim.x) {
        const int64_t a = ab % r, b = ab / r;
        if (a > b) continue;
        double d = 0.0;
        for (int64_t i = 0; i < alpha; ++i) d = fma(U[i + alpha * a], U[i + alpha * b], d);
        if (a == b) d -= 1.0;
        acc = fma(a == b ? 1.0 : 2.0, d * d, acc);
    }
    __shared__ double red[8];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        out[blockIdx.x] = sqrt(t);
    }
}

// truncated_svd.hpp:74-99 on sigma_i^2 = max(lambda_i, 0), i < k.
__global__ void rank_rule_kernel(const double* lambda, int64_t k, int64_t n, double eps_abs, int64_t min_rank,
                                 const double* trace_src, double* info) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double trace = 0.0;
    if (trace_src) {
        trace = trace_src[0];
    } else {
        for (int64_t i = 0; i < n; ++i) trace += fmax(lambda[i], 0.0);
    }
    if (trace == 0.0) {
        // zero input -> canonical columns (truncated_svd.hpp:66-72)
        const int64_t r = min(min_rank > 0 ? min_rank : int64_t(0), n);
        info[0] = static_cast<double>(r);
        info[1] = 0.0;
        info[2] = 0.0;
        return;
    }
    // tail[r] = sum_{i >= r} sigma_i^2 accumulated from the smallest value
    // upwards; the smallest r with sqrt(tail[r]) <= eps wins.
    int64_t rank = k;
    double tail = 0.0;
    double tail_at_rank = 0.0;
    // walk down from r = k: tail[k] = 0; remember the smallest qualifying r
    bool found = false;
    if (0.0 <= eps_abs) {
        rank = k;
        tail_at_rank = 0.0;
        found = true;
    }
    for (int64_t r = k - 1; r >= 0; --r) {
        const double l = fmax(lambda[r], 0.0);
        tail += l;
        if (sqrt(tail) <= eps_abs) {
            rank = r;
            tail_at_rank = tail;
            found = true;
        } else {
            break;  // tails only grow as r decreases
        }
    }
    if (!found) rank = k;
    int64_t final_rank = max(rank, min_rank);
    final_rank = min(final_rank, k);
    if (final_rank != rank) {
        // recompute the discarded tail at the adjusted rank
        double t = 0.0;
        for (int64_t r = k - 1; r >= final_rank; --r) t += fmax(lambda[r], 0.0);
        tail_at_rank = t;
    }
    info[0] = static_cast<double>(final_rank);
    info[1] = sqrt(tail_at_rank);
    info[2] = trace;
}

__global__ void take_columns_kernel(const double* V, int64_t n, int64_t r, double* U, const double* info) {
    const bool zero_input = info[2] == 0.0;
    const int64_t total = n * r;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx % n, j = idx / n;
        U[idx] = zero_input ? (i == j ? 1.0 : 0.0) : V[i + n * j];
    }
}

// X[a + ext * (i + inner * o)] = T[i + inner * (a + ext * o)]: the mode
// unfolding of T (viewed [inner, ext, outer]) as a contiguous ext-row matrix.
__global__ void unfold_kernel(const double* __restrict__ src, int64_t inner, int64_t ext, int64_t outer,
                              double* __restrict__ dst) {
    const int64_t total = inner * ext * outer;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx % inner;  // reads coalesced along the inner axis
        const int64_t rest = idx / inner;
        const int64_t a = rest % ext, o = rest / ext;
        dst[a + ext * (i + inner * o)] = src[idx];
    }
}

__global__ void pad_axis_kernel(const double* src, int64_t inner, int64_t ext, int64_t outer, int64_t extra,
                                double* dst) {
    const int64_t next = ext + extra;
    const int64_t total = inner * next * outer;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx % inner;
        const int64_t rest = idx / inner;
        const int64_t e = rest % next, o = rest / next;
        dst[idx] = e < ext ? src[i + inner * (e + ext * o)] : 0.0;
    }
}

__global__ void fill_kernel(double* dst, int64_t n, double v) {
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < n;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[idx] = v;
}

// Small mode product out[i, q, o] = sum_j M(q, j) t[i, j, o] for J, Q <= 32:
// one thread per (i, o) fibre, M broadcast from shared memory, every input
// element read once and every output written once (HBM-bound; the DMMA
// engine would pad such tiny extents to 32-64 rows). Optional residual
// energy sum_fibre ||t - M^T (M t)||^2 for orthonormal-basis projections
// (bht.hpp:361), written as one partial per CTA.
template <int JM, int QM>
__device__ __forceinline__ void small_fibre(const double (&x)[JM], const double* Ms, int J, double (&y)[QM],
                                            double* energy_acc) {
#pragma unroll
    for (int q = 0; q < QM; ++q) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < JM; ++j) acc = fma(Ms[q + QM * j], x[j], acc);
        y[q] = acc;
    }
    if (energy_acc) {
        // residual of the projection: x - M^T y (bht.hpp:361)
#pragma unroll
        for (int j = 0; j < JM; ++j) {
            if (j >= J) continue;
            double back = 0.0;
#pragma unroll
            for (int q = 0; q < QM; ++q) back = fma(Ms[q + QM * j], y[q], back);
            const double r = x[j] - back;
            *energy_acc = fma(r, r, *energy_acc);
        }
    }
}

template <int JM, int QM, bool MODE0>
__global__ void __launch_bounds__(256) mode_small_kernel(const double* __restrict__ t, int64_t I, int J, int64_t O,
                                                          const double* __restrict__ M, int Q, int64_t smq, int64_t smj,
                                                          double* __restrict__ out, double* energy, double* ysq) {
    __shared__ double Ms[QM * JM];  // zero-padded to QM x JM
    __shared__ double red[8];
    __shared__ double red_y[8];
    // MODE0 (I == 1): per-warp staging of 32 consecutive fibres (coalesced)
    __shared__ double stage[MODE0 ? 4 : 1][MODE0 ? 32 * (JM > QM ? JM : QM) + 32 : 1];  // 4 warps in MODE0
    for (int e = threadIdx.x; e < QM * JM; e += blockDim.x) {
        const int q = e % QM, j = e / QM;
        Ms[e] = (q < Q && j < J) ? M[q * smq + j * smj] : 0.0;
    }
    __syncthreads();
    double en = 0.0, ys = 0.0;  // residual energy, ||t||^2 (the input read once for both)
    double* enp = energy ? &en : nullptr;
    if constexpr (MODE0) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        double* st = stage[warp];
        const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
        for (int64_t base = (blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + warp) * 32; base < O;
             base += nwarps * 32) {
            const int nf = static_cast<int>(O - base < 32 ? O - base : 32);
            const double* src = t + base * J;
            for (int e = lane; e < nf * J; e += 32) {
                const int f = e / J, j = e - f * J;
                st[f * (JM + 1) + j] = __ldg(src + e);
            }
            __syncwarp();
            double x[JM], y[QM];
#pragma unroll
            for (int j = 0; j < JM; ++j) x[j] = (lane < nf && j < J) ? st[lane * (JM + 1) + j] : 0.0;
            if (ysq)
#pragma unroll
                for (int j = 0; j < JM; ++j) ys = fma(x[j], x[j], ys);
            small_fibre<JM, QM>(x, Ms, J, y, lane < nf ? enp : nullptr);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < QM; ++q)
                if (q < Q) st[lane * (QM + 1) + q] = y[q];
            __syncwarp();
            double* dst = out + base * Q;
            for (int e = lane; e < nf * Q; e += 32) {
                const int f = e / Q, q = e - f * Q;
                dst[e] = st[f * (QM + 1) + q];
            }
            __syncwarp();
        }
    } else {
        const int64_t fibres = I * O;
        for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < fibres;
             f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t o = f / I, i = f - o * I;
            const double* src = t + i + I * J * o;
            double x[JM], y[QM];
#pragma unroll
            for (int j = 0; j < JM; ++j) x[j] = j < J ? __ldg(src + I * j) : 0.0;
            if (ysq)
#pragma unroll
                for (int j = 0; j < JM; ++j) ys = fma(x[j], x[j], ys);
            small_fibre<JM, QM>(x, Ms, J, y, enp);
            double* dst = out + i + I * static_cast<int64_t>(Q) * o;
#pragma unroll
            for (int q = 0; q < QM; ++q)
                if (q < Q) dst[I * q] = y[q];
        }
    }
    if (energy || ysq) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            en += __shfl_xor_sync(0xffffffffu, en, off);
            ys += __shfl_xor_sync(0xffffffffu, ys, off);
        }
        if ((threadIdx.x & 31) == 0) {
            red[threadIdx.x >> 5] = en;
            red_y[threadIdx.x >> 5] = ys;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0, toty = 0.0;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
                tot += red[w];
                toty += red_y[w];
            }
            if (energy) energy[blockIdx.x] = tot;
            if (ysq) ysq[blockIdx.x] = toty;
        }
    }
}

// Two adjacent modes at once: out[i, q0, q1, o] = sum_{j0, j1} U0[j0, q0]
// t[i, j0, j1, o] U1[j1, q1], one thread per (i, o) plane of J0 x J1
// elements (read once, contracted in registers), plus per-CTA ||t||^2
// partials. Extents are templated upper bounds, zero-padded in shared memory.
template <int JM0, int JM1, int QM0, int QM1>
__global__ void __launch_bounds__(256) pair_project_kernel(const double* __restrict__ t, int64_t I, int J0, int J1,
                                                           int64_t O, const double* __restrict__ U0, int Q0,
                                                           const double* __restrict__ U1, int Q1,
                                                           double* __restrict__ out, double* ysq) {
    __shared__ double U0s[JM0 * QM0], U1s[JM1 * QM1];  // [j][q]
    __shared__ double red[8];
    for (int e = threadIdx.x; e < JM0 * QM0; e += blockDim.x) {
        const int j = e / QM0, q = e % QM0;
        U0s[e] = (j < J0 && q < Q0) ? U0[j + static_cast<int64_t>(J0) * q] : 0.0;
    }
    for (int e = threadIdx.x; e < JM1 * QM1; e += blockDim.x) {
        const int j = e / QM1, q = e % QM1;
        U1s[e] = (j < J1 && q < Q1) ? U1[j + static_cast<int64_t>(J1) * q] : 0.0;
    }
    __syncthreads();
    double ys = 0.0;
    const int64_t planes = I * O;
    for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < planes;
         f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t o = f / I, i = f - o * I;
        const double* src = t + i + I * static_cast<int64_t>(J0) * J1 * o;
        double acc[QM0][QM1];
#pragma unroll
        for (int a = 0; a < QM0; ++a)
#pragma unroll
            for (int b = 0; b < QM1; ++b) acc[a][b] = 0.0;
#pragma unroll
        for (int j1 = 0; j1 < JM1; ++j1) {
            if (j1 >= J1) break;
            double x[JM0];
#pragma unroll
            for (int j0 = 0; j0 < JM0; ++j0) x[j0] = j0 < J0 ? __ldg(src + I * (j0 + static_cast<int64_t>(J0) * j1)) : 0.0;
            double tq[QM0];
#pragma unroll
            for (int a = 0; a < QM0; ++a) {
                double v = 0.0;
#pragma unroll
                for (int j0 = 0; j0 < JM0; ++j0) v = fma(U0s[j0 * QM0 + a], x[j0], v);
                tq[a] = v;
            }
#pragma unroll
            for (int j0 = 0; j0 < JM0; ++j0) ys = fma(x[j0], x[j0], ys);
#pragma unroll
            for (int a = 0; a < QM0; ++a)
#pragma unroll
                for (int b = 0; b < QM1; ++b) acc[a][b] = fma(tq[a], U1s[j1 * QM1 + b], acc[a][b]);
        }
        double* dst = out + i + I * static_cast<int64_t>(Q0) * Q1 * o;
#pragma unroll
        for (int b = 0; b < QM1; ++b)
#pragma unroll
            for (int a = 0; a < QM0; ++a)
                if (a < Q0 && b < Q1) dst[I * (a + static_cast<int64_t>(Q0) * b)] = acc[a][b];
    }
    if (ysq) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ys += __shfl_xor_sync(0xffffffffu, ys, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ys;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
            ysq[blockIdx.x] = tot;
        }
    }
}

// pair_project for contiguous planes (I == 1): 8 lanes per plane, lane j1
// reads column j1 (J0 contiguous doubles), so a warp streams 4 whole planes
// (2 KB contiguous for 8x8); the column contributions are summed across the
// 8 lanes with xor shuffles and written as one contiguous Q0*Q1 block.
__global__ void __launch_bounds__(256) pair_project_contig_kernel(const double* __restrict__ t, int J0, int J1,
                                                                  int64_t O, const double* __restrict__ U0, int Q0,
                                                                  const double* __restrict__ U1, int Q1,
                                                                  double* __restrict__ out, double* ysq) {
    constexpr int JM = 8, QM = 4;
    __shared__ double U0s[JM * QM], U1s[JM * QM];  // [j][q]
    __shared__ double red[8];
    for (int e = threadIdx.x; e < JM * QM; e += blockDim.x) {
        const int j = e / QM, q = e % QM;
        U0s[e] = (j < J0 && q < Q0) ? U0[j + static_cast<int64_t>(J0) * q] : 0.0;
        U1s[e] = (j < J1 && q < Q1) ? U1[j + static_cast<int64_t>(J1) * q] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, j1 = lane & 7, sub = lane >> 3;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t wid = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t plane = static_cast<int64_t>(J0) * J1, QQ = static_cast<int64_t>(Q0) * Q1;
    double ys = 0.0;
    for (int64_t base = wid * 4; base < O; base += warps * 4) {
        const int64_t f = base + sub;
        const bool live = f < O && j1 < J1;
        const double* src = t + f * plane + static_cast<int64_t>(J0) * j1;
        double x[JM];
        if (live && J0 == JM && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0)) {
#pragma unroll
            for (int v = 0; v < JM / 2; ++v) {
                const double2 p2 = __ldg(reinterpret_cast<const double2*>(src) + v);
                x[2 * v] = p2.x;
                x[2 * v + 1] = p2.y;
            }
        } else {
#pragma unroll
            for (int j0 = 0; j0 < JM; ++j0) x[j0] = (live && j0 < J0) ? __ldg(src + j0) : 0.0;
        }
        double tq[QM];
#pragma unroll
        for (int a = 0; a < QM; ++a) {
            double v = 0.0;
#pragma unroll
            for (int j0 = 0; j0 < JM; ++j0) v = fma(U0s[j0 * QM + a], x[j0], v);
            tq[a] = v;
        }
#pragma unroll
        for (int j0 = 0; j0 < JM; ++j0) ys = fma(x[j0], x[j0], ys);
        double acc[QM * QM];
#pragma unroll
        for (int a = 0; a < QM; ++a)
#pragma unroll
            for (int b = 0; b < QM; ++b) acc[a + QM * b] = tq[a] * U1s[j1 * QM + b];
        // butterfly reduce-scatter over the plane's 8 lanes: each step keeps
        // half of the entries and adds the partner's copy of that half; lane
        // j1 ends with acc entries 2*j1 and 2*j1 + 1 (8 + 4 + 2 shuffles)
        double h8[8], h4[4], h2[2];
        {
            const bool up = (j1 & 4) != 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double other = __shfl_xor_sync(0xffffffffu, up ? acc[i] : acc[i + 8], 4);
                h8[i] = (up ? acc[i + 8] : acc[i]) + other;
            }
        }
        {
            const bool up = (j1 & 2) != 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double other = __shfl_xor_sync(0xffffffffu, up ? h8[i] : h8[i + 4], 2);
                h4[i] = (up ? h8[i + 4] : h8[i]) + other;
            }
        }
        {
            const bool up = (j1 & 1) != 0;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const double other = __shfl_xor_sync(0xffffffffu, up ? h4[i] : h4[i + 2], 1);
                h2[i] = (up ? h4[i + 2] : h4[i]) + other;
            }
        }
        if (f < O) {
            double* dst = out + f * QQ;
            if (Q0 == QM && Q1 == QM) {  // compact block == acc layout: one 16-byte store
                *reinterpret_cast<double2*>(dst + 2 * j1) = make_double2(h2[0], h2[1]);
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int kk = 2 * j1 + h, a = kk % QM, b = kk / QM;
                    if (a < Q0 && b < Q1) dst[a + Q0 * b] = h2[h];
                }
            }
        }
    }
    if (ysq) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ys += __shfl_xor_sync(0xffffffffu, ys, off);
        if (lane == 0) red[threadIdx.x >> 5] = ys;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
            ysq[blockIdx.x] = tot;
        }
    }
}

int blocks_for(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096))); }

}  // namespace

void launch_sumsq(const double* x, int64_t n, double* partials, double* out, cudaStream_t s, int64_t* launches) {
    const int nb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kReduceBlocks / 2, (n + 511) / 512)));
    sumsq_kernel<<<nb, 256, 0, s>>>(x, n, partials);
    sumsq_finish_kernel<<<1, 32, 0, s>>>(partials, nb, out);
    *launches += 2;
}

void launch_sum_partials(const double* partials, int64_t n, double* out, cudaStream_t s, int64_t* launches) {
    sum_partials_kernel<<<1, 32, 0, s>>>(partials, n, out);
    ++*launches;
}

void launch_rank_rule(const double* lambda, int64_t k, int64_t n, double eps_abs, int64_t min_rank,
                      const double* trace_src, double* info, cudaStream_t s, int64_t* launches) {
    rank_rule_kernel<<<1, 32, 0, s>>>(lambda, k, n, eps_abs, min_rank, trace_src, info);
    ++*launches;
}

void launch_take_columns(const double* V, int64_t n, int64_t r, double* U, const double* info, cudaStream_t s,
                         int64_t* launches) {
    if (n * r == 0) return;
    take_columns_kernel<<<blocks_for(n * r), 256, 0, s>>>(V, n, r, U, info);
    ++*launches;
}

void launch_pad_axis(const double* src, int64_t inner, int64_t ext, int64_t outer, int64_t extra, double* dst,
                     cudaStream_t s, int64_t* launches) {
    const int64_t total = inner * (ext + extra) * outer;
    if (total == 0) return;
    pad_axis_kernel<<<blocks_for(total), 256, 0, s>>>(src, inner, ext, outer, extra, dst);
    ++*launches;
}

void launch_unfold(const double* src, int64_t inner, int64_t ext, int64_t outer, double* dst, cudaStream_t s,
                   int64_t* launches) {
    const int64_t total = inner * ext * outer;
    if (total == 0) return;
    unfold_kernel<<<blocks_for(total), 256, 0, s>>>(src, inner, ext, outer, dst);
    ++*launches;
}

int launch_mode_small(const double* t, int64_t I, int64_t J, int64_t O, const double* M, int64_t Q, int64_t smq,
                      int64_t smj, double* out, double* energy, double* ysq, int num_sms, cudaStream_t s,
                      int64_t* launches) {
    if (J > 32 || Q > 32) return -1;
    const bool mode0 = I == 1;
    const int64_t units = mode0 ? (O + 31) / 32 * 32 : I * O;
    const int per_block = mode0 ? 128 : 256;
    const int blocks = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>((units + per_block - 1) / per_block, 8 * num_sms)));
    const int jm = J <= 4 ? 4 : J <= 8 ? 8 : J <= 16 ? 16 : 32;
    const int qm = Q <= 4 ? 4 : Q <= 8 ? 8 : Q <= 16 ? 16 : 32;
#define HTR_SMALL(JJ, QQ)                                                                                       \
    if (jm == JJ && qm == QQ) {                                                                                 \
        if (mode0)                                                                                              \
            mode_small_kernel<JJ, QQ, true><<<blocks, 128, 0, s>>>(t, I, static_cast<int>(J), O, M,              \
                                                                    static_cast<int>(Q), smq, smj, out, energy, ysq); \
        else                                                                                                    \
            mode_small_kernel<JJ, QQ, false><<<blocks, 256, 0, s>>>(t, I, static_cast<int>(J), O, M,             \
                                                                     static_cast<int>(Q), smq, smj, out, energy, ysq); \
        ++*launches;                                                                                            \
        return blocks;                                                                                          \
    }
    HTR_SMALL(4, 4) HTR_SMALL(4, 8) HTR_SMALL(4, 16) HTR_SMALL(4, 32)
    HTR_SMALL(8, 4) HTR_SMALL(8, 8) HTR_SMALL(8, 16) HTR_SMALL(8, 32)
    HTR_SMALL(16, 4) HTR_SMALL(16, 8) HTR_SMALL(16, 16) HTR_SMALL(16, 32)
    HTR_SMALL(32, 4) HTR_SMALL(32, 8) HTR_SMALL(32, 16) HTR_SMALL(32, 32)
#undef HTR_SMALL
    return -1;
}

int launch_pair_project(const double* t, int64_t I, int64_t J0, int64_t J1, int64_t O, const double* U0, int64_t Q0,
                        const double* U1, int64_t Q1, double* out, double* ysq, int num_sms, cudaStream_t s,
                        int64_t* launches) {
    if (J0 > 8 || J1 > 8 || Q0 > 4 || Q1 > 4) return -1;
    if (I == 1) {
        const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((O + 31) / 32, 8 * num_sms)));
        pair_project_contig_kernel<<<blocks, 256, 0, s>>>(t, static_cast<int>(J0), static_cast<int>(J1), O, U0,
                                                          static_cast<int>(Q0), U1, static_cast<int>(Q1), out, ysq);
        ++*launches;
        return blocks;
    }
    const int64_t planes = I * O;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((planes + 255) / 256, 8 * num_sms)));
    pair_project_kernel<8, 8, 4, 4><<<blocks, 256, 0, s>>>(t, I, static_cast<int>(J0), static_cast<int>(J1), O, U0,
                                                           static_cast<int>(Q0), U1, static_cast<int>(Q1), out, ysq);
    ++*launches;
    return blocks;
}

void launch_basis_defect(const double* const* U, const int64_t* alpha, const int64_t* r, int count, double* out,
                         cudaStream_t s, int64_t* launches) {
    for (int i0 = 0; i0 < count; i0 += kDefectMax) {
        DefectJobs jobs{};
        const int n = std::min(kDefectMax, count - i0);
        for (int i = 0; i < n; ++i) {
            jobs.U[i] = U[i0 + i];
            jobs.alpha[i] = alpha[i0 + i];
            jobs.r[i] = U[i0 + i] ? r[i0 + i] : 0;
        }
        basis_defect_kernel<<<n, 256, 0, s>>>(jobs, out + i0);
        ++*launches;
    }
}

// ---- per-field normalisation (metrics.hpp:93-197) ---------------------------
// The tensor as runs of `inner` elements cycling through F fields (field f of
// flat index e is (e / inner) % F). Each thread walks its grid-stride
// elements tracking (position in run, field) incrementally; per-field
// accumulators live in shared memory [field][thread] (fields [f0, f0 + nf),
// nf <= 16), reduced per CTA in a fixed order, then over CTAs.
constexpr int kFieldThreads = 256;
constexpr int kFieldMax = 16;

__global__ void __launch_bounds__(kFieldThreads) field_stat_kernel(const double* __restrict__ x, int64_t n,
                                                                   int64_t inner, int F, int kind,
                                                                   const double* __restrict__ mu, int f0, int nf,
                                                                   double* __restrict__ partials) {
    __shared__ double acc[kFieldMax][kFieldThreads];
    const int tid = threadIdx.x;
    for (int f = 0; f < nf; ++f) acc[f][tid] = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kFieldThreads;
    int64_t e = blockIdx.x * static_cast<int64_t>(kFieldThreads) + tid;
    int64_t r = e % inner;
    int f = static_cast<int>((e / inner) % F);
    const int64_t dr = stride % inner;
    const int df = static_cast<int>((stride / inner) % F);
    for (; e < n; e += stride) {
        const int lf = f - f0;
        if (lf >= 0 && lf < nf) {
            const double v = x[e];
            double& a = acc[lf][tid];
            if (kind == 0) a = fmax(a, fabs(v));
            else if (kind == 1) a = fma(v, v, a);
            else if (kind == 2) a += v;
            else {
                const double d = v - mu[f];
                a = fma(d, d, a);
            }
        }
        r += dr;
        f += df;
        if (r >= inner) {
            r -= inner;
            ++f;
        }
        if (f >= F) f -= F;
    }
    __syncthreads();
    // field lf: 32 lanes of warp (lf % warps) sum its 256 thread slots in a fixed tree
    const int warp = tid >> 5, lane = tid & 31, nw = kFieldThreads / 32;
    for (int lf = warp; lf < nf; lf += nw) {
        double v = kind == 0 ? 0.0 : 0.0;
        for (int t = lane; t < kFieldThreads; t += 32) v = kind == 0 ? fmax(v, acc[lf][t]) : v + acc[lf][t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(0xffffffffu, v, o);
            v = kind == 0 ? fmax(v, w) : v + w;
        }
        if (lane == 0) partials[static_cast<int64_t>(blockIdx.x) * nf + lf] = v;
    }
}

__global__ void field_finish_kernel(const double* __restrict__ partials, int nparts, int nf, int kind,
                                    double* __restrict__ out) {
    const int lf = blockIdx.x;
    double v = 0.0;
    for (int p = threadIdx.x; p < nparts; p += 32) {
        const double w = partials[static_cast<int64_t>(p) * nf + lf];
        v = kind == 0 ? fmax(v, w) : v + w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = kind == 0 ? fmax(v, w) : v + w;
    }
    if (threadIdx.x == 0) out[lf] = v;
}

__global__ void field_apply_kernel(const double* __restrict__ x, int64_t n, int64_t inner, int F,
                                   const double* __restrict__ mu, const double* __restrict__ sc, int inverse,
                                   double* __restrict__ out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    int64_t r = e % inner;
    int f = static_cast<int>((e / inner) % F);
    const int64_t dr = stride % inner;
    const int df = static_cast<int>((stride / inner) % F);
    for (; e < n; e += stride) {
        const double m = mu ? mu[f] : 0.0;
        out[e] = inverse ? fma(x[e], sc[f], m) : (x[e] - m) / sc[f];
        r += dr;
        f += df;
        if (r >= inner) {
            r -= inner;
            ++f;
        }
        if (f >= F) f -= F;
    }
}

int field_stat_blocks(int num_sms) { return 2 * num_sms; }

void launch_field_stat(const double* x, int64_t n, int64_t inner, int F, int kind, const double* mu, double* partials,
                       double* out, int num_sms, cudaStream_t s, int64_t* launches) {
    const int grid = field_stat_blocks(num_sms);
    for (int f0 = 0; f0 < F; f0 += kFieldMax) {
        const int nf = std::min(kFieldMax, F - f0);
        field_stat_kernel<<<grid, kFieldThreads, 0, s>>>(x, n, inner, F, kind, mu, f0, nf, partials);
        field_finish_kernel<<<nf, 32, 0, s>>>(partials, grid, nf, kind, out + f0);
        *launches += 2;
    }
}

void launch_field_apply(const double* x, int64_t n, int64_t inner, int F, const double* mu, const double* sc,
                        bool inverse, double* out, int num_sms, cudaStream_t s, int64_t* launches) {
    if (n == 0) return;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4 * num_sms, (n + 255) / 256)));
    field_apply_kernel<<<grid, 256, 0, s>>>(x, n, inner, F, mu, sc, inverse ? 1 : 0, out);
    ++*launches;
}

constexpr int kPermMax = 16;
struct PermArgs {
    int d;
    int64_t out_ext[kPermMax];
    int64_t src_stride[kPermMax];  // stride in the source of output mode k
};

__global__ void permute_kernel(const double* __restrict__ src, int64_t n, const __grid_constant__ PermArgs a,
                               double* __restrict__ dst) {
    for (int64_t flat = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; flat < n;
         flat += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t rem = flat, off = 0;
        for (int k = 0; k < a.d; ++k) {
            const int64_t e = a.out_ext[k];
            const int64_t i = rem % e;
            rem /= e;
            off += i * a.src_stride[k];
        }
        dst[flat] = src[off];
    }
}

void launch_permute(const double* src, const int64_t* shape, int d, const int64_t* perm, double* dst, cudaStream_t s,
                    int64_t* launches) {
    PermArgs a{};
    a.d = d;
    int64_t in_stride[kPermMax];
    int64_t acc = 1, n = 1;
    for (int k = 0; k < d; ++k) {
        in_stride[k] = acc;
        acc *= shape[k];
    }
    for (int k = 0; k < d; ++k) {
        a.out_ext[k] = shape[perm[k]];
        a.src_stride[k] = in_stride[perm[k]];
        n *= a.out_ext[k];
    }
    if (n == 0) return;
    permute_kernel<<<blocks_for(n), 256, 0, s>>>(src, n, a, dst);
    ++*launches;
}

void launch_fill(double* dst, int64_t n, double value, cudaStream_t s, int64_t* launches) {
    if (n == 0) return;
    fill_kernel<<<blocks_for(n), 256, 0, s>>>(dst, n, value);
    ++*launches;
}

}  // namespace htr
