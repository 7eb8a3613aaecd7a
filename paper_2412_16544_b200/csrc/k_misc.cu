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

void launch_fill(double* dst, int64_t n, double value, cudaStream_t s, int64_t* launches) {
    if (n == 0) return;
    fill_kernel<<<blocks_for(n), 256, 0, s>>>(dst, n, value);
    ++*launches;
}

}  // namespace htr
