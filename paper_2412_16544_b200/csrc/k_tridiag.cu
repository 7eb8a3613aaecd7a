// Symmetric eigen-truncation through a tridiagonal reduction: the device
// replacement of the reference's thin SVD (Eigen::BDCSVD,
// truncated_svd.hpp:29-45) on the Gram G = M M^T of an unfolding.
//
//   tridiag_eigvals_kernel   one CTA per Gram: Householder reduction
//                            Q^T G Q = T (the matrix in shared memory up to
//                            n = 160, else in the L2-resident workspace),
//                            then every eigenvalue of T by parallel
//                            multisection on Sturm counts (8 lanes per
//                            eigenvalue). Writes lambda (descending) and the
//                            reflectors / T into the workspace.
//   tridiag_vectors_kernel   one CTA per Gram, after the rank rule: the r
//                            leading eigenvectors of T by inverse iteration
//                            (a warp per cluster of close eigenvalues,
//                            re-orthogonalised within the cluster as LAPACK
//                            dstein does), then U = Q Z by applying the
//                            reflectors column-parallel (no block barrier).
//
// The reference's rank rule needs the eigenvalues to absolute accuracy
// ~u ||G|| (the Gram itself carries ~n u ||G|| of rounding), which the
// backward-stable reduction plus bisection to ~2 ulp of ||T|| provides; only
// the retained subspace's basis is formed (any orthonormal basis of it is a
// valid truncated_svd factor up to rotation; parity is checked by principal
// angles). Everything is deterministic (fixed reduction trees, no atomics),
// so ranks of a sharded run, which solve bit-identical Grams, agree.
#include <algorithm>
#include <cfloat>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kTriThreads = 1024;
constexpr int kTriSmemMaxN = 160;  // A (n x n) in shared memory: 200 KB at n = 160
constexpr int kTriBatch = 16;
constexpr int kVecThreads = 512;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

/// Sum over the CTA, the same value (same bits) in every thread.
__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();  // red is free
    if (lane == 0) red[w] = v;
    __syncthreads();
    return warp_sum(lane < nw ? red[lane] : 0.0);
}
__device__ double block_max(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    return warp_max(lane < nw ? red[lane] : -DBL_MAX);
}
__device__ double block_min(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_min(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    return warp_min(lane < nw ? red[lane] : DBL_MAX);
}

// workspace layout per job (doubles): [A n*n | d n | e n | tau n | lam_asc n | scale 1]
__host__ __device__ __forceinline__ int64_t tri_off_d(int n) { return static_cast<int64_t>(n) * n; }

struct TriJobs {
    const double* G[kTriBatch];
    double* lam[kTriBatch];  // n eigenvalues, descending (unscaled)
    double* W[kTriBatch];    // workspace, tridiag_workspace_doubles(n)
    int n[kTriBatch];
};

/// Number of eigenvalues of T (d, e2 = e^2) below x (Sturm count on the LDL^T
/// pivots, LAPACK dlaebz's pivmin safeguard).
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    double q = d[0] - x;
    if (fabs(q) <= pivmin) q = -pivmin;
    int c = q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = (d[i] - x) - e2[i - 1] / q;
        if (fabs(q) <= pivmin) q = -pivmin;
        c += q < 0.0;
    }
    return c;
}

/// The Householder scalars of a column (alpha its first entry, xn2 the squared
/// norm of the rest): hs[0] = tau, hs[1] = 1 / (alpha - beta), hs[2] = beta.
/// FP64 sqrt and divisions are long instruction sequences; they are computed
/// by one thread and read by everyone (all 32 warps computing them
/// redundantly cost more issue slots per step than the matrix update).
__device__ __forceinline__ void house_scalars(double alpha, double xn2, double* hs) {
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (xn2 > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
    }
    hs[0] = tau;
    hs[1] = scale;
    hs[2] = beta;
}

/// Householder reduction Q^T G Q = T (dsytd2, lower) of one Gram per CTA.
/// Three block barriers per column: the reflector is formed from the
/// column's norm (accumulated by the previous column's update), the
/// matrix-vector product p = tau A22 v also accumulates p . v per warp, and
/// the rank-2 update A22 -= v w^T + w v^T (w = p - K v formed on the fly)
/// also accumulates the next column's norm. Writes d, e, tau, the
/// reflectors (below the subdiagonal of the workspace matrix) and the scale.
/// T > 0: every row of the trailing matrix is held by one lane as
/// i = lane + 32 t, t < T (n <= 32 T + 1), with v and w in registers; T = 0:
/// strided loops (the global-memory path, larger n).
template <int T>
__global__ void __launch_bounds__(kTriThreads) tridiag_reduce_kernel(const __grid_constant__ TriJobs jobs,
                                                                     int use_smem) {
    const int n = jobs.n[blockIdx.x];
    const double* __restrict__ G = jobs.G[blockIdx.x];
    double* __restrict__ W = jobs.W[blockIdx.x];
    extern __shared__ double smem[];
    __shared__ double red[32];
    __shared__ double pdp[32];
    __shared__ double hs[4];  // the current column's tau, scale, beta (house_scalars)
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int64_t nn = static_cast<int64_t>(n) * n;
    double* A = use_smem ? smem : W;
    double* vv = use_smem ? smem + nn : W + tri_off_d(n) + 5 * n + 1;  // 2 vectors of n
    double* pw = vv + n;
    double* dg = W + tri_off_d(n);
    double* eg = dg + n;
    double* taug = eg + n;

    // exact power-of-two scaling to max |G| ~ 1 (no overflow in the norms)
    double gm = 0.0;
    for (int64_t i = tid; i < nn; i += nt) gm = fmax(gm, fabs(G[i]));
    gm = block_max(gm, red);
    int ex = 0;
    if (gm > 0.0 && gm <= DBL_MAX) frexp(gm, &ex);
    const double sc = ldexp(1.0, -ex), unsc = ldexp(1.0, ex);
    for (int c = 0; c < n; ++c)
        for (int r = tid; r < n; r += nt) A[r + static_cast<int64_t>(n) * c] = 0.5 * (G[r + static_cast<int64_t>(n) * c] + G[c + static_cast<int64_t>(n) * r]) * sc;
    __syncthreads();
    double xn2 = 0.0;
    if (n > 2) {
        double ps = 0.0;
        for (int i = 2 + tid; i < n; i += nt) ps = fma(A[i], A[i], ps);
        xn2 = block_sum(ps, red);
    }
    if (tid == 0 && n > 2) house_scalars(A[1], xn2, hs);
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
        double* x = A + (k + 1) + static_cast<int64_t>(n) * k;
        // written for this column by the previous step (the warp that updated
        // it) before that step's closing barrier; rewritten after this step's
        // second barrier
        const double tau = hs[0], scale = hs[1], beta = hs[2];
        for (int i = tid; i < m; i += nt) {
            const double vi = i == 0 ? 1.0 : x[i] * scale;
            vv[i] = vi;
            if (i > 0) x[i] = vi;  // reflector stored below the subdiagonal
        }
        if (tid == 0) {
            x[0] = beta;
            taug[k] = tau;
        }
        __syncthreads();
        double* A22 = A + (k + 1) + static_cast<int64_t>(n) * (k + 1);
        if (tau == 0.0) {
            // nothing to update; the next column's norm directly
            double ps = 0.0;
            for (int i = 2 + tid; i < m; i += nt) ps = fma(A22[i], A22[i], ps);
            xn2 = block_sum(ps, red);
            if (tid == 0 && m >= 2) house_scalars(A22[1], xn2, hs);
            __syncthreads();
            continue;
        }
        // p = tau A22 v (column j dotted with v), and p . v per warp
        double pdw = 0.0;
        if constexpr (T > 0) {
            double vr[T];
#pragma unroll
            for (int t = 0; t < T; ++t) vr[t] = lane + 32 * t < m ? vv[lane + 32 * t] : 0.0;
            for (int j = warp; j < m; j += nw) {
                const double* col = A22 + static_cast<int64_t>(n) * j;
                double s = 0.0;
#pragma unroll
                for (int t = 0; t < T; ++t)
                    if (lane + 32 * t < m) s = fma(col[lane + 32 * t], vr[t], s);
                s = tau * warp_sum(s);
                if (lane == 0) pw[j] = s;
                pdw = fma(s, vv[j], pdw);
            }
            if (lane == 0) pdp[warp] = pdw;
            __syncthreads();
            const double K = 0.5 * tau * warp_sum(lane < nw ? pdp[lane] : 0.0);
            double wr[T];
#pragma unroll
            for (int t = 0; t < T; ++t) wr[t] = lane + 32 * t < m ? fma(-K, vr[t], pw[lane + 32 * t]) : 0.0;
            // A22 -= v w^T + w v^T with w = p - K v; the warp holding column 0
            // (the next column to reduce) also sums its rows >= 2 squared
            for (int j = warp; j < m; j += nw) {
                double* col = A22 + static_cast<int64_t>(n) * j;
                const double vj = vv[j], wj = fma(-K, vj, pw[j]);
                double s = 0.0, a0 = 0.0;  // a0: the updated entry i = lane (t = 0)
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const int i = lane + 32 * t;
                    if (i < m) {
                        const double a = col[i] - fma(vr[t], wj, wr[t] * vj);
                        col[i] = a;
                        if (t == 0) a0 = a;
                        if (i >= 2) s = fma(a, a, s);
                    }
                }
                if (j == 0) {
                    // the next column: its head (row 1) and the rest's norm
                    s = warp_sum(s);
                    const double head = __shfl_sync(0xffffffffu, a0, 1);
                    if (lane == 0) house_scalars(head, s, hs);
                }
            }
        } else {
            for (int j = warp; j < m; j += nw) {
                const double* col = A22 + static_cast<int64_t>(n) * j;
                double s = 0.0;
                for (int i = lane; i < m; i += 32) s = fma(col[i], vv[i], s);
                s = tau * warp_sum(s);
                if (lane == 0) pw[j] = s;
                pdw = fma(s, vv[j], pdw);
            }
            if (lane == 0) pdp[warp] = pdw;
            __syncthreads();
            const double K = 0.5 * tau * warp_sum(lane < nw ? pdp[lane] : 0.0);
            for (int j = warp; j < m; j += nw) {
                double* col = A22 + static_cast<int64_t>(n) * j;
                const double vj = vv[j], wj = fma(-K, vj, pw[j]);
                double s = 0.0, a0 = 0.0;
                for (int i = lane; i < m; i += 32) {
                    const double wi = fma(-K, vv[i], pw[i]);
                    const double a = col[i] - fma(vv[i], wj, wi * vj);
                    col[i] = a;
                    if (i == lane) a0 = a;
                    if (j == 0 && i >= 2) s = fma(a, a, s);
                }
                if (j == 0) {
                    s = warp_sum(s);
                    const double head = __shfl_sync(0xffffffffu, a0, 1);
                    if (lane == 0) house_scalars(head, s, hs);
                }
            }
        }
        __syncthreads();
    }
    // T: diagonal and subdiagonal; reflectors to the workspace
    for (int i = tid; i < n; i += nt) {
        dg[i] = A[i + static_cast<int64_t>(n) * i];
        eg[i] = i + 1 < n ? A[i + 1 + static_cast<int64_t>(n) * i] : 0.0;
        if (i + 2 >= n) taug[i] = 0.0;
    }
    if (use_smem)
        for (int c = 0; c + 2 < n; ++c)
            for (int r = c + 2 + tid; r < n; r += nt) W[r + static_cast<int64_t>(n) * c] = A[r + static_cast<int64_t>(n) * c];
    if (tid == 0) W[tri_off_d(n) + 4 * n] = unsc;
}

/// Every eigenvalue of T by multisection on Sturm counts: one warp per
/// eigenvalue (32 points per step, 5 bits), 4 warps per CTA, CTAs of all
/// jobs side by side (grid.y = job). Absolute accuracy ~4 u ||T||.
constexpr int kBisWarps = 4;
__global__ void __launch_bounds__(kBisWarps * 32) tridiag_bisect_kernel(const __grid_constant__ TriJobs jobs) {
    const int job = blockIdx.y;
    const int n = jobs.n[job];
    const int j = blockIdx.x * kBisWarps + (threadIdx.x >> 5);
    if (blockIdx.x * kBisWarps >= n) return;
    const double* __restrict__ W = jobs.W[job];
    double* __restrict__ lam_out = jobs.lam[job];
    extern __shared__ double bsm[];  // d, e^2 (2 n doubles)
    double* d = bsm;
    double* e2 = bsm + n;
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const double* dg = W + tri_off_d(n);
    const double* eg = dg + n;
    const double unsc = W[tri_off_d(n) + 4 * n];
    double lo_g = DBL_MAX, hi_g = -DBL_MAX, emax = 0.0;
    for (int i = tid; i < n; i += nt) {
        const double di = dg[i], ei = i + 1 < n ? eg[i] : 0.0, em = i > 0 ? eg[i - 1] : 0.0;
        d[i] = di;
        e2[i] = ei * ei;
        const double r = fabs(em) + fabs(ei);
        lo_g = fmin(lo_g, di - r);
        hi_g = fmax(hi_g, di + r);
        emax = fmax(emax, ei * ei);
    }
    lo_g = block_min(lo_g, red);
    hi_g = block_max(hi_g, red);
    emax = block_max(emax, red);
    __syncthreads();
    if (j >= n) return;
    const double bnorm = fmax(fabs(lo_g), fabs(hi_g));
    const double pivmin = DBL_MIN * fmax(1.0, emax);
    const double atol = 4.0 * DBL_EPSILON * bnorm + pivmin;
    double lo = lo_g - (atol + 2.0 * DBL_EPSILON * bnorm * n);
    double hi = hi_g + (atol + 2.0 * DBL_EPSILON * bnorm * n);
    for (int it = 0; it < 40; ++it) {
        if (hi - lo <= fmax(atol, 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)))) break;  // warp-uniform
        const double xs = lo + (hi - lo) * (lane + 1) * (1.0 / 33.0);
        const int cnt = sturm_count(d, e2, n, xs, pivmin);
        const unsigned ball = __ballot_sync(0xffffffffu, cnt > j);
        const int p = ball ? __ffs(ball) - 1 : 32;
        const double xp = __shfl_sync(0xffffffffu, xs, p < 32 ? p : 31);
        const double xq = __shfl_sync(0xffffffffu, xs, p > 0 ? p - 1 : 0);
        const double nlo = p > 0 ? xq : lo;
        const double nhi = p < 32 ? xp : hi;
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) {
        const double l = 0.5 * (lo + hi);
        const_cast<double*>(W)[tri_off_d(n) + 3 * n + j] = l;  // ascending, scaled (inverse iteration)
        lam_out[n - 1 - j] = l * unsc;
    }
}

struct VecJobs {
    const double* W[kTriBatch];
    const double* info[kTriBatch];  // rank rule output: [2] = trace (0 -> zero input)
    double* U[kTriBatch];           // n x r
    int n[kTriBatch], r[kTriBatch];
};

/// (T - x I) y = b by Gaussian elimination with partial pivoting of the
/// tridiagonal matrix (one thread; LAPACK dlagtf/dlagts). Pivots below `tol`
/// in magnitude are perturbed to +-tol (inverse iteration's standard guard);
/// u0 holds the pivots' reciprocals.
struct TriLU {
    double *u0, *u1, *u2, *l;
    unsigned char* piv;
};
__device__ void tri_factor(const double* d, const double* e, int n, double x, double tol, const TriLU& f) {
    double p0 = d[0] - x, p1 = n > 1 ? e[0] : 0.0, p2 = 0.0;
    for (int k = 0; k + 1 < n; ++k) {
        const double q0 = e[k], q1 = d[k + 1] - x, q2 = k + 2 < n ? e[k + 1] : 0.0;
        if (fabs(p0) >= fabs(q0)) {
            if (fabs(p0) < tol) p0 = p0 < 0.0 ? -tol : tol;
            const double rp = 1.0 / p0;
            const double mult = q0 * rp;
            f.u0[k] = rp; f.u1[k] = p1; f.u2[k] = p2; f.l[k] = mult; f.piv[k] = 0;
            p0 = q1 - mult * p1;
            p1 = q2 - mult * p2;
        } else {
            const double mult = p0 / q0;
            f.u0[k] = 1.0 / q0; f.u1[k] = q1; f.u2[k] = q2; f.l[k] = mult; f.piv[k] = 1;
            const double np0 = p1 - mult * q1, np1 = p2 - mult * q2;
            p0 = np0;
            p1 = np1;
        }
        p2 = 0.0;
    }
    if (fabs(p0) < tol) p0 = p0 < 0.0 ? -tol : tol;
    f.u0[n - 1] = 1.0 / p0;
    f.u1[n - 1] = 0.0;
    f.u2[n - 1] = 0.0;
}
__device__ void tri_solve(int n, const TriLU& f, double* y) {
    double yk = y[0];
    for (int k = 0; k + 1 < n; ++k) {
        double yn = y[k + 1];
        if (f.piv[k]) {
            const double t = yk;
            yk = yn;
            yn = t;
        }
        y[k] = yk;
        yk = yn - f.l[k] * yk;
    }
    y[n - 1] = yk;
    double x1 = 0.0, x2 = 0.0;  // y[k + 1], y[k + 2]
    for (int k = n - 1; k >= 0; --k) {
        const double xk = (y[k] - f.u1[k] * x1 - f.u2[k] * x2) * f.u0[k];
        y[k] = xk;
        x2 = x1;
        x1 = xk;
    }
}

__device__ __forceinline__ double hash_uniform(uint32_t a, uint32_t b) {
    uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    return (static_cast<double>(h) + 0.5) * (2.0 / 4294967296.0) - 1.0;  // (-1, 1)
}

/// Reflectors staged in shared memory for the back-transform up to this n
/// (the strictly-below-subdiagonal part, column k at offset koff(k)).
constexpr int kVecSmemRefN = 128;
/// Above this n the vector kernel keeps T and its scratch in the workspace.
constexpr int kVecSmemN = 1024;
constexpr int kTriMaxN = 8192;
/// Clusters of 2..kBlockMax close eigenvalues are iterated by the whole CTA
/// (solves dealt to the warps, block re-orthonormalisation by CholeskyQR2).
constexpr int kBlockMax = 48;
constexpr int kBlockGramDoubles = kBlockMax * (kBlockMax + 1);
/// Eigenvectors built in shared memory up to n * r doubles (n <= 128).
__host__ __device__ __forceinline__ bool jobs_z_smem(int n, int r) { return n <= kVecSmemRefN && n * r <= 4096; }
__device__ __forceinline__ int refl_off(int k, int n) { return k * (n - 2) - (k * (k - 1)) / 2; }

__global__ void __launch_bounds__(kVecThreads) tridiag_vectors_kernel(const __grid_constant__ VecJobs jobs,
                                                                      int vec_warps) {
    const int n = jobs.n[blockIdx.x], r = jobs.r[blockIdx.x];
    const double* __restrict__ W = jobs.W[blockIdx.x];
    double* __restrict__ U = jobs.U[blockIdx.x];
    const bool zero = jobs.info[blockIdx.x][2] == 0.0;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    if (r <= 0) return;
    if (zero) {  // zero input: the reference's canonical identity columns (truncated_svd.hpp:66-72)
        for (int64_t i = tid; i < static_cast<int64_t>(n) * r; i += nt) U[i] = (i % n == i / n) ? 1.0 : 0.0;
        return;
    }
    extern __shared__ double smem[];
    const double* dg = W + tri_off_d(n);
    const double* eg = dg + n;
    const double* taug = eg + n;
    const double* lam_g = taug + n;
    // clusters of the r leading eigenvalues (ascending j = n - r .. n - 1):
    // eigenvalues closer than 1e-9 ||T||_1 are iterated together and
    // re-orthogonalised against each other (LAPACK dstein's scheme, with a
    // tighter cluster radius: vectors of eigenvalues further apart are
    // independent to ~u ||T|| / gap and the caller's CholeskyQR2 polish
    // makes them orthonormal within the retained span)
    // n > kVecSmemN: T, the cluster table and the per-warp scratch stay in
    // the (L2-resident) workspace instead of shared memory
    const bool big = n > kVecSmemN;
    double* wbig = const_cast<double*>(W) + tri_off_d(n) + 8 * n + 8;
    __shared__ int cstart_s[kVecSmemN + 1];
    __shared__ int ncl;
    int* cstart = big ? reinterpret_cast<int*>(wbig) : cstart_s;
    double* d = big ? const_cast<double*>(dg) : smem;
    double* e = big ? const_cast<double*>(eg) : smem + n;
    double* lam_asc = big ? const_cast<double*>(lam_g) : smem + 2 * n;
    const bool refl_smem = n <= kVecSmemRefN;
    double* refl = smem + 3 * n;  // staged reflectors (n <= kVecSmemRefN)
    const int nrefl = refl_smem && n > 2 ? refl_off(n - 2, n) : 0;
    // the eigenvectors are formed in shared memory when they fit (z_smem)
    double* Z = smem + 3 * n + nrefl;
    const bool z_smem = jobs_z_smem(n, r);
    double* Zc = z_smem ? Z : U;
    for (int i = tid; i < n && !big; i += nt) {
        d[i] = dg[i];
        e[i] = eg[i];
        lam_asc[i] = lam_g[i];
    }
    // (one flat loop over the (n - 2) x (n - 2) index square: every thread has
    // its loads in flight at once instead of one short column per iteration)
    if (refl_smem && n > 2) {
        const int q = n - 2;
        for (int idx = tid; idx < q * q; idx += nt) {
            const int k = idx / q, i = idx - k * q;
            if (i < q - k) refl[refl_off(k, n) + i] = W[(k + 2 + i) + static_cast<int64_t>(n) * k];
        }
    }
    __syncthreads();
    __shared__ double onenrm;
    if (tid == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i)
            t = fmax(t, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0));
        onenrm = t;
        const double ortol = 1e-9 * t;
        int c = 0;
        for (int j = n - r; j < n; ++j)
            if (j == n - r || lam_asc[j] - lam_asc[j - 1] > ortol) cstart[c++] = j;
        cstart[c] = n;
        ncl = c;
    }
    __syncthreads();
    const double tol = fmax(DBL_EPSILON * onenrm, DBL_MIN);
    // per-warp scratch: u0 u1 u2 l y (5 n doubles) + piv (n bytes)
    double* scratch = big ? wbig + (n + 2) : Z + (z_smem ? n * r : 0);
    const int per = 5 * n + (n + 7) / 8;
    // normalise v (n values, warp-wide), the largest entry made positive when `sign`
    auto normalise = [&](double* v, bool sign) {
        double s = 0.0, mx = 0.0;
        int imx = 0;
        for (int i = lane; i < n; i += 32) {
            s = fma(v[i], v[i], s);
            if (fabs(v[i]) > mx) { mx = fabs(v[i]); imx = i; }
        }
        s = warp_sum(s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double om = __shfl_xor_sync(0xffffffffu, mx, o);
            const int oi = __shfl_xor_sync(0xffffffffu, imx, o);
            if (om > mx || (om == mx && oi < imx)) { mx = om; imx = oi; }
        }
        double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
        if (sign && v[imx] < 0.0) inv = -inv;
        __syncwarp();
        for (int i = lane; i < n; i += 32) v[i] *= inv;
        __syncwarp();
    };
    // clusters the whole CTA iterates together (below): 2..kBlockMax members
    // with the vectors in shared memory; larger ones stay with one warp
    auto block_cluster = [&](int cl) {
        const int m = cstart[cl + 1] - cstart[cl];
        return !big && m > 1 && m <= kBlockMax;
    };
    for (int cl = warp; cl < ncl && warp < vec_warps; cl += vec_warps) {
        double* ws = scratch + static_cast<int64_t>(warp) * per;
        TriLU f{ws, ws + n, ws + 2 * n, ws + 3 * n, reinterpret_cast<unsigned char*>(ws + 5 * n)};
        const int j0 = cstart[cl], j1 = cstart[cl + 1];
        if (block_cluster(cl)) continue;
        if (j1 - j0 == 1) {
            // an isolated eigenvalue: two inverse-iteration steps
            double* y = Zc + static_cast<int64_t>(n) * (n - 1 - j0);
            if (lane == 0) tri_factor(d, e, n, lam_asc[j0], tol, f);
            for (int i = lane; i < n; i += 32) y[i] = hash_uniform(static_cast<uint32_t>(j0), static_cast<uint32_t>(i));
            __syncwarp();
            for (int it = 0; it < 2; ++it) {
                if (lane == 0) tri_solve(n, f, y);
                __syncwarp();
                normalise(y, it == 1);
            }
            continue;
        }
        // a cluster: block inverse iteration -- every member solved from its
        // current vector, then the block re-orthonormalised (modified
        // Gram-Schmidt, twice) -- so that no member is formed from the small
        // remainder of a vector already inside its predecessors' span
        // (which would leave rounding-level noise as a large component)
        for (int j = j0; j < j1; ++j) {
            double* y = Zc + static_cast<int64_t>(n) * (n - 1 - j);
            for (int i = lane; i < n; i += 32) y[i] = hash_uniform(static_cast<uint32_t>(j), static_cast<uint32_t>(i));
        }
        __syncwarp();
        for (int it = 0; it < 3; ++it) {
            double xprev = 0.0;
            for (int j = j0; j < j1; ++j) {
                double xj = lam_asc[j];
                if (j > j0) {  // separate coincident eigenvalues slightly (dstein)
                    const double pertol = 10.0 * fabs(DBL_EPSILON * xj);
                    if (xj - xprev < pertol) xj = xprev + pertol;
                }
                xprev = xj;
                double* y = Zc + static_cast<int64_t>(n) * (n - 1 - j);
                if (lane == 0) {
                    tri_factor(d, e, n, xj, tol, f);
                    tri_solve(n, f, y);
                }
                __syncwarp();
                normalise(y, false);
            }
            for (int j = j0; j < j1; ++j) {
                double* y = Zc + static_cast<int64_t>(n) * (n - 1 - j);
                for (int pass = 0; pass < 2; ++pass)
                    for (int p = j0; p < j; ++p) {
                        const double* up = Zc + static_cast<int64_t>(n) * (n - 1 - p);
                        double s = 0.0;
                        for (int i = lane; i < n; i += 32) s = fma(up[i], y[i], s);
                        s = warp_sum(s);
                        for (int i = lane; i < n; i += 32) y[i] -= s * up[i];
                        __syncwarp();
                    }
                normalise(y, it == 2);
            }
        }
    }
    __syncthreads();
    // ---- clusters iterated by the whole CTA: three rounds of (every member
    // solved from its current vector, one member per warp at a time; then the
    // block re-orthonormalised by CholeskyQR2: S = Y^T Y, S = R^T R, Y <- Y R^-1,
    // twice). The same scheme as the one-warp path above (solve all, then
    // Gram-Schmidt in member order -- CholeskyQR yields that same QR factor),
    // with the serial work spread over the CTA: a noise-floor cluster of 20
    // vectors of a 25-row Gram took 0.39 ms on one warp.
    if (!big) {
        double* S = scratch + static_cast<int64_t>(vec_warps) * per;  // [m][m + 1]
        for (int cl = 0; cl < ncl; ++cl) {
            if (!block_cluster(cl)) continue;
            const int j0 = cstart[cl], j1 = cstart[cl + 1], m = j1 - j0, sp = m + 1;
            // member q (eigenvalue j0 + q) is column n - 1 - j0 - q: Yb[-n q]
            double* Yb = Zc + static_cast<int64_t>(n) * (n - 1 - j0);
            for (int e = tid; e < n * m; e += nt) {
                const int q = e / n, i = e - q * n;
                Yb[i - static_cast<int64_t>(n) * q] = hash_uniform(static_cast<uint32_t>(j0 + q), static_cast<uint32_t>(i));
            }
            __syncthreads();
            for (int it = 0; it < 3; ++it) {
                if (warp < vec_warps) {
                    double* ws = scratch + static_cast<int64_t>(warp) * per;
                    TriLU f{ws, ws + n, ws + 2 * n, ws + 3 * n, reinterpret_cast<unsigned char*>(ws + 5 * n)};
                    for (int q = warp; q < m; q += vec_warps) {
                        // coincident eigenvalues separated slightly (dstein): the
                        // shift of member q is at least 10 u |x| above member q - 1's
                        double xj = lam_asc[j0];
                        for (int t = 1; t <= q; ++t) {
                            const double xt = lam_asc[j0 + t], pertol = 10.0 * fabs(DBL_EPSILON * xt);
                            xj = xt - xj < pertol ? xj + pertol : xt;
                        }
                        double* y = Yb - static_cast<int64_t>(n) * q;
                        if (lane == 0) {
                            tri_factor(d, e, n, xj, tol, f);
                            tri_solve(n, f, y);
                        }
                        __syncwarp();
                        normalise(y, false);
                    }
                }
                __syncthreads();
                for (int pass = 0; pass < 2; ++pass) {
                    // S = Y^T Y (lower triangle)
                    for (int idx = tid; idx < m * m; idx += nt) {
                        const int p = idx / m, q = idx - p * m;
                        if (q > p) continue;
                        const double* yp = Yb - static_cast<int64_t>(n) * p;
                        const double* yq = Yb - static_cast<int64_t>(n) * q;
                        double acc = 0.0;
                        for (int i = 0; i < n; ++i) acc = fma(yp[i], yq[i], acc);
                        S[p * sp + q] = acc;
                    }
                    __syncthreads();
                    // Cholesky S = L L^T in place (one warp; R = L^T). A
                    // non-positive pivot (a numerically dependent member) is
                    // replaced by 1: that column keeps its current direction
                    // and the next round's solve separates it.
                    if (warp == 0) {
                        for (int k = 0; k < m; ++k) {
                            double dk = S[k * sp + k];
                            dk = dk > 0.0 ? sqrt(dk) : 1.0;
                            const double inv = 1.0 / dk;
                            __syncwarp();
                            for (int i = k + 1 + lane; i < m; i += 32) S[i * sp + k] *= inv;
                            if (lane == 0) S[k * sp + k] = dk;
                            __syncwarp();
                            for (int idx = lane; idx < (m - k - 1) * (m - k - 1); idx += 32) {
                                const int i = k + 1 + idx / (m - k - 1), j = k + 1 + idx % (m - k - 1);
                                if (j <= i) S[i * sp + j] = fma(-S[i * sp + k], S[j * sp + k], S[i * sp + j]);
                            }
                            __syncwarp();
                        }
                    }
                    __syncthreads();
                    // Y <- Y R^-1: row i of Y by forward substitution (column q
                    // needs the finished columns p < q), one thread per row
                    for (int i = tid; i < n; i += nt) {
                        for (int q = 0; q < m; ++q) {
                            double v = Yb[i - static_cast<int64_t>(n) * q];
                            for (int p = 0; p < q; ++p) v = fma(-Yb[i - static_cast<int64_t>(n) * p], S[q * sp + p], v);
                            Yb[i - static_cast<int64_t>(n) * q] = v / S[q * sp + q];
                        }
                    }
                    __syncthreads();
                }
            }
            // unit norm and a fixed sign (largest entry positive), a warp per member
            for (int q = warp; q < m; q += nt >> 5) normalise(Yb - static_cast<int64_t>(n) * q, true);
            __syncthreads();
        }
    }
    // U = H_0 H_1 ... H_{n-3} Z: 8 lanes per column, every reflector applied
    // last-to-first (no block barrier: a group owns its column)
    const int g = tid >> 3, gl = tid & 7, ngroups = nt >> 3;
    const unsigned gmask = 0xffu << (lane & ~7);
    for (int c0 = 0; c0 < r; c0 += ngroups) {
        const int c = c0 + g;
        const bool active = c < r;
        double* z = Zc + static_cast<int64_t>(n) * (active ? c : 0);
        if (!active) continue;
        for (int k = n - 3; k >= 0; --k) {
            const double tau = taug[k];
            if (tau == 0.0) continue;
            const int m = n - k - 1;
            const double* v = refl_smem ? refl + refl_off(k, n) - 1 : W + (k + 1) + static_cast<int64_t>(n) * k;
            double s = 0.0;
            for (int i = gl; i < m; i += 8) s = fma(i == 0 ? 1.0 : v[i], z[k + 1 + i], s);
            s += __shfl_xor_sync(gmask, s, 1);
            s += __shfl_xor_sync(gmask, s, 2);
            s += __shfl_xor_sync(gmask, s, 4);
            s *= tau;
            for (int i = gl; i < m; i += 8) z[k + 1 + i] -= s * (i == 0 ? 1.0 : v[i]);
            __syncwarp(gmask);
        }
    }
    if (z_smem) {
        __syncthreads();
        for (int e = tid; e < n * r; e += nt) U[e] = Z[e];
    }
}

}  // namespace

int64_t tridiag_workspace_doubles(int64_t n) {
    // + for n > kVecSmemN: the cluster table and 16 warps' inverse-iteration scratch
    const int64_t big = n > kVecSmemN ? (n + 2) + (kVecThreads / 32) * (5 * n + (n + 7) / 8) : 0;
    return n * n + 8 * n + 8 + big;
}

bool tridiag_supported(int64_t n) { return n >= 1 && n <= kTriMaxN; }

void launch_tridiag_eigvals(const double* const* G, const int64_t* n, double* const* lambda, double* const* W,
                            int count, cudaStream_t s, int64_t* launches) {
    for (int i0 = 0; i0 < count;) {
        // reduction: one launch per run of jobs with the same storage mode
        const bool sm = n[i0] <= kTriSmemMaxN;
        TriJobs jobs{};
        int k = 0;
        int64_t nmax = 0;
        while (i0 + k < count && k < kTriBatch && (n[i0 + k] <= kTriSmemMaxN) == sm) {
            jobs.G[k] = G[i0 + k];
            jobs.lam[k] = lambda[i0 + k];
            jobs.W[k] = W[i0 + k];
            jobs.n[k] = static_cast<int>(n[i0 + k]);
            nmax = std::max(nmax, n[i0 + k]);
            ++k;
        }
        const int T = sm ? static_cast<int>((nmax - 1 + 31) / 32) : 0;  // m = n - 1 rows at most
        // (small matrices: fewer threads, cheaper barriers and loop overhead)
        const int threads = nmax <= 32 ? 128 : (nmax <= 64 ? 256 : kTriThreads);
        const size_t smem = sm ? sizeof(double) * static_cast<size_t>(nmax * nmax + 2 * nmax) : 0;
        auto kfn = T == 0 ? tridiag_reduce_kernel<0>
                 : T == 1 ? tridiag_reduce_kernel<1>
                 : T == 2 ? tridiag_reduce_kernel<2>
                 : T == 3 ? tridiag_reduce_kernel<3>
                 : T == 4 ? tridiag_reduce_kernel<4>
                          : tridiag_reduce_kernel<5>;
        if (smem > 0) ensure_smem_limit(reinterpret_cast<const void*>(kfn), smem);
        kfn<<<k, threads, smem, s>>>(jobs, sm ? 1 : 0);
        // eigenvalues: a warp per eigenvalue over many CTAs
        dim3 grid(static_cast<unsigned>((nmax + kBisWarps - 1) / kBisWarps), static_cast<unsigned>(k));
        const size_t bsmem = sizeof(double) * static_cast<size_t>(2 * nmax);
        ensure_smem_limit(reinterpret_cast<const void*>(tridiag_bisect_kernel), bsmem);
        tridiag_bisect_kernel<<<grid, kBisWarps * 32, bsmem, s>>>(jobs);
        *launches += 2;
        i0 += k;
    }
}

void launch_tridiag_vectors(const double* const* W, const double* const* info, const int64_t* n, const int64_t* r,
                            double* const* U, int count, cudaStream_t s, int64_t* launches) {
    for (int i0 = 0; i0 < count;) {
        VecJobs jobs{};
        // a job above kVecSmemN runs alone (its memory lives in the workspace)
        int k = 0;
        while (i0 + k < count && k < kTriBatch && (k == 0 || (n[i0 + k] <= kVecSmemN && n[i0] <= kVecSmemN))) ++k;
        int64_t nmax = 1;
        for (int i = 0; i < k; ++i) {
            jobs.W[i] = W[i0 + i];
            jobs.info[i] = info[i0 + i];
            jobs.U[i] = U[i0 + i];
            jobs.n[i] = static_cast<int>(n[i0 + i]);
            jobs.r[i] = static_cast<int>(r[i0 + i]);
            nmax = std::max(nmax, n[i0 + i]);
        }
        // shared memory: d, e, the staged reflectors (n <= 128) and per-warp
        // inverse-iteration scratch
        const int64_t refl = nmax <= kVecSmemRefN && nmax > 2 ? (nmax - 2) * (nmax - 1) / 2 : 0;
        int64_t zs = 0;
        for (int i = 0; i < k; ++i)
            if (jobs_z_smem(jobs.n[i], jobs.r[i])) zs = std::max<int64_t>(zs, static_cast<int64_t>(jobs.n[i]) * jobs.r[i]);
        const int64_t per = 5 * nmax + (nmax + 7) / 8;
        const bool big = nmax > kVecSmemN;
        const int64_t budget = 200 * 1024 / 8 - 3 * nmax - refl - zs - kBlockGramDoubles;
        const int vw = big ? kVecThreads / 32
                           : static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kVecThreads / 32, budget / per)));
        const size_t smem =
            big ? 0 : sizeof(double) * static_cast<size_t>(3 * nmax + refl + zs + vw * per + kBlockGramDoubles);
        if (smem > 0) ensure_smem_limit(reinterpret_cast<const void*>(tridiag_vectors_kernel), smem);
        tridiag_vectors_kernel<<<k, kVecThreads, smem, s>>>(jobs, vw);
        ++*launches;
        i0 += k;
    }
}

}  // namespace htr
